// engine_dev.cuh — device context shared by the bookkeeping kernels.
#pragma once
#include "../../include/ppsd.h"
#include "kernels.cuh"

namespace ppsd {

// Everything the per-tick bookkeeping kernels need, in device memory so the
// captured graphs keep fixed arguments while buffers change per call.
struct TickCtx {
  Sched* sched;
  Work* work;
  Work* work_ar;
  int32_t* tokens;     // [max_ctx + 8] prompt + committed/drafted tokens
  uint64_t* pdig;      // ToyLM prefix digests [max_ctx + 9]
  uint64_t* chain_dig; // ToyLM per-slot chain digests
  TraceRow* trace;
  int64_t trace_cap;
  const __nv_bfloat16* embed;
  float* x;
  int32_t d;
  int32_t model;
  int32_t lo, hi;      // local stages
  // ToyLM parameters (toylm.py:55-60)
  int32_t n_layers, vocab;
  double beta;
  uint64_t toy_seed;
  // multi-rank exchange (null / 0 on a single-rank engine). A box is
  // kBoxHeader int32 words {exit_tok, final_tok, act_slot, act_pos} followed by
  // the d fp32 activation leaving this rank's last local stage.
  float* outbox;
  const float* inbox;   // world boxes, all-gathered by the caller
  int32_t box_words;
  int32_t box_logits;  // sampling across ranks: boxes also carry the exit and final logits [2][V]
  int32_t box_used;    // words of a box written / published (<= box_words, the stride)
  int32_t rank, world;
  int32_t owner_k, owner_S, owner_prev;  // ranks owning the exit stage, stage S, stage lo-1
  int32_t n_prompt;
  int32_t model_stages;  // S
  // sampling mode (mode == "sampling"): stream seeds and float64 scratch
  int32_t greedy;
  uint64_t draft_seed, commit_seed;  // derive_seed(rng.seed, "draft" | "commit")
  const float* logits32;  // transformer heads [2][V]
  double* logits64;       // ToyLM heads [2][V]
  double* pdist;          // per-chain draft distribution [nbuf][V]
  double* qbuf;           // target / sampling scratch [V]
  double* wbuf;           // residual scratch [V]
  // NVLink peer-store transport (p2p.cuh); p2p == 0: caller-driven all-gather
  int32_t p2p;
  float* const* peer_xbuf;  // [world] device pointers (IPC-mapped) of every rank's exchange buffer
  float* my_xbuf;           // this rank's exchange buffer
  uint64_t* xcount;         // exchange counter (device)
  int32_t* xerr;            // sticky p2p wait timeout flag (device)
  int32_t prefill_chunk; // prompt tokens per batched prefill launch (<= kMaxVec)
  // folded single-GPU execution (sched.h: sched_fold_plan): `work` carries
  // the launched chain's shallow stages + exit head, `work_deep` the deep
  // batch + final heads, gated by the graph conditional `cond`
  int32_t fold;
  Work* work_deep;
  unsigned long long cond;  // cudaGraphConditionalHandle of the folded tick graph
  int32_t has_cond;         // 0: deep part captured inline (PPSD_FOLD_COND=0, profiling)
  // folded stage range of one rank (sched.h: sched_rfold_plan; multi-rank,
  // greedy): deferred batches in activation rows rf_row0 .. rf_row0 + width
  int32_t rfold;
  int32_t rf_row0;
  // folded tick with a deep batch: the launched chain's exit head runs as
  // vector 0 of the batch's final-head launch, on a copy of its exit state in
  // row comb_row (the batch advances the chain's own row past the exit)
  int32_t fold_comb;
  int32_t comb_row;
  // transformer-layer exit head (ppsd_model_desc.exit_head_layer): the draft
  // is the norm head on that decoder layer's output for a COPY of the
  // exit-layer state (rows head_row..), so the chain's own state continues
  int32_t hl;               // 1: exit head has a decoder layer
  int32_t hl_layer;         // its global layer index (= n_layers)
  int32_t hl_split;         // layers before the exit (k*E): prefill runs [0, split), head, [split, N)
  int32_t head_row;         // first activation row of the head layer
  Work* work_head;          // the head layer's work (copy source in src_slot)
  Work* work_p2;            // prefill: layers [split, N) of the chunk
  Work* work_head_pf;  // prefill's exit-head layer (the tick's work_head may already be planned)
  // logits tap (ppsd_set_logits_tap, parity tests): single-rank transformer
  // decodes copy the exit / final logits row each head produced into
  // tap[(pos * 2 + which) * vocab], pos = the generated position it predicts
  // (1 .. tap_max); a later row for the same position overwrites, so after
  // the run each position holds the rows of its committed prefix
  float* tap;
  int32_t tap_max;
};

constexpr int kBoxHeader = 4;

struct ArCtl {
  int32_t j;           // token index being processed
  int32_t first_layer; // first local layer
  int32_t n_layers;    // local layer count
  int32_t end;         // batched prefill: tokens [0, end) are processed
};

// Draft-then-verify (EESD) round machine, pkg/src/specpipe/pipesim.py:435-551.
struct EesdState {
  int32_t gamma, k, S, per, dt, n_prompt, horizon, n_layers, exit_layer, model;
  double alpha;          // Bernoulli verdicts
  uint64_t verify_seed;
  uint64_t verify_counter;
  int32_t t, committed, accepts, rejects, drafted, done, error, len;  // len = sequence length
  int64_t trace_n;
  uint64_t draft_counter, commit_counter;  // sampling mode (_ToyVerifier streams)
};

__global__ void sched_tick_kernel(const TickCtx* ctxp, int begin);
__global__ void head_copy_kernel(const TickCtx* ctxp, const Work* wh);
__global__ void ar_begin_kernel(const TickCtx* ctxp, ArCtl* ctl, int with_head);
__global__ void ar_end_kernel(const TickCtx* ctxp, ArCtl* ctl, int with_head);
__global__ void toy_tick_kernel(const TickCtx* ctxp);
__global__ void pack_outbox_kernel(const TickCtx* ctxp, int prefill);
__global__ void rf_cond_kernel(const TickCtx* ctxp, unsigned long long handle);
__global__ void rf_gather_kernel(const TickCtx* ctxp);
__global__ void fold_exit_copy_kernel(const TickCtx* ctxp);
__global__ void mr_prefill_begin_kernel(const TickCtx* ctxp, ArCtl* ctl);
__global__ void p2p_wait_kernel(const TickCtx* ctxp);
__global__ void toy_ar_kernel(const TickCtx* ctxp, int n_prompt, int max_tokens);
__global__ void toy_alignment_kernel(const uint64_t* pdig, int n_layers, int exit_depth, int vocab,
                                     uint64_t toy_seed, double beta, double* scratch, double* minsum,
                                     int* agree);
__global__ void prefill_chunk_kernel(const TickCtx* ctxp, ArCtl* ctl);
__global__ void eesd_draft_begin_kernel(const TickCtx* ctxp, EesdState* es);
__global__ void eesd_draft_end_kernel(const TickCtx* ctxp, EesdState* es);
__global__ void eesd_verify_begin_kernel(const TickCtx* ctxp, EesdState* es);
__global__ void eesd_scan_kernel(const TickCtx* ctxp, EesdState* es);
__global__ void eesd_toy_round_kernel(const TickCtx* ctxp, EesdState* es);
__global__ void init_weight_kernel(__nv_bfloat16* dst, int layout, int tiled, long long rows, long long cols,
                                   uint64_t b0, uint64_t b1, uint64_t b2, float a0, float a1, float a2,
                                   int H, int KV, int hd);

}  // namespace ppsd
