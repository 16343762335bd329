/*
 * ppsd.h — C ABI of the B200 greedy PPSD decode engine (libppsd.so).
 *
 * This is the drop-in boundary for the reference's decode path. The reference
 * (`specpipe`, pure Python) exposes the path as Python functions; each entry
 * point below is what a ctypes binding inside the reference would call in
 * place of the named reference function (binding shown in INTEGRATION.md):
 *
 *   ppsd_engine_create   <- the (model, PipelineConfig) pair handed to
 *                           decode_ppsd: ToyLM(...) pkg/src/specpipe/toylm.py:55-68,
 *                           PipelineConfig(...) pkg/src/specpipe/pipesim.py:60-114
 *   ppsd_decode          <- decode_ppsd, pkg/src/specpipe/pipesim.py:595-633
 *                           (its machine: _ppsd_machine, pipesim.py:670-789)
 *   ppsd_decode_ar       <- decode_autoregressive, pkg/src/specpipe/pipesim.py:390-409
 *   ppsd_decode_eesd     <- simulate_eesd with a greedy model oracle,
 *                           pkg/src/specpipe/pipesim.py:435-551
 *   ppsd_simulate        <- simulate_ppsd with AcceptanceOracle.bernoulli,
 *                           pkg/src/specpipe/pipesim.py:571-592, 636-667
 *   ppsd_metrics         <- RunMetrics, pkg/src/specpipe/pipesim.py:235-275
 *   ppsd_trace_row       <- TraceRow / EventTrace, pkg/src/specpipe/pipesim.py:145-189
 *
 * Conventions: every function returns PPSD_OK (0) or a negative status;
 * PPSD_EINVAL maps to the reference's ValueError (pipesim.py:412-428, 76-99),
 * PPSD_ECUDA / PPSD_ESTATE to RuntimeError. ppsd_last_error() returns a
 * thread-local message for the last failure. Device pointers passed in are
 * BORROWED for the engine's lifetime; the engine owns only its KV pool,
 * activation slots and scheduler state. One host thread drives one engine.
 */
#ifndef PPSD_H
#define PPSD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPSD_OK 0
#define PPSD_EINVAL (-1)
#define PPSD_ECUDA (-2)
#define PPSD_ESTATE (-3)
#define PPSD_EUNSUPPORTED (-4)

#define PPSD_MODEL_BERNOULLI 0  /* schedule-only oracle, no model compute  */
#define PPSD_MODEL_TOYLM 1      /* the reference ToyLM, bit-exact on GPU    */
#define PPSD_MODEL_TRANSFORMER 2 /* Llama-style decoder, bf16 weights       */

/* trace row kinds, pipesim.py:47-51; verdicts "", "accept", "reject" */
#define PPSD_ACTIVATION 0
#define PPSD_DRAFT_TOKEN 1
#define PPSD_FINAL_TOKEN 2
#define PPSD_CHECK_TOKEN 3
#define PPSD_VERDICT_NONE 0
#define PPSD_VERDICT_ACCEPT 1
#define PPSD_VERDICT_REJECT 2
#define PPSD_NO_TOKEN (-1) /* the reference's `token=None` */

typedef struct ppsd_engine ppsd_engine;

typedef struct {
  int32_t kind;        /* PPSD_MODEL_* */
  int32_t n_layers;    /* N, pipesim.py:69 / toylm.py:57 */
  int32_t vocab;       /* V */
  /* transformer shape (ignored for other kinds) */
  int32_t d_model, n_heads, n_kv_heads, head_dim, ffn_dim;
  float rms_eps, rope_theta;
  int32_t kv_bf16;     /* 1: bf16 KV cache, 0: fp32 KV cache */
  int32_t max_ctx;     /* prompt + generated tokens capacity */
  /* ToyLM (toylm.py:55-68) */
  uint64_t toy_seed;
  double toy_misalignment;
  /* transformer exit head: 0 = norm head (exit RMSNorm + tied LM head);
   * 1 = one decoder layer (ppsd_weights.exit_layer, its own KV cache) on the
   * exit-layer state, then the norm head — the paper's main configuration
   * (PAPER.md:404-408). Single-device engines only. */
  int32_t exit_head_layer;
} ppsd_model_desc;

/* one decoder layer's weights (layouts as in ppsd_weights) */
typedef struct {
  const void* qkv;
  const void* o;
  const void* gu;
  const void* down;
  const float* attn_norm;
  const float* mlp_norm;
} ppsd_layer_weights;

/* Transformer weights, device pointers in the engine's physical layout
 * (see DESIGN.md §"Data layout"): bf16 matrices row-major [rows][cols],
 * q/k rows pair-interleaved for RoPE, gate/up rows interleaved. Arrays of
 * per-layer pointers are HOST arrays of length n_layers (entries for layers
 * that are not local to this engine may be NULL). */
typedef struct {
  const void* embed;        /* [V][d] bf16 */
  const void* lm_head;      /* [V][d] bf16, shared by the exit and final heads */
  const float* final_norm;  /* [d] */
  const float* exit_norm;   /* [d] */
  const void* const* w_qkv; /* [(H+2KV)*hd][d] bf16 */
  const void* const* w_o;   /* [d][H*hd]       bf16 */
  const void* const* w_gu;  /* [2*ffn][d]      bf16 */
  const void* const* w_down;/* [d][ffn]        bf16 */
  const float* const* attn_norm; /* [d] */
  const float* const* mlp_norm;  /* [d] */
  const float* rope_cos;    /* [max_ctx][hd/2] */
  const float* rope_sin;
  ppsd_layer_weights exit_layer;  /* exit_head_layer = 1: the exit head's decoder layer (exit stage's rank) */
} ppsd_weights;

typedef struct {
  int32_t n_layers, exit_depth;
  int32_t exit_stage;   /* 0 = default (1), pipesim.py:92-99 */
  int32_t comm_latency; /* pipesim.py:72, 107-110 */
  int32_t stage_lo, stage_hi; /* local stages (1-based, inclusive); 0,0 = all */
  int32_t device;
  int32_t schedule;     /* PPSD_SCHEDULE_*: how one device executes the machine */
} ppsd_pipeline_desc;

/* Execution schedule of a single-device engine (all stages local). Both give
 * the machine's exact tokens, metrics and trace; they differ in when the
 * stage forwards run:
 *   PIPELINED: every planned (stage, chain) forward in its tick, the stages'
 *              work grouped into one launch per layer slot;
 *   FOLDED:    shallow stages + exit head at launch, deep stages of all
 *              in-flight chains in one batched weight pass when a verdict
 *              needs them (greedy, or sampling with exit_stage 1);
 *   AUTO:      FOLDED where it applies and the batched GEMVs fit their
 *              registers (d_model <= 4096), else PIPELINED. */
#define PPSD_SCHEDULE_AUTO 0
#define PPSD_SCHEDULE_PIPELINED 1
#define PPSD_SCHEDULE_FOLDED 2

typedef struct {
  int64_t committed_tokens, ticks, accepts, rejects; /* RunMetrics order */
  int32_t alpha_valid;
  double alpha_all_measured, throughput, speedup_vs_ar;
  double decode_ms;     /* CUDA-event time of the decode loop (prefill excluded) */
  double prefill_ms;    /* CUDA-event time of the prompt prefill */
  int64_t gpu_launches; /* kernels this engine launched for the call */
  /* execution accounting (not RunMetrics): the schedule that ran
   * (PPSD_SCHEDULE_PIPELINED / FOLDED) and, folded, the deep batches, the
   * chains they carried and the sum of those chains' positions */
  int32_t schedule;
  int64_t deep_batches, deep_vectors, deep_pos_sum;
  /* folded: deep batches whose final-head pass also ran the launched chain's
   * exit head (one LM-head pass instead of two) */
  int64_t comb_heads;
} ppsd_metrics;

typedef struct {
  int32_t tick, stage, kind, position, token, verdict;
} ppsd_trace_row;

const char* ppsd_last_error(void);
const char* ppsd_build_info(void);

int ppsd_engine_create(const ppsd_model_desc* model, const ppsd_weights* weights,
                       const ppsd_pipeline_desc* pipe, void* cuda_stream,
                       ppsd_engine** out);
int ppsd_engine_destroy(ppsd_engine* e);

/* verify-while-draft decode; tokens/trace are HOST buffers. greedy = 1:
 * greedy_match verdicts (the parity contract); greedy = 0: sampling mode —
 * draft / verify / commit draws from the streams derive_seed(rng_seed,
 * "draft" | "verify" | "commit") exactly as _ToyVerifier (pipesim.py:339-365);
 * rng_seed = the caller's RngStream.seed. */
int ppsd_decode(ppsd_engine* e, int32_t greedy, uint64_t rng_seed, const int32_t* prompt,
                int32_t n_prompt, int32_t max_tokens, int32_t force_reject, int32_t* out_tokens,
                ppsd_metrics* out, ppsd_trace_row* trace, int64_t trace_cap,
                int64_t* trace_len);

/* Change the engine's schedule (PPSD_SCHEDULE_*) for later decodes;
 * PPSD_EUNSUPPORTED when FOLDED cannot apply. get_schedule reports the
 * schedule a ppsd_decode in the given mode would run. */
int ppsd_set_schedule(ppsd_engine* e, int32_t schedule);
int ppsd_get_schedule(ppsd_engine* e, int32_t greedy, int32_t* schedule);

/* ToyLM.empirical_alpha / greedy_agreement (pkg/src/specpipe/toylm.py:160-192)
 * on a ToyLM engine: for each of n_prefixes prefixes (row-major, prefix_len
 * tokens each) out_minsum[i] = sum(min(p, q)) and out_agree[i] = (argmax p ==
 * argmax q), p = exit head at exit_depth, q = full model. */
int ppsd_toy_alignment(ppsd_engine* e, int32_t exit_depth, int32_t n_prefixes, int32_t prefix_len,
                       const int32_t* prefixes, double* out_minsum, int32_t* out_agree);

/* full-model autoregressive decode (the oracle / AR baseline); sampling mode
 * draws one commit-stream uniform per token (pipesim.py:397-406) */
int ppsd_decode_ar(ppsd_engine* e, int32_t greedy, uint64_t rng_seed, const int32_t* prompt,
                   int32_t n_prompt, int32_t max_tokens, int32_t* out_tokens, ppsd_metrics* out);

/* greedy draft-then-verify rounds of gamma drafts (EESD baseline,
 * simulate_eesd with a greedy model oracle, pipesim.py:435-551): gamma
 * one-token drafts through the first exit_stage*exit_depth layers, one batched
 * verify of the gamma+1 positions, acceptance scan, bonus / truncate. Returns
 * the committed tokens (up to out_cap; the last round may overshoot horizon). */
int ppsd_decode_eesd(ppsd_engine* e, int32_t gamma, const int32_t* prompt, int32_t n_prompt,
                     int32_t horizon, int32_t* out_tokens, int32_t out_cap,
                     ppsd_metrics* out, ppsd_trace_row* trace, int64_t trace_cap,
                     int64_t* trace_len);

/* the same rounds in the given mode: greedy = 1 as above; greedy = 0 draws
 * drafts, accept_draft verdicts, residual resamples and the bonus from the
 * streams derive_seed(rng_seed, "draft" | "verify" | "commit") exactly as
 * _ToyVerifier (pipesim.py:339-365, 475-541). */
int ppsd_decode_eesd_mode(ppsd_engine* e, int32_t gamma, int32_t greedy, uint64_t rng_seed,
                          const int32_t* prompt, int32_t n_prompt, int32_t horizon, int32_t* out_tokens,
                          int32_t out_cap, ppsd_metrics* out, ppsd_trace_row* trace, int64_t trace_cap,
                          int64_t* trace_len);

/* simulate_eesd with AcceptanceOracle.bernoulli (verify_seed =
 * derive_seed(rng.seed, "verify"), pipesim.py:467) */
int ppsd_simulate_eesd(ppsd_engine* e, int32_t gamma, double alpha, uint64_t verify_seed,
                       int32_t horizon, ppsd_metrics* out, ppsd_trace_row* trace,
                       int64_t trace_cap, int64_t* trace_len);

/* schedule-only PPSD with Bernoulli(alpha) verdicts drawn from the counter
 * stream seeded verify_seed (= derive_seed(rng.seed, "verify")) */
int ppsd_simulate(ppsd_engine* e, double alpha, uint64_t verify_seed, int32_t horizon,
                  int32_t force_reject, ppsd_metrics* out, ppsd_trace_row* trace,
                  int64_t trace_cap, int64_t* trace_len);

/* Multi-rank stepping: one engine per GPU owning stages [stage_lo, stage_hi]
 * of the pipeline. The scheduler is replicated on every rank
 * and advances identically; per tick the caller all-gathers every rank's
 * outbox (kBoxHeader int32 words + d fp32, ppsd_exchange_info) into every
 * rank's inbox (world boxes) — NCCL all_gather on the engine stream — between
 * ppsd_step_compute and ppsd_step_finish. The prompt prefill is pipelined the
 * same way: ppsd_prefill_steps() rounds of {ppsd_prefill_compute, exchange}.
 * stage_owner[st] (st = 1..S, index 0 unused) is the rank owning stage st.
 * outbox / inbox are device buffers owned by the caller. */
int ppsd_exchange_info(ppsd_engine* e, int64_t* outbox_bytes, void** cuda_stream);
/* Decode mode of the next ppsd_step_begin (default greedy). Sampling
 * (pipesim.py:412-414 mode "sampling", streams derive_seed(rng_seed, "draft" |
 * "verify" | "commit")): boxes grow by the exit and final logits (2 * vocab
 * fp32 after the activation) and every rank runs the same draws from the
 * owners' logits, so tokens, metrics and trace equal the single-device
 * sampling decode. Applies to ppsd_step_begin and ppsd_p2p_decode (the
 * peer-store buffers are sized for the larger box). */
int ppsd_step_mode(ppsd_engine* e, int32_t greedy, uint64_t rng_seed);
int ppsd_step_begin(ppsd_engine* e, const int32_t* prompt, int32_t n_prompt, int32_t max_tokens,
                    int32_t force_reject, const int32_t* stage_owner, int32_t world, int32_t rank,
                    void* outbox, void* inbox);
int ppsd_prefill_steps(ppsd_engine* e, int32_t* n_steps);
int ppsd_prefill_compute(ppsd_engine* e);
int ppsd_step_compute(ppsd_engine* e);
int ppsd_step_finish(ppsd_engine* e);
int ppsd_step_poll(ppsd_engine* e, int32_t* done, int64_t* committed, int64_t* ticks);
int ppsd_step_end(ppsd_engine* e, int32_t* out_tokens, ppsd_metrics* out,
                  ppsd_trace_row* trace, int64_t trace_cap, int64_t* trace_len);

/* NVLink peer-store transport (the fused alternative to the all-gather):
 * every rank's pack kernel stores its box straight into every rank's
 * exchange buffer (CUDA IPC-mapped, NVLink/NVSwitch) and releases a flag; the
 * scheduler kernel acquire-waits on the flags, so a whole tick is one graph
 * and ticks run back to back with no host work. prepare() allocates this
 * rank's buffer and returns its cudaIpcMemHandle_t (64 bytes) and device
 * pointer; connect() maps the peers from their handles (separate processes)
 * or takes their device pointers directly (engines in one process). */
int ppsd_p2p_prepare(ppsd_engine* e, int32_t world, void* ipc_handle, void** xbuf);
int ppsd_p2p_connect(ppsd_engine* e, int32_t rank, const void* ipc_handles, void* const* local_xbufs,
                     const int32_t* stage_owner);
int ppsd_p2p_decode(ppsd_engine* e, const int32_t* prompt, int32_t n_prompt, int32_t max_tokens,
                    int32_t force_reject, int32_t* out_tokens, ppsd_metrics* out,
                    ppsd_trace_row* trace, int64_t trace_cap, int64_t* trace_len);

/* Device weight initialiser: the counter-hash init of oracle/transformer.py,
 * written straight into the engine's physical layout.
 * layout: 0 plain [rows][cols]; 1 = fused qkv (q,k pair-interleaved);
 * 2 = fused gate/up (row-interleaved), optionally | PPSD_LAYOUT_TC_TILED:
 * the tensor-core GEMV's tiled matrix layout (the buffer holds
 * ppsd_weight_elems(1, rows, cols) bf16). For layouts 1/2 tid0..tid2 are the
 * logical tensors' ids and a0..a2 their scales. */
#define PPSD_LAYOUT_TC_TILED 16
/* bf16 elements of a [rows][cols] matrix in the plain (tiled = 0) or the
 * TC-tiled (tiled = 1: K padded to a multiple of 64) layout */
int ppsd_weight_elems(int32_t tiled, int64_t rows, int64_t cols, int64_t* elems);
/* bf16 index of element (r, k) of a [rows][cols] matrix in the TC-tiled
 * layout (k < cols padded to a multiple of 64; padding holds zeros) — for
 * loaders that tile checkpoints on the host (paper_2509_19368_b200.tc_tile) */
int ppsd_tc_offset(int64_t rows, int64_t cols, int64_t r, int64_t k, int64_t* off);
int ppsd_init_weight(void* dst_bf16, int32_t layout, int64_t rows, int64_t cols,
                     uint64_t seed, const uint64_t* tids, const float* scales,
                     int32_t n_heads, int32_t n_kv_heads, int32_t head_dim,
                     void* cuda_stream);

/* GEMV unit check (parity tests): y_v = W x_v through the shipped kernel for
 * the O (which = 1) or down (which = 3) projection of global layer `layer`;
 * nv vectors (<= 5 decode-tick plan, <= 16 batched plan); in [nv][K], out
 * [nv][R], host fp32. */
int ppsd_debug_matvec(ppsd_engine* e, int32_t which, int32_t layer, int32_t nv, int32_t batched,
                      const float* in, float* out);

/* Tensor-core GEMV pipeline timeline (debugging; needs a build with
 * -DPPSD_TC_TRACE, else zeros): on >= 0 enables (1) / disables (0) recording,
 * out (or NULL) receives [8][128] CTA-0 events then [160][4] per-CTA marks,
 * %globaltimer ns. */
int ppsd_debug_tc_trace(int32_t on, uint64_t* out);

/* fp32 logits of the last head evaluation: which 0 = exit head, 1 = final
 * head (length vocab) — debugging / tolerance tests. */
int ppsd_read_logits(ppsd_engine* e, int32_t which, float* out);

/* Logits tap (parity tests): while set, single-rank ppsd_decode calls on a
 * transformer engine copy every exit / final head's fp32 logits row into
 * dev_tap[(pos * 2 + which) * vocab] (device buffer, which 0 = exit, 1 =
 * final; pos = the generated position the row predicts, 1 .. max_pos). Rows
 * of flushed chains are overwritten by the committed prefix's rows, so after
 * a decode every position holds the logits its verdict / draft used. The
 * scheduler kernel does the copies; the graphs are unchanged. NULL clears it.
 * Replaces nothing in the reference: it is the GPU side of the logits
 * tolerance check (the reference's ProbVecs, pipesim.py:743, :714). */
int ppsd_set_logits_tap(ppsd_engine* e, float* dev_tap, int32_t max_pos);

/* Kernel-time probe for the roofline: times `reps` launches of the engine's
 * dominant layer GEMV (gate/up) with CUDA events on the engine stream. */
int ppsd_probe_gemv(ppsd_engine* e, int32_t which, int32_t n_groups, int32_t reps,
                    double* avg_ms, double* bytes_per_launch);

/* Kernel-time probe of decode attention: one group of n_vec query vectors,
 * longest context ctx, timed over `reps` launches on the engine stream;
 * bytes = the K/V rows one launch must read. */
int ppsd_probe_attn(ppsd_engine* e, int32_t n_vec, int32_t ctx, int32_t reps, double* avg_ms,
                    double* bytes_per_launch);

#ifdef __cplusplus
}
#endif
#endif /* PPSD_H */
