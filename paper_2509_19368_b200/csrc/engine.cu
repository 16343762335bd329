// engine.cu — libppsd.so: the C ABI declared in include/ppsd.h.
//
// A tick of the verify-while-draft machine is one CUDA graph:
//   [per layer slot i of the local stages: qkv_rope, attention, o_proj+res,
//    gate_up+swiglu, down+res] -> [tied exit/final LM head + argmax]
//   -> [sched_tick: verdict/draft/rollback for tick t, plan tick t+1, embed]
// Graph arguments never change; per-call state lives in device memory
// (TickCtx / Sched / Work), so the host enqueues ticks back to back and only
// synchronises when the lower bound on the remaining ticks is exhausted.
#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "engine_dev.cuh"

using namespace ppsd;

namespace ppsd {
bool attn_supported(int hd, int qpk);
}

static thread_local std::string g_err;
namespace ppsd {
bool g_pdl = true;
}

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
#define CU(x)                                                                                 \
  do {                                                                                        \
    cudaError_t _e = (x);                                                                     \
    if (_e != cudaSuccess)                                                                    \
      return fail(PPSD_ECUDA, std::string(#x) + ": " + cudaGetErrorString(_e) + " @" +        \
                                  std::to_string(__LINE__));                                  \
  } while (0)

// layers whose matrices of one kind sit at a fixed stride (one allocation)
struct WStride {
  const void* base = nullptr;
  long long stride = 0;
  int n = 0;  // layers [0, n) follow base + l * stride
};

// persistent layer pass (tcpass.cu): ring / shared-memory plan for one B width
struct PassPlan {
  bool ok = false;
  int nblk = 1, ns = 0, slot_bytes = 0, b_stage = 0, attn_off = 0, attn_kv_bytes = 0, scr_off = 0, bar_off = 0,
      workers = 1;
  int nb[4] = {1, 1, 1, 1};
  size_t smem = 0;
};

struct GemvPlan {
  int m = 1, R = 0, K = 0;  // vectors per weight pass, matrix shape
  TcPlan tc;                // tensor-core GEMV plan (tcgemv.cu)
};

struct ppsd_engine {
  ppsd_model_desc md{};
  ppsd_pipeline_desc pd{};
  int device = 0, num_sms = 148;
  int attn_per_sm = 8;  // attention CTAs per SM: one resident wave
  bool attn_cl = false;  // one-vector launches use the cluster attention kernel (attn.cu)
  bool attn_clb = false;  // batched launches may use it too (clusters of 4, attn_clb_vec rows)
  int attn_clb_cs = 4;    // their cluster size (4, or 8 = the one-vector kernel's)
  int attn_clb_vec = 0;   // vectors the batched capture in progress can hold (0: split-K kernel)
  bool tick_g1 = false;  // capturing tick launches whose `work` has one group (folded shallow, rank-fold eager)
  bool comb_capture = false;  // capturing the folded body's final heads with the combined exit head
  WStride wstride[4];  // per matrix kind (kMatQKV..kMatDown), when the layers are strided
  bool small_batch = false;  // capturing batched launches of <= 5 vectors (tick plans serve them)
  int hint_first = -1;       // capturing single-problem launches whose first layer is known (speculative start)
  // persistent layer pass: [0] groups of <= 5 vectors, [1] <= 16
  bool pass = false;
  int pass_cs = 1;
  PassPlan pp[2];
  unsigned long long* d_pass_bar = nullptr;  // [0] arrivals, [1] base of the next pass, [2] done count
  cudaStream_t st = nullptr;
  SchedCfg cfg{};
  int S = 0, lo = 1, hi = 1, max_local_layers = 0, first_local_layer = 0, n_local_layers = 0;
  Dims dm{};
  // device state
  Sched* d_sched = nullptr;
  Work* d_work = nullptr;
  Work* d_work_ar = nullptr;
  Work* d_work_deep = nullptr;  // folded schedule: the deep batch
  Work* d_work_head = nullptr;  // exit-head layer (md.exit_head_layer)
  Work* d_work_p2 = nullptr;       // prefill: layers after the exit (exit-head layer)
  Work* d_work_head_pf = nullptr;  // prefill's exit-head layer
  int32_t* d_kerr = nullptr;       // sticky GEMV error word (K-split wait timeout)
  bool hl = false;              // exit head has a decoder layer
  TickCtx* d_ctx = nullptr;
  ArCtl* d_arctl = nullptr;
  int32_t* d_tokens = nullptr;
  uint64_t* d_pdig = nullptr;
  uint64_t* d_chain_dig = nullptr;
  TraceRow* d_trace = nullptr;
  int64_t trace_cap = 0;
  // transformer buffers
  std::vector<LayerW> h_layers;
  LayerW* d_layers = nullptr;
  float *d_x = nullptr, *d_q = nullptr, *d_o = nullptr, *d_h = nullptr, *d_logits = nullptr;
  float *d_attn_part = nullptr, *d_head_part = nullptr;
  int32_t *d_attn_cnt = nullptr, *d_head_cnt = nullptr, *d_page_table = nullptr;
  void* d_kv = nullptr;
  int max_pages = 0;
  GemvPlan gp[kNumMats];   // decode tick: one vector per weight pass (head: exit + final)
  GemvPlan gpb[kNumMats];  // batched prefill / EESD verify: up to 4 vectors per pass
  int nbuf = 0;            // activation slots (>= nslot, >= kMaxVec)
  uint64_t verify_seed = 0;  // sampling mode: derive_seed(rng.seed, "verify")
  double *d_pdist = nullptr, *d_qbuf = nullptr, *d_wbuf = nullptr, *d_logits64 = nullptr;
  const __nv_bfloat16* lm_head = nullptr;
  const float* final_norm = nullptr;
  const float* exit_norm = nullptr;
  const float* rope_cos = nullptr;
  const float* rope_sin = nullptr;
  // graphs
  cudaGraphExec_t g_tick = nullptr, g_ar = nullptr, g_prefill = nullptr;
  // folded schedule (sched.h: sched_fold_plan): one graph per tick =
  // [sched, shallow layers, exit head, IF(deep batch){deep layers, final heads}]
  cudaGraphExec_t g_fold = nullptr;
  bool fold_ok = false;      // engine can run the folded schedule
  bool fold_auto = false;    // ...and PPSD_SCHEDULE_AUTO picks it
  int schedule = PPSD_SCHEDULE_AUTO;
  int64_t fold_tick_launches = 0, fold_deep_launches = 0;
  cudaGraphExec_t g_compute = nullptr, g_finish = nullptr, g_mr_prefill = nullptr;  // multi-rank
  std::map<int, std::pair<cudaGraphExec_t, int64_t>> eesd_graphs;  // per gamma: round graph, launches
  EesdState* d_eesd = nullptr;
  int64_t compute_launches = 0, finish_launches = 0, mr_prefill_launches = 0;
  int mr_world = 0, mr_rank = 0, mr_stop = 0, mr_n_prompt = 0;
  int mr_greedy = 1;          // ppsd_step_mode
  uint64_t mr_rng_seed = 0;
  int64_t mr_launches = 0, mr_ticks_launched = 0;
  // NVLink peer-store transport
  float* d_xbuf = nullptr;          // [2][world][box] + world flags, shared via IPC
  float* d_p2p_outbox = nullptr;    // local box scratch
  uint64_t* d_xcount = nullptr;
  int32_t* d_xerr = nullptr;
  std::vector<void*> retired;  // buffers replaced while peers may still run (freed at destroy)
  float** d_peer_xbuf = nullptr;
  std::vector<void*> ipc_opened;    // peer mappings to close
  int p2p_world = 0;
  cudaGraphExec_t g_p2p_tick = nullptr;
  int64_t p2p_tick_launches = 0;
  // rank fold (sched.h: sched_rfold_plan), greedy multi-rank: one graph per
  // tick = [IF setter, eager stages, exit head, IF(batch){gather, deferred
  // layers, final heads}, pack (, scheduler: p2p)]
  bool rfold_ok = false;   // this stage range folds (>= 2 deferred stages, batch fits)
  bool mr_rf = false;      // the current multi-rank decode runs it
  cudaGraphExec_t g_compute_rf = nullptr, g_p2p_tick_rf = nullptr;
  int64_t compute_rf_launches = 0, p2p_tick_rf_launches = 0, rf_body_launches = 0;
  int64_t tick_launches = 0, ar_launches = 0, prefill_launches = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
  // host staging
  Sched* h_sched = nullptr;  // pinned
  // p2p: pinned staging for the per-decode uploads (ctx, ArCtl, prompt) so a
  // decode never issues a pageable copy or an allocation while peer engines
  // of this process spin on flags it has yet to set
  char* h_p2p_pin = nullptr;
  int32_t* h_p2p_out = nullptr;
  TickCtx h_ctx{};
};

extern "C" const char* ppsd_last_error(void) { return g_err.c_str(); }

extern "C" const char* ppsd_build_info(void) {
  return "libppsd sm_100a: tcgen05 weight-streaming GEMV (TMEM accumulators, bulk-copy ring, cluster split-K), "
         "split-K paged attention, device tick machine";
}

// NVTX ranges (header-only nvtx3: free unless a profiler is attached):
// ppsd.prefill / ppsd.decode / ppsd.ticks (one per launched batch of tick
// graphs, named with the tick range) / ppsd.ar / ppsd.eesd / ppsd.p2p
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* what, long long a, long long b) {
    char buf[96];
    snprintf(buf, sizeof(buf), "%s %lld..%lld", what, a, b);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

static int attn_grid(const ppsd_engine* e) { return e->attn_per_sm * e->num_sms; }

// first failed launch inside a graph capture (the capture itself only
// reports "invalidated")
static thread_local cudaError_t g_launch_err = cudaSuccess;
static cudaError_t note_launch(cudaError_t e) {
  if (e != cudaSuccess && g_launch_err == cudaSuccess) g_launch_err = e;
  return e;
}

// ---------------------------------------------------------------------------
// enqueue helpers (also used while capturing graphs)

static GemvArgs make_gemv_args(ppsd_engine* e, Work* w, int layer_i, int mat, const GemvPlan& p, float* logits);

static cudaError_t enqueue_gemv(ppsd_engine* e, Work* w, int layer_i, int mat, bool batched = false,
                                float* logits = nullptr) {
  // tensor-core GEMV: groups of <= 5 vectors (the folded deep batch at
  // E >= N/5) run the decode-tick plan, whose smaller operand stages leave
  // room for a deeper weight ring; the arithmetic is the same in every plan
  const bool use_b = batched && !e->small_batch;
  const GemvPlan& p = use_b ? e->gpb[mat] : e->gp[mat];
  GemvArgs a = make_gemv_args(e, w, layer_i, mat, p, logits);
  const TcPlan& t = p.tc;
  return note_launch(tc_launch(a, t.cs, t.smem, t.grid, e->st));
}

static GemvArgs make_gemv_args(ppsd_engine* e, Work* w, int layer_i, int mat, const GemvPlan& p, float* logits) {
  GemvArgs a{};
  a.work = w;
  a.layer_i = layer_i;
  a.desc_early = !(mat == kMatQKV && layer_i == 0);  // first kernel after the scheduler
  a.mat = mat;
  a.layers = e->d_layers;
  a.head_w = e->lm_head;
  a.head_norm0 = e->exit_norm;
  a.head_norm1 = e->final_norm;
  a.R = p.R;
  a.K = p.K;
  a.dm = e->dm;
  a.x = e->d_x;
  a.q = e->d_q;
  a.o = e->d_o;
  a.h = e->d_h;
  a.logits = logits ? logits : e->d_logits;
  a.rope_cos = e->rope_cos;
  a.rope_sin = e->rope_sin;
  a.page_table = e->d_page_table;
  a.head_part = e->d_head_part;
  a.head_cnt = e->d_head_cnt;
  a.err = e->d_kerr;
  a.hint_li = -1;
  a.comb_exit = mat == kMatHeadV && e->comb_capture ? 1 : 0;
  {
    const TcPlan& t = p.tc;
    // speculative start: measured slower on the 7B bench (427 vs 437 tok/s,
    // DESIGN.md §8), opt-in PPSD_TC_HINT=1
    static const int hints = getenv("PPSD_TC_HINT") ? atoi(getenv("PPSD_TC_HINT")) : 0;
    if ((hints & 1) && (mat == kMatHead || mat == kMatHeadV)) a.hint_li = 0;  // one problem at most, the LM head
    else if ((hints & 2) && e->hint_first >= 0 && ((hints & 4) || a.desc_early)) a.hint_li = e->hint_first + layer_i;
    if (mat == kMatHead || mat == kMatHeadV) {
      a.wp[0] = e->lm_head;
    } else {
      const WStride& ws = e->wstride[mat];
      a.wbase = ws.base;
      a.wstride = ws.stride;
      a.wn = ws.n;
      if (e->h_layers.size() <= (size_t)kTcMaxWp)
        for (size_t l = 0; l < e->h_layers.size(); ++l) {
          const LayerW& L = e->h_layers[l];
          a.wp[l] = mat == kMatQKV ? (const void*)L.qkv : mat == kMatO ? (const void*)L.o
                  : mat == kMatGU ? (const void*)L.gu : (const void*)L.down;
        }
    }
    a.nstage = t.ns;
    a.js = t.js;
    a.nj = t.nj;
    a.nb = t.nb;
    a.tg = t.tg;
    a.nblk = t.nblk;
    a.bar_off = t.bar_off;
    // L2 prefetch of the next GEMV of the layer: QKV -> O the whole O slice
    // (attention leaves HBM idle in between), O -> GU, GU -> down, down -> next
    // QKV the first 48 KB per CTA (the next launch's first stages; re-measured
    // after the cluster attention: 0 KB 459.4, 32 466.1, 48 466.4, 64 464.1,
    // 96 461.3 tok/s). PPSD_TC_NEXT=<KB> overrides.
    static const int nx_kb = getenv("PPSD_TC_NEXT") ? atoi(getenv("PPSD_TC_NEXT")) : 48;
    if (mat <= kMatDown && (mat == kMatQKV || nx_kb > 0)) {
      const int nm = (mat + 1) % 4;
      const GemvPlan& np_ = &p == &e->gpb[mat] ? e->gpb[nm] : e->gp[nm];
      const WStride& ws = e->wstride[nm];
      if (ws.stride) {
        TcNext& X = a.nx;
        X.wbase = ws.base;
        X.wstride = ws.stride;
        X.wn = ws.n;
        X.dli = mat == kMatDown ? 1 : 0;
        X.R = np_.tc.R;
        X.js = np_.tc.js;
        X.nj = np_.tc.nj;
        X.tg = np_.tc.tg;
        X.cs = np_.tc.cs;
        const long long slice = (long long)np_.tc.R * np_.tc.K * 2 / std::max(1, np_.tc.grid) + (1 << 16);
        X.bytes = mat == kMatQKV ? (int)std::min<long long>(slice, 1 << 30) : nx_kb * 1024;
      }
    }
  }
  return a;
}

static AttnArgs make_attn_args(ppsd_engine* e, Work* w, int layer_i) {
  AttnArgs a{};
  a.work = w;
  a.layer_i = layer_i;
  a.layers = e->d_layers;
  a.dm = e->dm;
  a.q = e->d_q;
  a.o = e->d_o;
  a.part = e->d_attn_part;
  a.cnt = e->d_attn_cnt;
  a.page_table = e->d_page_table;
  a.max_pages = e->max_pages;
  a.kv_base = e->d_kv;
  a.kv_layer_bytes = (long long)e->max_pages * kPage * e->dm.KV * e->dm.hd * (e->dm.kv_bf16 ? 2 : 4);
  a.first_local = e->first_local_layer;
  a.hl_global = e->hl ? e->md.n_layers : -1;
  a.hl_local = e->n_local_layers;
  a.err = e->d_kerr;
  return a;
}

static cudaError_t enqueue_attn(ppsd_engine* e, Work* w, int layer_i, bool batched = true) {
  // PPSD_PROFILE_SKIP_ATTN=1: timing experiments only (wrong results)
  static const bool skip = getenv("PPSD_PROFILE_SKIP_ATTN") && atoi(getenv("PPSD_PROFILE_SKIP_ATTN")) != 0;
  if (skip) return cudaSuccess;
  if (!batched && e->attn_cl) {
    // one vector per group: a cluster per (group, kv head) row. Rows: the
    // tick descriptor's groups (one per local stage) unless the capture has
    // one group (AR, EESD draft, exit-head layer, folded shallow, rank-fold eager)
    const bool one = w != e->d_work || e->tick_g1;
    const int rows = (one ? 1 : e->hi - e->lo + 1) * e->dm.KV;
    return attn_cl_launch(make_attn_args(e, w, layer_i), rows, e->st);
  }
  if (batched && e->attn_clb && e->attn_clb_vec > 0) {
    // a bounded batch (folded deep batch): a cluster of 4 per (vector, kv
    // head) row; the same page partials and ordered merge as attn_kernel
    AttnArgs a = make_attn_args(e, w, layer_i);
    a.multi = 1;
    return attn_cl_launch(a, e->attn_clb_vec * e->dm.KV, e->st, e->attn_clb_cs);
  }
  return attn_launch(make_attn_args(e, w, layer_i), attn_grid(e), e->st);
}

// Prompt layers for a chunk of <= kMaxVec vectors in group 0 of `w`: the
// batched tensor-core GEMV plans (every vector of the chunk in one weight
// pass). Returns launches enqueued, or -1.
static int enqueue_layers(ppsd_engine* e, Work* w, int n_slots, bool batched);
static int enqueue_prefill_layers(ppsd_engine* e, Work* w, int n_slots) {
  return enqueue_layers(e, w, n_slots, true);
}

static int setup_pass(ppsd_engine* e);

// One persistent launch for n_slots layer slots (tcpass.cu); -1 on error.
static int enqueue_pass(ppsd_engine* e, Work* w, int n_slots, bool batched) {
  const bool big = batched && !e->small_batch;
  const PassPlan& pl = e->pp[big ? 1 : 0];
  TcPassArgs a{};
  const GemvPlan& pq = big ? e->gpb[kMatQKV] : e->gp[kMatQKV];
  a.g = make_gemv_args(e, w, 0, kMatQKV, pq, nullptr);
  a.at = make_attn_args(e, w, 0);
  for (int m = 0; m < 4; ++m) {
    const TcPlan& t = (big ? e->gpb[m] : e->gp[m]).tc;
    TcPassMat& M = a.mat[m];
    M.R = t.R;
    M.K = t.K;
    M.js = t.js;
    M.nj = t.nj;
    M.tg = t.tg;
    M.cs = t.cs;
    M.nb = pl.nb[m];
    M.wbase = e->wstride[m].base;
    M.wstride = e->wstride[m].stride;
    M.wn = e->wstride[m].n;
  }
  a.n_slots = n_slots;
  a.desc_early = 0;
  a.ns = pl.ns;
  a.slot_bytes = pl.slot_bytes;
  a.b_stage = pl.b_stage;
  a.nblk = pl.nblk;
  a.attn_off = pl.attn_off;
  a.attn_kv_bytes = pl.attn_kv_bytes;
  a.scr_off = pl.scr_off;
  a.bar_off = pl.bar_off;
  a.attn_workers = pl.workers;
  // L2 prefetch distance per CTA (PPSD_PASS_PREFETCH=<KB>, default 384): the
  // grid's prefetched weights (~57 MB) stay well inside the 126 MB L2
  static const unsigned long long pf = getenv("PPSD_PASS_PREFETCH") ? (unsigned long long)atoll(getenv("PPSD_PASS_PREFETCH")) * 1024
                                                                    : 384ull * 1024;
  a.prefetch_bytes = pf;
  a.bar_cnt = e->d_pass_bar;
  a.bar_seq = e->d_pass_bar + 1;
  a.done_cnt = reinterpret_cast<uint32_t*>(e->d_pass_bar + 2);
  const cudaError_t ce = note_launch(tc_pass_launch(a, e->pass_cs, e->dm.hd, e->dm.H / e->dm.KV, e->dm.kv_bf16,
                                                    pl.smem, e->num_sms / e->pass_cs * e->pass_cs, e->st));
  return ce == cudaSuccess ? 1 : -1;
}

// returns launches enqueued, or -1 on error
static int enqueue_layers(ppsd_engine* e, Work* w, int n_slots, bool batched) {
  if (e->pass && n_slots > 0) return enqueue_pass(e, w, n_slots, batched);
  int n = 0;
  for (int i = 0; i < n_slots; ++i) {
    if (enqueue_gemv(e, w, i, kMatQKV, batched) != cudaSuccess) return -1;
    if (enqueue_attn(e, w, i, batched) != cudaSuccess) return -1;
    if (enqueue_gemv(e, w, i, kMatO, batched) != cudaSuccess) return -1;
    if (enqueue_gemv(e, w, i, kMatGU, batched) != cudaSuccess) return -1;
    if (enqueue_gemv(e, w, i, kMatDown, batched) != cudaSuccess) return -1;
    n += 5;
  }
  return n;
}

// Exit-head layer: copy the drafting chain's exit state into the head rows,
// then run the head's decoder layer on the copies (prefill: the whole chunk,
// tcgen05 when planned). Returns launches enqueued, or -1.
static int enqueue_head_layer(ppsd_engine* e, bool prefill) {
  Work* wh = prefill ? e->d_work_head_pf : e->d_work_head;
  if (launch_pdl(head_copy_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx, (const Work*)wh) !=
      cudaSuccess)
    return -1;
  const int m = prefill ? enqueue_prefill_layers(e, wh, 1) : enqueue_layers(e, wh, 1, false);
  return m < 0 ? -1 : m + 1;
}

template <class F>
static int capture(ppsd_engine* e, F body, cudaGraphExec_t* out, int64_t* nlaunch) {
  cudaGraph_t g = nullptr;
  g_launch_err = cudaSuccess;
  CU(cudaStreamBeginCapture(e->st, cudaStreamCaptureModeThreadLocal));
  int n = body();
  cudaError_t ce = cudaStreamEndCapture(e->st, &g);
  if (n < 0) {
    if (g) cudaGraphDestroy(g);
    const cudaError_t le = g_launch_err != cudaSuccess ? g_launch_err : cudaGetLastError();
    return fail(PPSD_ECUDA, std::string("kernel launch failed during capture: ") + cudaGetErrorString(le));
  }
  CU(ce);
  CU(cudaGraphInstantiate(out, g, 0));
  CU(cudaGraphDestroy(g));
  *nlaunch = n;
  return PPSD_OK;
}

// Folded tick graph. The deep batch runs only in ticks that need a verdict
// the batch has not produced yet, so it sits behind a graph IF node whose
// condition the scheduler kernel (first node) sets for this launch; the
// handle resets to 0 at every launch (cudaGraphCondAssignDefault).
static int build_fold_graph(ppsd_engine* e) {
  const int shallow = e->cfg.shallow_layers, deep = e->md.n_layers - shallow;
  // exit head inside the deep batch's final-head launch (one LM-head pass
  // instead of two in batch ticks): the batch plus the exit vector must fit
  // the tick plan (<= 5 vectors), no exit-head layer; PPSD_FOLD_COMB=0: off
  const char* cbv = getenv("PPSD_FOLD_COMB");
  const char* fcv = getenv("PPSD_FOLD_COND");
  const bool comb = !(cbv && cbv[0] == '0') && !e->hl && sched_fold_width(&e->cfg) + 1 <= 5 &&
                    !(fcv && atoi(fcv) == 0) && e->nbuf - 1 >= sched_fold_width(&e->cfg);
  e->h_ctx.fold_comb = comb ? 1 : 0;
  e->h_ctx.comb_row = e->nbuf - 1;
  cudaStream_t main_st = e->st, body_st = nullptr;
  CU(cudaStreamCreateWithFlags(&body_st, cudaStreamNonBlocking));
  cudaGraph_t g = nullptr;
  int n_outer = 0, n_body = 0;
  bool ok = true;
  std::string err;
  auto need = [&](bool cond, const char* what) {
    if (!cond && ok) {
      ok = false;
      err = std::string(what) + ": " + cudaGetErrorString(cudaGetLastError());
    }
  };
  cudaError_t ce = cudaStreamBeginCapture(main_st, cudaStreamCaptureModeThreadLocal);
  if (ce != cudaSuccess) {
    cudaStreamDestroy(body_st);
    CU(ce);
  }
  need(launch_pdl(sched_tick_kernel, dim3(1), dim3(256), 0, main_st, (const TickCtx*)e->d_ctx, 0) ==
           cudaSuccess, "sched");
  n_outer = 1;
  if (ok) {
    e->hint_first = e->lo == 1 ? 0 : -1;  // sched.cu: the launched chain's layers [0, shallow)
    e->tick_g1 = true;
    const int m = enqueue_layers(e, e->d_work, shallow, false);
    e->tick_g1 = false;
    e->hint_first = -1;
    need(m >= 0, "shallow layers");
    n_outer += m;
  }
  if (ok && e->hl) {
    const int m = enqueue_head_layer(e, false);
    need(m >= 0, "exit-head layer");
    n_outer += m;
  }
  need(ok && enqueue_gemv(e, e->d_work, 0, kMatHead) == cudaSuccess, "exit head");
  n_outer += 1;
  cudaGraphNode_t cnode = nullptr;
  cudaGraph_t body = nullptr;
  // PPSD_FOLD_COND=0 (profiling only: ncu does not profile graphs with
  // conditional nodes): the deep part is captured inline and launched every
  // tick; without a batch its kernels find no work and exit
  const char* cv = getenv("PPSD_FOLD_COND");
  if (ok && cv && atoi(cv) == 0) {
    e->hint_first = shallow;
    e->attn_clb_vec = sched_fold_width(&e->cfg);
    const int m = enqueue_layers(e, e->d_work_deep, deep, true);
    e->attn_clb_vec = 0;
    e->hint_first = -1;
    need(m >= 0, "deep layers");
    need(ok && enqueue_gemv(e, e->d_work_deep, 0, kMatHeadV, true, e->d_logits + e->dm.V) == cudaSuccess,
         "final heads");
    n_outer += m + 1;
    e->h_ctx.cond = 0;
    e->h_ctx.has_cond = 0;
  } else if (ok) {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    cudaGraph_t cg = nullptr;
    need(cudaStreamGetCaptureInfo(main_st, &cs, nullptr, &cg, &deps, &nd) == cudaSuccess, "capture info");
    cudaGraphConditionalHandle h = 0;
    if (ok) need(cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault) == cudaSuccess,
                 "conditional handle");
    if (ok) {
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeIf;
      cp.conditional.size = 1;
      need(cudaGraphAddNode(&cnode, cg, deps, nd, &cp) == cudaSuccess, "conditional node");
      if (ok) body = cp.conditional.phGraph_out[0];
      if (ok) need(cudaStreamUpdateCaptureDependencies(main_st, &cnode, 1, cudaStreamSetCaptureDependencies) ==
                       cudaSuccess, "capture deps");
      e->h_ctx.cond = h;
      e->h_ctx.has_cond = 1;
    }
  }
  if (ok && body) {  // body: deep layers of the batch (batched plans), final heads
    need(cudaStreamBeginCaptureToGraph(body_st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
             cudaSuccess, "body capture");
    if (ok) {
      e->st = body_st;
      e->small_batch = sched_fold_width(&e->cfg) <= 5;
      if (comb) {  // the launched chain's exit state, before the deep layers advance its row
        need(launch_pdl(fold_exit_copy_kernel, dim3(1), dim3(256), 0, body_st, (const TickCtx*)e->d_ctx) ==
                 cudaSuccess, "exit copy");
        n_body += 1;
      }
      e->hint_first = shallow;  // sched.cu: the batch's layers [shallow, N)
      e->attn_clb_vec = sched_fold_width(&e->cfg);
      const int m = enqueue_layers(e, e->d_work_deep, deep, true);
      e->attn_clb_vec = 0;
      e->hint_first = -1;
      need(m >= 0, "deep layers");
      n_body += m;
      e->comb_capture = comb;
      need(ok && enqueue_gemv(e, e->d_work_deep, 0, kMatHeadV, true,
                              comb ? e->d_logits : e->d_logits + e->dm.V) == cudaSuccess,
           "final heads");
      e->comb_capture = false;
      n_body += 1;
      e->small_batch = false;
      e->st = main_st;
      cudaGraph_t bg = body;
      need(cudaStreamEndCapture(body_st, &bg) == cudaSuccess, "body end capture");
    }
  }
  e->st = main_st;
  ce = cudaStreamEndCapture(main_st, &g);
  cudaStreamDestroy(body_st);
  if (!ok) {
    if (g) cudaGraphDestroy(g);
    return fail(PPSD_ECUDA, "folded tick graph: " + err);
  }
  CU(ce);
  ce = cudaGraphInstantiate(&e->g_fold, g, 0);
  cudaGraphDestroy(g);
  CU(ce);
  e->fold_tick_launches = n_outer;
  e->fold_deep_launches = n_body;
  return PPSD_OK;
}

static int build_graphs(ppsd_engine* e) {
  const int kind = e->md.kind;
  int rc = capture(
      e,
      [&]() -> int {
        int n = 0;
        if (kind == PPSD_MODEL_TRANSFORMER) {
          int m = enqueue_layers(e, e->d_work, e->max_local_layers, false);
          if (m < 0) return -1;
          n += m;
          if (e->hl) {  // exit-head layer on a copy of the exit chain's state
            m = enqueue_head_layer(e, false);
            if (m < 0) return -1;
            n += m;
          }
          if (enqueue_gemv(e, e->d_work, 0, kMatHead) != cudaSuccess) return -1;
          n += 1;
        } else if (kind == PPSD_MODEL_TOYLM) {
          if (launch_pdl(toy_tick_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx) != cudaSuccess)
            return -1;
          n += 1;
        }
        if (launch_pdl(sched_tick_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx, 0) !=
            cudaSuccess)
          return -1;
        return n + 1;
      },
      &e->g_tick, &e->tick_launches);
  if (rc) return rc;
  if (kind != PPSD_MODEL_TRANSFORMER) return PPSD_OK;
  rc = capture(  // autoregressive token step (decode_autoregressive)
      e,
      [&]() -> int {
        if (launch_pdl(ar_begin_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx, e->d_arctl, 1) !=
            cudaSuccess)
          return -1;
        e->hint_first = e->first_local_layer;  // ar_begin_kernel: first = the first local layer
        int m = enqueue_layers(e, e->d_work_ar, e->n_local_layers, false);
        e->hint_first = -1;
        if (m < 0) return -1;
        if (enqueue_gemv(e, e->d_work_ar, 0, kMatHead) != cudaSuccess) return -1;
        if (launch_pdl(ar_end_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx, e->d_arctl, 1) !=
            cudaSuccess)
          return -1;
        return m + 3;
      },
      &e->g_ar, &e->ar_launches);
  if (rc) return rc;
  rc = capture(  // batched prompt prefill: one chunk of up to kMaxVec tokens per launch
      e,
      [&]() -> int {
        if (launch_pdl(prefill_chunk_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx,
                       e->d_arctl) != cudaSuccess)
          return -1;
        int m;
        if (e->hl) {  // [0, split), head layer on copies of the chunk, [split, N)
          const int split = e->h_ctx.hl_split;
          m = enqueue_prefill_layers(e, e->d_work_ar, split);
          if (m < 0) return -1;
          const int mh = enqueue_head_layer(e, true);
          if (mh < 0) return -1;
          const int m2 = enqueue_prefill_layers(e, e->d_work_p2, e->n_local_layers - split);
          if (m2 < 0) return -1;
          m += mh + m2;
        } else {
          m = enqueue_prefill_layers(e, e->d_work_ar, e->n_local_layers);
          if (m < 0) return -1;
        }
        return m + 1;
      },
      &e->g_prefill, &e->prefill_launches);
  if (rc) return rc;
  if (e->fold_ok) return build_fold_graph(e);
  return PPSD_OK;
}

// ---------------------------------------------------------------------------

static void free_engine(ppsd_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->st) cudaStreamSynchronize(e->st);
  if (e->g_tick) cudaGraphExecDestroy(e->g_tick);
  if (e->g_fold) cudaGraphExecDestroy(e->g_fold);
  if (e->g_ar) cudaGraphExecDestroy(e->g_ar);
  if (e->g_prefill) cudaGraphExecDestroy(e->g_prefill);
  if (e->g_compute) cudaGraphExecDestroy(e->g_compute);
  if (e->g_finish) cudaGraphExecDestroy(e->g_finish);
  if (e->g_mr_prefill) cudaGraphExecDestroy(e->g_mr_prefill);
  for (auto& kv : e->eesd_graphs) cudaGraphExecDestroy(kv.second.first);
  if (e->g_p2p_tick) cudaGraphExecDestroy(e->g_p2p_tick);
  if (e->g_compute_rf) cudaGraphExecDestroy(e->g_compute_rf);
  if (e->g_p2p_tick_rf) cudaGraphExecDestroy(e->g_p2p_tick_rf);
  for (void* p : e->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* b : {(void*)e->d_xbuf, (void*)e->d_p2p_outbox, (void*)e->d_xcount, (void*)e->d_peer_xbuf,
                  (void*)e->d_xerr})
    if (b) cudaFree(b);
  if (e->d_eesd) cudaFree(e->d_eesd);
  for (void* b : {(void*)e->d_pass_bar})
    if (b) cudaFree(b);
  for (void* b : e->retired) cudaFree(b);
  void* bufs[] = {e->d_sched, e->d_work, e->d_work_ar, e->d_work_deep, e->d_work_head, e->d_work_p2,
                  e->d_work_head_pf, e->d_kerr, e->d_ctx, e->d_arctl, e->d_tokens, e->d_pdig,
                  e->d_chain_dig, e->d_trace, e->d_layers, e->d_x, e->d_q, e->d_o, e->d_h, e->d_logits,
                  e->d_attn_part, e->d_head_part, e->d_attn_cnt, e->d_head_cnt, e->d_page_table, e->d_kv,
                  e->d_pdist, e->d_qbuf, e->d_wbuf, e->d_logits64};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (e->h_sched) cudaFreeHost(e->h_sched);
  if (e->h_p2p_pin) cudaFreeHost(e->h_p2p_pin);
  if (e->ev0) cudaEventDestroy(e->ev0);
  if (e->ev1) cudaEventDestroy(e->ev1);
  if (e->ev2) cudaEventDestroy(e->ev2);
  if (e->st) cudaStreamDestroy(e->st);
  delete e;
}

template <class T>
static cudaError_t dalloc(T** p, size_t bytes) {
  cudaError_t r = cudaMalloc(reinterpret_cast<void**>(p), bytes);
  if (r == cudaSuccess) r = cudaMemset(*p, 0, bytes);
  return r;
}

static int create_impl(const ppsd_model_desc* md, const ppsd_weights* w, const ppsd_pipeline_desc* pd,
                       ppsd_engine* e) {
  e->md = *md;
  e->pd = *pd;
  {
    const char* v = getenv("PPSD_PDL");  // read at engine creation; graphs capture it
    ppsd::g_pdl = v ? atoi(v) != 0 : true;
  }
  e->device = pd->device;
  CU(cudaSetDevice(e->device));
  CU(cudaDeviceGetAttribute(&e->num_sms, cudaDevAttrMultiProcessorCount, e->device));
  CU(cudaStreamCreateWithFlags(&e->st, cudaStreamNonBlocking));
  CU(cudaEventCreate(&e->ev0));
  CU(cudaEventCreate(&e->ev1));
  CU(cudaEventCreate(&e->ev2));
  if (md->n_layers != pd->n_layers)
    return fail(PPSD_EINVAL, "pipeline is " + std::to_string(pd->n_layers) + " layers deep but the model has " +
                                 std::to_string(md->n_layers));
  if (sched_configure(&e->cfg, pd->n_layers, pd->exit_depth, pd->exit_stage, pd->comm_latency) != 0)
    return fail(PPSD_EINVAL, "invalid pipeline (needs 2..96 stages, 1 <= exit_stage <= S-1, comm_latency >= 0)");
  e->S = e->cfg.S;
  e->lo = pd->stage_lo > 0 ? pd->stage_lo : 1;
  e->hi = pd->stage_hi > 0 ? pd->stage_hi : e->S;
  if (e->lo > e->hi || e->hi > e->S) return fail(PPSD_EINVAL, "bad local stage range");
  e->first_local_layer = e->cfg.stage_first[e->lo];
  e->n_local_layers = 0;
  for (int s = e->lo; s <= e->hi; ++s) {
    e->max_local_layers = std::max(e->max_local_layers, (int)e->cfg.stage_layers[s]);
    e->n_local_layers += e->cfg.stage_layers[s];
  }
  const int max_ctx = md->max_ctx > 0 ? md->max_ctx : 4096;
  e->md.max_ctx = max_ctx;
  const int nslot = e->cfg.nslot;
  e->nbuf = std::max(nslot, (int)kMaxVec);  // + a prefill chunk / EESD verify group

  CU(dalloc(&e->d_sched, sizeof(Sched)));
  CU(dalloc(&e->d_work, sizeof(Work)));
  CU(dalloc(&e->d_work_ar, sizeof(Work)));
  CU(dalloc(&e->d_work_deep, sizeof(Work)));
  CU(dalloc(&e->d_work_head, sizeof(Work)));
  CU(dalloc(&e->d_work_p2, sizeof(Work)));
  CU(dalloc(&e->d_work_head_pf, sizeof(Work)));
  CU(dalloc(&e->d_ctx, sizeof(TickCtx)));
  CU(dalloc(&e->d_arctl, sizeof(ArCtl)));
  CU(dalloc(&e->d_tokens, sizeof(int32_t) * (max_ctx + 8)));
  CU(dalloc(&e->d_eesd, sizeof(EesdState)));
  CU(dalloc(&e->d_kerr, sizeof(int32_t)));
  CU(cudaMallocHost(reinterpret_cast<void**>(&e->h_sched), sizeof(Sched)));

  TickCtx& c = e->h_ctx;
  c.sched = e->d_sched;
  c.work = e->d_work;
  c.work_ar = e->d_work_ar;
  c.work_deep = e->d_work_deep;
  c.work_head = e->d_work_head;
  c.work_p2 = e->d_work_p2;
  c.work_head_pf = e->d_work_head_pf;
  c.tokens = e->d_tokens;
  c.model = md->kind;
  c.lo = e->lo;
  c.hi = e->hi;
  c.n_layers = md->n_layers;
  c.vocab = md->vocab;
  c.model_stages = e->cfg.S;
  c.prefill_chunk = kMaxVec;

  if (md->kind == PPSD_MODEL_TOYLM) {
    if (md->vocab < 2) return fail(PPSD_EINVAL, "vocab must be >= 2");
    if (md->toy_misalignment < 0) return fail(PPSD_EINVAL, "misalignment must be non-negative");
    CU(dalloc(&e->d_pdig, sizeof(uint64_t) * (max_ctx + 9)));
    CU(dalloc(&e->d_chain_dig, sizeof(uint64_t) * nslot));
    c.pdig = e->d_pdig;
    c.chain_dig = e->d_chain_dig;
    c.beta = md->toy_misalignment;
    c.toy_seed = md->toy_seed;
    CU(dalloc(&e->d_logits64, sizeof(double) * 2 * (size_t)md->vocab));
    c.logits64 = e->d_logits64;
  } else if (md->kind == PPSD_MODEL_TRANSFORMER) {
    Dims& d = e->dm;
    d.d = md->d_model;
    d.H = md->n_heads;
    d.KV = md->n_kv_heads;
    d.hd = md->head_dim;
    d.ffn = md->ffn_dim;
    d.V = md->vocab;
    d.max_ctx = max_ctx;
    d.nslot = e->nbuf;
    d.eps = md->rms_eps;
    d.kv_bf16 = md->kv_bf16;
    if (d.KV <= 0 || d.H % d.KV != 0 || !attn_supported(d.hd, d.H / d.KV))
      return fail(PPSD_EUNSUPPORTED, "unsupported head geometry (head_dim in {16,32,64,128}, H/KV in {1,2,4,8})");
    if (d.d % 8 || d.ffn % 8 || (d.H * d.hd) % 8)
      return fail(PPSD_EUNSUPPORTED, "d_model, ffn_dim and H*head_dim must be multiples of 8");
    const bool need_head = (e->cfg.k >= e->lo && e->cfg.k <= e->hi) || e->hi == e->S;
    if (!w || !w->final_norm || !w->exit_norm || !w->rope_cos || (e->lo == 1 && !w->embed) ||
        (need_head && !w->lm_head))
      return fail(PPSD_EINVAL, "missing transformer weights");
    const int Rq = (d.H + 2 * d.KV) * d.hd;
    const int shapes[kNumMats][2] = {{Rq, d.d}, {d.d, d.H * d.hd}, {2 * d.ffn, d.d},
                                     {d.d, d.ffn}, {d.V, d.d}, {d.V, d.d}};
    for (int m = 0; m < kNumMats; ++m) {
      for (int b = 0; b < 2; ++b) {
        if (m == kMatHead && b) continue;
        GemvPlan& p = b ? e->gpb[m] : e->gp[m];
        p.R = shapes[m][0];
        p.K = shapes[m][1];
        // one weight pass for every vector of a group: one 16-column B block
        // (<= 5 vectors x 3 parts) for the decode tick, the folded deep batch
        // and the PPSD head; 3 (<= 16 vectors) for prefill chunks and EESD
        const int nblk = b ? 3 : 1;
        // PPSD_TC_GRID=<qkv>,<o>,<gu>,<down>: SMs a matrix's plan spreads over
        // (experiments; 0 or absent: all)
        int sms = e->num_sms;
        if (const char* gv = getenv("PPSD_TC_GRID")) {
          int f[4] = {0, 0, 0, 0};
          sscanf(gv, "%d,%d,%d,%d", &f[0], &f[1], &f[2], &f[3]);
          if (m < 4 && f[m] > 0 && f[m] <= e->num_sms) sms = f[m];
        }
        if (tc_pick(p.K, p.R, nblk, sms, &p.tc, m) != 0)
          return fail(PPSD_EUNSUPPORTED, "no tensor-core GEMV plan for matrix " + std::to_string(m) + " [" +
                                             std::to_string(p.R) + " x " + std::to_string(p.K) + "]");
        CU(tc_set_attrs(m, p.tc.cs, p.tc.smem));
        if (getenv("PPSD_TC_VERBOSE"))
          fprintf(stderr, "tc plan mat %d b %d: R %d K %d JS %d NJ %d CS %d grid %d TG %d nb %d NS %d smem %zu\n", m, b,
                  p.R, p.K, p.tc.js, p.tc.nj, p.tc.cs, p.tc.grid, p.tc.tg, p.tc.nb, p.tc.ns, p.tc.smem);
        p.m = b ? kMaxVec : (m == kMatHead ? 2 : 1);
      }
    }
    {
      AttnArgs aa{};
      aa.dm = d;
      CU(attn_set_attrs(aa));
      e->attn_per_sm = std::max(1, std::min(8, attn_ctas_per_sm()));
      // cluster attention for the one-vector launches (PPSD_ATTN_CL=0: off)
      const char* cv = getenv("PPSD_ATTN_CL");
      e->attn_cl = !(cv && cv[0] == '0') && attn_cl_setup(aa);
      // batched cluster launches (PPSD_ATTN_CLB=0: split-K kernel for every batch)
      const char* cb = getenv("PPSD_ATTN_CLB");
      e->attn_clb = e->attn_cl && !(cb && cb[0] == '0') && attn_cl4_ok();
      e->attn_clb_cs = cb && atoi(cb) == 8 ? 8 : 4;
    }
    e->lm_head = reinterpret_cast<const __nv_bfloat16*>(w->lm_head);
    e->final_norm = w->final_norm;
    e->exit_norm = w->exit_norm;
    e->rope_cos = w->rope_cos;
    e->rope_sin = w->rope_sin;
    c.embed = reinterpret_cast<const __nv_bfloat16*>(w->embed);
    c.d = d.d;
    // KV page pool for the local layers; identity page table
    e->max_pages = (max_ctx + kPage - 1) / kPage;
    const size_t esz = d.kv_bf16 ? 2 : 4;
    const size_t per_layer = (size_t)e->max_pages * kPage * d.KV * d.hd * esz;
    // exit-head layer: one more decoder layer (global index N) with its own KV
    // (after the local layers in the pool) and activation rows from nbuf on
    // Across ranks only the rank that owns the exit stage k runs (and holds)
    // the head layer; the replicated scheduler plans it there alone.
    e->hl = md->exit_head_layer != 0 && e->cfg.k >= e->lo && e->cfg.k <= e->hi;
    if (e->hl) {
      const ppsd_layer_weights& X = w->exit_layer;
      if (!X.qkv || !X.o || !X.gu || !X.down || !X.attn_norm || !X.mlp_norm)
        return fail(PPSD_EINVAL, "missing exit-head layer weights");
      c.hl = 1;
      c.hl_layer = md->n_layers;
      c.hl_split = e->cfg.shallow_layers - e->first_local_layer;  // local layers before the exit
      c.head_row = e->nbuf;
    }
    const int kv_layers = e->n_local_layers + (e->hl ? 1 : 0);
    CU(cudaMalloc(&e->d_kv, per_layer * 2 * kv_layers));
    std::vector<int32_t> pt(e->max_pages);
    for (int i = 0; i < e->max_pages; ++i) pt[i] = i;
    CU(dalloc(&e->d_page_table, sizeof(int32_t) * e->max_pages));
    CU(cudaMemcpy(e->d_page_table, pt.data(), sizeof(int32_t) * e->max_pages, cudaMemcpyHostToDevice));
    e->h_layers.assign(md->n_layers + (e->hl ? 1 : 0), LayerW{});
    for (int l = 0; l < md->n_layers; ++l) {
      LayerW& L = e->h_layers[l];
      const int li = l - e->first_local_layer;
      if (li < 0 || li >= e->n_local_layers) continue;
      if (!w->w_qkv[l] || !w->w_o[l] || !w->w_gu[l] || !w->w_down[l] || !w->attn_norm[l] || !w->mlp_norm[l])
        return fail(PPSD_EINVAL, "missing weights for local layer " + std::to_string(l));
      L.qkv = reinterpret_cast<const __nv_bfloat16*>(w->w_qkv[l]);
      L.o = reinterpret_cast<const __nv_bfloat16*>(w->w_o[l]);
      L.gu = reinterpret_cast<const __nv_bfloat16*>(w->w_gu[l]);
      L.down = reinterpret_cast<const __nv_bfloat16*>(w->w_down[l]);
      L.attn_norm = w->attn_norm[l];
      L.mlp_norm = w->mlp_norm[l];
      L.kc = static_cast<char*>(e->d_kv) + per_layer * (2 * li);
      L.vc = static_cast<char*>(e->d_kv) + per_layer * (2 * li + 1);
    }
    if (e->hl) {
      LayerW& L = e->h_layers[md->n_layers];
      const ppsd_layer_weights& X = w->exit_layer;
      L.qkv = reinterpret_cast<const __nv_bfloat16*>(X.qkv);
      L.o = reinterpret_cast<const __nv_bfloat16*>(X.o);
      L.gu = reinterpret_cast<const __nv_bfloat16*>(X.gu);
      L.down = reinterpret_cast<const __nv_bfloat16*>(X.down);
      L.attn_norm = X.attn_norm;
      L.mlp_norm = X.mlp_norm;
      L.kc = static_cast<char*>(e->d_kv) + per_layer * (2 * e->n_local_layers);
      L.vc = static_cast<char*>(e->d_kv) + per_layer * (2 * e->n_local_layers + 1);
    }
    CU(dalloc(&e->d_layers, sizeof(LayerW) * e->h_layers.size()));
    CU(cudaMemcpy(e->d_layers, e->h_layers.data(), sizeof(LayerW) * e->h_layers.size(), cudaMemcpyHostToDevice));
    // weights of one matrix kind at a fixed stride across the local layers
    // (one allocation per kind, models.py): the GEMV producer computes the
    // address instead of loading it
    for (int m = kMatQKV; m <= kMatDown; ++m) {
      auto ptr = [&](int l) -> long long {
        const LayerW& L = e->h_layers[l];
        return (long long)(uintptr_t)(m == kMatQKV ? (const void*)L.qkv : m == kMatO ? (const void*)L.o
                                      : m == kMatGU ? (const void*)L.gu : (const void*)L.down);
      };
      const int l0 = e->first_local_layer, nl = e->n_local_layers;
      e->wstride[m] = WStride{};
      if (nl < 2) continue;
      const long long st = ptr(l0 + 1) - ptr(l0);
      bool ok = st > 0;
      for (int l = l0 + 2; ok && l < l0 + nl; ++l) ok = ptr(l) - ptr(l - 1) == st;
      if (ok) e->wstride[m] = WStride{(const void*)(uintptr_t)(ptr(l0) - (long long)l0 * st), st, l0 + nl};
    }
    const int qd = d.H * d.hd;
    // rank fold: a stage range of a multi-rank split (not the whole model)
    // whose deferred stages span >= 2 stages and whose batch fits one group;
    // runs in greedy decodes unless the schedule is PIPELINED (ppsd_get_schedule)
    e->rfold_ok = (e->lo > 1 || e->hi < e->S) && !e->hl && sched_rfold_useful(&e->cfg, e->lo, e->hi) &&
                  sched_rfold_width(&e->cfg, e->lo, e->hi) <= kMaxVec;
    c.rf_row0 = e->nbuf;
    // rows: chains / prefill chunk [0, nbuf); exit-head layer copies or the
    // rank fold's batch rows [nbuf, 2*nbuf)
    const size_t nb = (size_t)e->nbuf * (e->hl || e->rfold_ok ? 2 : 1);
    CU(dalloc(&e->d_x, sizeof(float) * nb * d.d));
    CU(dalloc(&e->d_q, sizeof(float) * nb * qd));
    CU(dalloc(&e->d_o, sizeof(float) * nb * qd));
    CU(dalloc(&e->d_h, sizeof(float) * nb * d.ffn));
    CU(dalloc(&e->d_logits, sizeof(float) * (kMaxVec + 1) * (size_t)d.V));  // folded: exit + batch rows
    CU(dalloc(&e->d_attn_part, sizeof(float) * nb * d.H * e->max_pages * (d.hd + 2)));
    CU(dalloc(&e->d_attn_cnt, sizeof(int32_t) * nb * d.KV));
    CU(dalloc(&e->d_head_part, sizeof(float) * 2 * kMaxVec * (size_t)e->num_sms));
    CU(dalloc(&e->d_head_cnt, sizeof(int32_t) * kMaxVec));
    c.logits32 = e->d_logits;
    c.x = e->d_x;
    // prompt tokens per prefill chunk: one batched weight pass
    {
      const int cmax = (int)kMaxVec;
      c.prefill_chunk = cmax;
      if (const char* v = getenv("PPSD_PREFILL_CHUNK")) c.prefill_chunk = std::min(std::max(atoi(v), 1), cmax);
    }
    // folded schedule: single-device engine, every in-flight chain fits one batch
    e->schedule = pd->schedule;
    e->fold_ok = e->lo == 1 && e->hi == e->S && sched_fold_width(&e->cfg) <= kMaxVec &&
                 pd->schedule != PPSD_SCHEDULE_PIPELINED;
    // AUTO folds wherever it can: the tensor-core GEMV streams a weight once
    // for every vector of the deep batch at the cost of one vector
    e->fold_auto = e->fold_ok;
    if (int rc = setup_pass(e)) return rc;
    if (pd->schedule == PPSD_SCHEDULE_FOLDED && !e->fold_ok)
      return fail(PPSD_EUNSUPPORTED, "folded schedule needs all stages on this device and at most " +
                                         std::to_string(kMaxVec) + " chains in flight");
  } else if (md->kind != PPSD_MODEL_BERNOULLI) {
    return fail(PPSD_EINVAL, "unknown model kind");
  }
  if (md->kind != PPSD_MODEL_BERNOULLI) {  // sampling-mode float64 scratch
    CU(dalloc(&e->d_pdist, sizeof(double) * (size_t)std::max(nslot, (int)kMaxVec) * md->vocab));
    CU(dalloc(&e->d_qbuf, sizeof(double) * (size_t)md->vocab));
    CU(dalloc(&e->d_wbuf, sizeof(double) * (size_t)md->vocab));
    c.pdist = e->d_pdist;
    c.qbuf = e->d_qbuf;
    c.wbuf = e->d_wbuf;
  }
  c.greedy = 1;
  CU(cudaMemcpy(e->d_ctx, &c, sizeof(TickCtx), cudaMemcpyHostToDevice));
  return build_graphs(e);
}

extern "C" int ppsd_engine_create(const ppsd_model_desc* model, const ppsd_weights* weights,
                                  const ppsd_pipeline_desc* pipe, void* cuda_stream, ppsd_engine** out) {
  (void)cuda_stream;
  if (!model || !pipe || !out) return fail(PPSD_EINVAL, "null argument");
  ppsd_engine* e = new ppsd_engine();
  int rc = create_impl(model, weights, pipe, e);
  if (rc != PPSD_OK) {
    std::string keep = g_err;
    free_engine(e);
    g_err = keep;
    return rc;
  }
  *out = e;
  return PPSD_OK;
}

extern "C" int ppsd_engine_destroy(ppsd_engine* e) {
  free_engine(e);
  return PPSD_OK;
}

// Persistent layer pass (tcpass.cu): on when the engine owns its device (all
// stages local, PDL on: the grid barriers need every CTA resident; several
// engines sharing a GPU run the per-kernel sequence, same arithmetic), the
// head geometry has a pass instantiation and PPSD_PASS != 0.
static int setup_pass(ppsd_engine* e) {
  e->pass = false;
  // measured slower than the per-kernel sequence on the 7B shape (DESIGN.md
  // §8): opt-in experiment (PPSD_PASS=1)
  const char* ev = getenv("PPSD_PASS");
  if (!(ev && ev[0] == '1') || e->lo != 1 || e->hi != e->S || !ppsd::g_pdl) return PPSD_OK;
  const int qpk = e->dm.H / e->dm.KV;
  if (!tc_pass_supported(e->dm.hd, qpk)) return PPSD_OK;
  int cs = 1;
  for (int m = 0; m < 4; ++m) cs = std::max(cs, std::max(e->gp[m].tc.cs, e->gpb[m].tc.cs));
  if (cs > 2) return PPSD_OK;
  const size_t kv_el = e->dm.kv_bf16 ? 2 : 4;
  const size_t kvb = 2 * (size_t)kPage * e->dm.hd * kv_el;          // one worker's K + V page blocks
  const size_t scr = (tc_pass_scratch_bytes(e->dm.hd, qpk, e->dm.kv_bf16) + 127) / 128 * 128;
  const size_t cap = 221 * 1024;
  for (int v = 0; v < 2; ++v) {
    PassPlan& pl = e->pp[v];
    pl = PassPlan{};
    pl.nblk = v ? 3 : 1;
    size_t slot = 0, over = 0;
    for (int m = 0; m < 4; ++m) {
      const TcPlan& t = (v ? e->gpb[m] : e->gp[m]).tc;
      slot = std::max(slot, (size_t)t.tg * t.js * 1024);
      over = std::max(over, (size_t)(16 - t.tg) * t.js * 1024);
    }
    size_t bst = 0;
    for (int m = 0; m < 4; ++m) {
      const TcPlan& t = (v ? e->gpb[m] : e->gp[m]).tc;
      const size_t jb = (size_t)t.tg * t.js * 1024;
      int nb = (int)(slot / jb);
      const int njr = (t.nj + t.cs - 1) / t.cs;
      nb = std::max(1, std::min(nb, njr));
      pl.nb[m] = nb;
      bst = std::max(bst, (size_t)nb * pl.nblk * t.js * 2048);
    }
    const size_t recv = cs > 1 ? (size_t)kMaxVec * 128 * 4 : 0;
    const int cands[][2] = {{4, 2}, {3, 2}, {4, 1}, {3, 1}, {2, 2}, {2, 1}};
    for (const auto& c : cands) {
      const int ns = c[0], wk = c[1];
      const size_t ring = (size_t)ns * slot;
      const size_t uni = std::max((size_t)ns * bst, (size_t)wk * kvb);
      const size_t pad = over > uni ? over - uni : 0;
      const size_t scr_off = (ring + uni + pad + 127) / 128 * 128;
      const size_t bar_off = scr_off + (size_t)wk * scr;
      const size_t total = bar_off + 256 + recv + 1024;
      if (total > cap) continue;
      pl.ok = true;
      pl.ns = ns;
      pl.workers = wk;
      pl.slot_bytes = (int)slot;
      pl.b_stage = (int)bst;
      pl.attn_off = (int)ring;
      pl.attn_kv_bytes = (int)kvb;
      pl.scr_off = (int)scr_off;
      pl.bar_off = (int)bar_off;
      pl.smem = total;
      break;
    }
    if (!pl.ok) return PPSD_OK;
    CU(tc_pass_set_attrs(cs, e->dm.hd, qpk, e->dm.kv_bf16, cap));  // one kernel serves both plans
    if (getenv("PPSD_TC_VERBOSE"))
      fprintf(stderr, "tc pass plan %d: CS %d NS %d workers %d slot %d b_stage %d smem %zu\n", v, cs, pl.ns,
              pl.workers, pl.slot_bytes, pl.b_stage, pl.smem);
  }
  CU(cudaSetDevice(e->device));
  CU(dalloc(&e->d_pass_bar, 3 * sizeof(unsigned long long)));
  CU(cudaMemset(e->d_pass_bar, 0, 3 * sizeof(unsigned long long)));
  e->pass_cs = cs;
  e->pass = true;
  return PPSD_OK;
}

// ---------------------------------------------------------------------------
// decode

// Sticky GEMV error word (tcgemv.cu / tcpass.cu: a speculative-start hint
// that did not match the work descriptor, a layer-pass grid barrier that
// timed out): such a decode is reported as PPSD_ESTATE, never returned as
// tokens. Called after the stream drained.
static int check_kerr(ppsd_engine* e) {
  int32_t v = 0;
  CU(cudaMemcpy(&v, e->d_kerr, sizeof(v), cudaMemcpyDeviceToHost));
  if (v == 0) return PPSD_OK;
  CU(cudaMemset(e->d_kerr, 0, sizeof(v)));
  return fail(PPSD_ESTATE, v & kAttnErrRows ? "cluster attention: more active vectors than launched rows (results discarded)"
                          : v & kGemvErrHint ? "GEMV speculative start: hint did not match the work (results discarded)"
                          : "layer pass: a grid barrier timed out (results discarded)");
}

static int check_prompt(const ppsd_engine* e, const int32_t* prompt, int n_prompt) {
  if (n_prompt <= 0 || !prompt) return fail(PPSD_EINVAL, "prompt must be non-empty");
  for (int i = 0; i < n_prompt; ++i)
    if (prompt[i] < 0 || prompt[i] >= e->md.vocab)
      return fail(PPSD_EINVAL, "prompt token " + std::to_string(prompt[i]) + " outside vocab of " +
                                   std::to_string(e->md.vocab));
  return PPSD_OK;
}

static int upload_prompt(ppsd_engine* e, const int32_t* prompt, int n_prompt) {
  CU(cudaMemcpyAsync(e->d_tokens, prompt, sizeof(int32_t) * n_prompt, cudaMemcpyHostToDevice, e->st));
  if (e->md.kind == PPSD_MODEL_TOYLM) {
    std::vector<uint64_t> pd(n_prompt + 1);
    pd[0] = hmix64(e->md.toy_seed ^ kSeqSalt);  // toylm.py:72-74
    for (int i = 0; i < n_prompt; ++i) pd[i + 1] = toy_extend(pd[i], prompt[i]);
    CU(cudaMemcpyAsync(e->d_pdig, pd.data(), sizeof(uint64_t) * (n_prompt + 1), cudaMemcpyHostToDevice, e->st));
    CU(cudaStreamSynchronize(e->st));  // pd is a host temporary
  }
  return PPSD_OK;
}

// Run the prompt prefill (transformer): KV for tokens 0..n_prompt-2.
static int prefill(ppsd_engine* e, int n_prompt, double* ms, int64_t* launches) {
  *ms = 0;
  if (e->md.kind != PPSD_MODEL_TRANSFORMER || n_prompt < 2) return PPSD_OK;
  ArCtl ctl{0, e->first_local_layer, e->n_local_layers, n_prompt - 1};
  CU(cudaMemcpyAsync(e->d_arctl, &ctl, sizeof(ctl), cudaMemcpyHostToDevice, e->st));
  CU(cudaEventRecord(e->ev0, e->st));
  const int chunks = (n_prompt - 1 + e->h_ctx.prefill_chunk - 1) / e->h_ctx.prefill_chunk;
  NvtxRange nv("ppsd.prefill chunks", 0, chunks);
  for (int i = 0; i < chunks; ++i) CU(cudaGraphLaunch(e->g_prefill, e->st));
  CU(cudaEventRecord(e->ev1, e->st));
  CU(cudaEventSynchronize(e->ev1));
  float f = 0;
  CU(cudaEventElapsedTime(&f, e->ev0, e->ev1));
  *ms = f;
  *launches += (int64_t)chunks * e->prefill_launches;
  return PPSD_OK;
}

static int ensure_trace(ppsd_engine* e, int64_t cap) {
  if (cap <= e->trace_cap) return PPSD_OK;
  // no cudaFree here: it synchronizes the device, which would wait on other
  // engines of this process spinning on p2p flags this engine has yet to set
  if (e->d_trace) e->retired.push_back(e->d_trace);
  e->d_trace = nullptr;
  e->trace_cap = 0;
  CU(cudaMalloc(&e->d_trace, sizeof(TraceRow) * cap));
  e->trace_cap = cap;
  return PPSD_OK;
}

static void fill_metrics(const ppsd_engine* e, const Sched& s, ppsd_metrics* m) {
  m->committed_tokens = s.committed;
  m->ticks = s.t;
  m->accepts = s.accepts;
  m->rejects = s.rejects;
  const int64_t drafted = s.accepts + s.rejects;
  m->alpha_valid = drafted > 0;
  m->alpha_all_measured = drafted > 0 ? (double)s.accepts / (double)drafted : 0.0;
  m->throughput = s.t > 0 ? (double)s.committed / (double)s.t : 0.0;
  m->speedup_vs_ar = m->throughput * (double)(e->S * e->cfg.per);  // pipesim.py:274
}

static int run_machine(ppsd_engine* e, int model, int n_prompt, int stop, int force_reject, double alpha,
                       uint64_t verify_seed, ppsd_metrics* out, ppsd_trace_row* trace, int64_t trace_cap,
                       int64_t* trace_len, int64_t launches) {
  const int64_t max_ticks = (int64_t)stop * e->S * e->cfg.per + (int64_t)e->S * e->cfg.per + 8;
  int64_t cap = 0;
  if (trace) {
    cap = max_ticks * (e->S + 2);
    if (trace_cap < cap) cap = trace_cap;
    int rc = ensure_trace(e, cap);
    if (rc) return rc;
  }
  // folded schedule: greedy model decodes, and sampling when the draft is
  // drawn in the launch tick (exit_stage 1: the eager exit logits are current)
  const bool fold = e->fold_ok && (e->schedule == PPSD_SCHEDULE_FOLDED ||
                                   (e->schedule == PPSD_SCHEDULE_AUTO && e->fold_auto)) &&
                    model != 0 && (e->h_ctx.greedy || e->cfg.k == 1);
  Sched& s = *e->h_sched;
  memset(&s, 0, sizeof(Sched));
  s.c = e->cfg;
  s.c.fold = fold ? 1 : 0;
  s.c.model = model;
  s.c.force_reject = force_reject;
  s.c.stop = stop;
  s.c.n_prompt = n_prompt;
  s.c.alpha = alpha;
  s.c.verify_seed = verify_seed;
  sched_reset(&s);
  e->h_ctx.trace = trace ? e->d_trace : nullptr;
  e->h_ctx.inbox = nullptr;  // single-rank run
  e->h_ctx.outbox = nullptr;
  e->h_ctx.trace_cap = cap;
  e->h_ctx.fold = fold ? 1 : 0;
  CU(cudaMemcpyAsync(e->d_ctx, &e->h_ctx, sizeof(TickCtx), cudaMemcpyHostToDevice, e->st));
  CU(cudaMemcpyAsync(e->d_sched, &s, sizeof(Sched), cudaMemcpyHostToDevice, e->st));
  CU(cudaEventRecord(e->ev0, e->st));
  cudaGraphExec_t tick = e->g_tick;
  int64_t per_tick = e->tick_launches;
  if (fold) {  // the graph's scheduler node plans tick 1 (finishing "tick 0" is a no-op)
    tick = e->g_fold;
    per_tick = e->fold_tick_launches;
  } else {
    sched_tick_kernel<<<1, 256, 0, e->st>>>(e->d_ctx, 1);
    CU(cudaGetLastError());
    launches += 1;
  }
  int64_t committed = 0, ticks_launched = 0;
  // small readback: committed .. error (8 int32 after SchedCfg)
  const size_t off = offsetof(Sched, t);
  const size_t len = offsetof(Sched, verify_counter) - off;
  NvtxRange nv_decode("ppsd.decode");
  for (;;) {
    const int64_t n = std::max<int64_t>(1, (int64_t)stop - committed);
    {
      NvtxRange nv("ppsd.ticks", ticks_launched + 1, ticks_launched + n);
      for (int64_t i = 0; i < n; ++i) CU(cudaGraphLaunch(tick, e->st));
    }
    ticks_launched += n;
    CU(cudaMemcpyAsync(reinterpret_cast<char*>(&s) + off, reinterpret_cast<char*>(e->d_sched) + off, len,
                       cudaMemcpyDeviceToHost, e->st));
    CU(cudaStreamSynchronize(e->st));
    if (s.error) break;
    if (s.done) break;
    committed = s.committed;
    if (ticks_launched > max_ticks + 4)
      return fail(PPSD_ESTATE, "tick machine did not converge (internal error)");
  }
  CU(cudaEventRecord(e->ev1, e->st));
  CU(cudaMemcpyAsync(&s, e->d_sched, sizeof(Sched), cudaMemcpyDeviceToHost, e->st));
  CU(cudaEventSynchronize(e->ev1));
  CU(cudaStreamSynchronize(e->st));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
  if (int rc = check_kerr(e)) return rc;
  if (s.error & kErrOrder) return fail(PPSD_ESTATE, "verdicts must land in position order");
  if (s.error & kErrTransit) return fail(PPSD_ESTATE, "transit queue overflow");
  if (s.error & kErrTrace) return fail(PPSD_ESTATE, "trace buffer too small");
  fill_metrics(e, s, out);
  out->decode_ms = ms;
  out->gpu_launches = launches + ticks_launched * per_tick + (int64_t)s.fold_batches * e->fold_deep_launches;
  out->schedule = fold ? PPSD_SCHEDULE_FOLDED : PPSD_SCHEDULE_PIPELINED;
  out->deep_batches = s.fold_batches;
  out->deep_vectors = s.fold_vectors;
  out->deep_pos_sum = s.fold_pos_sum;
  out->comb_heads = s.fold_comb;
  if (trace) {
    const int64_t nrows = std::min<int64_t>(s.trace_n, trace_cap);
    if (nrows > 0)
      CU(cudaMemcpy(trace, e->d_trace, sizeof(TraceRow) * nrows, cudaMemcpyDeviceToHost));
    if (trace_len) *trace_len = nrows;
  } else if (trace_len) {
    *trace_len = 0;
  }
  return PPSD_OK;
}

// Sampling mode: the three _ToyVerifier streams (pipesim.py:339-344) derived
// from the caller's RngStream seed; greedy runs draw nothing.
static int set_mode(ppsd_engine* e, int greedy, uint64_t rng_seed) {
  e->h_ctx.greedy = greedy ? 1 : 0;
  e->h_ctx.draft_seed = derive_seed_str(rng_seed, "draft");
  e->h_ctx.commit_seed = derive_seed_str(rng_seed, "commit");
  e->verify_seed = derive_seed_str(rng_seed, "verify");
  CU(cudaMemcpyAsync(e->d_ctx, &e->h_ctx, sizeof(TickCtx), cudaMemcpyHostToDevice, e->st));
  return PPSD_OK;
}

extern "C" int ppsd_decode(ppsd_engine* e, int32_t greedy, uint64_t rng_seed, const int32_t* prompt,
                           int32_t n_prompt, int32_t max_tokens, int32_t force_reject, int32_t* out_tokens,
                           ppsd_metrics* out, ppsd_trace_row* trace, int64_t trace_cap, int64_t* trace_len) {
  if (!e || !out) return fail(PPSD_EINVAL, "null argument");
  if (e->lo != 1 || e->hi != e->S) return fail(PPSD_EINVAL, "engine holds a stage subset: use ppsd_step_*");
  if (e->md.kind == PPSD_MODEL_BERNOULLI) return fail(PPSD_EINVAL, "Bernoulli engines run ppsd_simulate");
  int rc = check_prompt(e, prompt, n_prompt);
  if (rc) return rc;
  if (max_tokens < 0) return fail(PPSD_EINVAL, "max_tokens must be >= 0");
  memset(out, 0, sizeof(*out));
  if (trace_len) *trace_len = 0;
  if (max_tokens == 0) return PPSD_OK;  // pipesim.py:620-621
  const int64_t need = (int64_t)n_prompt + max_tokens + (int64_t)e->S * e->cfg.per + 2;
  if (need > e->md.max_ctx)
    return fail(PPSD_EINVAL, "prompt + max_tokens exceeds the engine's max_ctx (" + std::to_string(e->md.max_ctx) + ")");
  CU(cudaSetDevice(e->device));
  rc = set_mode(e, greedy, rng_seed);
  if (rc) return rc;
  rc = upload_prompt(e, prompt, n_prompt);
  if (rc) return rc;
  int64_t launches = 0;
  double pre_ms = 0;
  rc = prefill(e, n_prompt, &pre_ms, &launches);
  if (rc) return rc;
  rc = run_machine(e, 1, n_prompt, max_tokens, force_reject, 0.0, greedy ? 0 : e->verify_seed, out, trace,
                   trace_cap, trace_len, launches);
  if (rc) return rc;
  out->prefill_ms = pre_ms;
  if (out_tokens)
    CU(cudaMemcpy(out_tokens, e->d_tokens + n_prompt, sizeof(int32_t) * max_tokens, cudaMemcpyDeviceToHost));
  return PPSD_OK;
}

extern "C" int ppsd_set_schedule(ppsd_engine* e, int32_t schedule) {
  if (!e) return fail(PPSD_EINVAL, "null argument");
  if (schedule < PPSD_SCHEDULE_AUTO || schedule > PPSD_SCHEDULE_FOLDED) return fail(PPSD_EINVAL, "unknown schedule");
  if (schedule == PPSD_SCHEDULE_FOLDED && !e->fold_ok && !e->rfold_ok)
    return fail(PPSD_EUNSUPPORTED, "this engine cannot run the folded schedule");
  e->schedule = schedule;
  return PPSD_OK;
}

extern "C" int ppsd_get_schedule(ppsd_engine* e, int32_t greedy, int32_t* schedule) {
  if (!e || !schedule) return fail(PPSD_EINVAL, "null argument");
  const bool fold = e->fold_ok && e->md.kind == PPSD_MODEL_TRANSFORMER &&
                    (e->schedule == PPSD_SCHEDULE_FOLDED || (e->schedule == PPSD_SCHEDULE_AUTO && e->fold_auto)) &&
                    (greedy || e->cfg.k == 1);
  // a rank of a multi-rank split: the per-rank fold (greedy)
  const bool rfold = e->rfold_ok && greedy && e->schedule != PPSD_SCHEDULE_PIPELINED;
  *schedule = fold || rfold ? PPSD_SCHEDULE_FOLDED : PPSD_SCHEDULE_PIPELINED;
  return PPSD_OK;
}

// ToyLM.empirical_alpha / greedy_agreement (toylm.py:160-192): per-prefix
// sum(min(p, q)) and argmax agreement of the exit head at exit_depth, for
// n_prefixes prefixes of prefix_len tokens (row-major). The caller sums the
// per-prefix values in order, as the reference does.
extern "C" int ppsd_toy_alignment(ppsd_engine* e, int32_t exit_depth, int32_t n_prefixes, int32_t prefix_len,
                                  const int32_t* prefixes, double* out_minsum, int32_t* out_agree) {
  if (!e || !prefixes || !out_minsum || !out_agree) return fail(PPSD_EINVAL, "null argument");
  if (e->md.kind != PPSD_MODEL_TOYLM) return fail(PPSD_EINVAL, "alignment needs a ToyLM engine");
  if (n_prefixes < 1) return fail(PPSD_EINVAL, "n_prefixes must be >= 1");
  if (prefix_len < 1) return fail(PPSD_EINVAL, "prefix must be non-empty");
  if (exit_depth < 1 || exit_depth > e->md.n_layers)
    return fail(PPSD_EINVAL, "exit_depth must lie in [1, " + std::to_string(e->md.n_layers) + "], got " +
                                 std::to_string(exit_depth));
  for (int64_t i = 0; i < (int64_t)n_prefixes * prefix_len; ++i)
    if (prefixes[i] < 0 || prefixes[i] >= e->md.vocab) return fail(PPSD_EINVAL, "prefix token outside vocab");
  CU(cudaSetDevice(e->device));
  std::vector<uint64_t> pd(n_prefixes);
  for (int i = 0; i < n_prefixes; ++i) {  // sequence digests (toylm.py:72-86)
    uint64_t d = hmix64(e->md.toy_seed ^ kSeqSalt);
    for (int j = 0; j < prefix_len; ++j) d = toy_extend(d, prefixes[(size_t)i * prefix_len + j]);
    pd[i] = d;
  }
  const size_t V = (size_t)e->md.vocab;
  uint64_t* d_pd = nullptr;
  double *d_scr = nullptr, *d_ms = nullptr;
  int* d_ag = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_pd);
    cudaFree(d_scr);
    cudaFree(d_ms);
    cudaFree(d_ag);
  };
  if (cudaMalloc(&d_pd, sizeof(uint64_t) * n_prefixes) != cudaSuccess ||
      cudaMalloc(&d_scr, sizeof(double) * 4 * V * n_prefixes) != cudaSuccess ||
      cudaMalloc(&d_ms, sizeof(double) * n_prefixes) != cudaSuccess ||
      cudaMalloc(&d_ag, sizeof(int) * n_prefixes) != cudaSuccess) {
    cleanup();
    return fail(PPSD_ECUDA, "alignment scratch allocation failed");
  }
  cudaError_t ce = cudaMemcpyAsync(d_pd, pd.data(), sizeof(uint64_t) * n_prefixes, cudaMemcpyHostToDevice, e->st);
  if (ce == cudaSuccess) {
    toy_alignment_kernel<<<n_prefixes, 256, 0, e->st>>>(d_pd, e->md.n_layers, exit_depth, e->md.vocab,
                                                        e->md.toy_seed, e->md.toy_misalignment, d_scr, d_ms, d_ag);
    ce = cudaGetLastError();
  }
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(out_minsum, d_ms, sizeof(double) * n_prefixes, cudaMemcpyDeviceToHost, e->st);
  if (ce == cudaSuccess) ce = cudaMemcpyAsync(out_agree, d_ag, sizeof(int) * n_prefixes, cudaMemcpyDeviceToHost, e->st);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(e->st);
  cleanup();
  CU(ce);
  return PPSD_OK;
}

extern "C" int ppsd_simulate(ppsd_engine* e, double alpha, uint64_t verify_seed, int32_t horizon,
                             int32_t force_reject, ppsd_metrics* out, ppsd_trace_row* trace, int64_t trace_cap,
                             int64_t* trace_len) {
  if (!e || !out) return fail(PPSD_EINVAL, "null argument");
  if (e->md.kind != PPSD_MODEL_BERNOULLI) return fail(PPSD_EINVAL, "ppsd_simulate needs a Bernoulli engine");
  if (horizon < 1) return fail(PPSD_EINVAL, "horizon must be >= 1");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(PPSD_EINVAL, "BERNOULLI oracle needs alpha in [0, 1]");
  memset(out, 0, sizeof(*out));
  CU(cudaSetDevice(e->device));
  return run_machine(e, 0, 0, horizon, force_reject, alpha, verify_seed, out, trace, trace_cap, trace_len, 0);
}

extern "C" int ppsd_decode_ar(ppsd_engine* e, int32_t greedy, uint64_t rng_seed, const int32_t* prompt,
                              int32_t n_prompt, int32_t max_tokens, int32_t* out_tokens, ppsd_metrics* out) {
  if (!e || !out) return fail(PPSD_EINVAL, "null argument");
  if (e->md.kind == PPSD_MODEL_BERNOULLI) return fail(PPSD_EINVAL, "Bernoulli engines have no model");
  if (e->lo != 1 || e->hi != e->S) return fail(PPSD_EINVAL, "engine holds a stage subset");
  int rc = check_prompt(e, prompt, n_prompt);
  if (rc) return rc;
  if (max_tokens < 0) return fail(PPSD_EINVAL, "max_tokens must be >= 0");
  memset(out, 0, sizeof(*out));
  if (max_tokens == 0) return PPSD_OK;
  if ((int64_t)n_prompt + max_tokens + 2 > e->md.max_ctx) return fail(PPSD_EINVAL, "exceeds max_ctx");
  CU(cudaSetDevice(e->device));
  rc = set_mode(e, greedy, rng_seed);
  if (rc) return rc;
  rc = upload_prompt(e, prompt, n_prompt);
  if (rc) return rc;
  int64_t launches = 0;
  if (e->md.kind == PPSD_MODEL_TOYLM) {
    CU(cudaEventRecord(e->ev0, e->st));
    toy_ar_kernel<<<1, 256, 0, e->st>>>(e->d_ctx, n_prompt, max_tokens);
    CU(cudaGetLastError());
    CU(cudaEventRecord(e->ev1, e->st));
    launches = 1;
  } else {
    double pre_ms = 0;
    rc = prefill(e, n_prompt, &pre_ms, &launches);
    if (rc) return rc;
    out->prefill_ms = pre_ms;
    // end = first decoded index: commit-stream draw of step j is j - end
    ArCtl ctl{n_prompt - 1, e->first_local_layer, e->n_local_layers, n_prompt - 1};
    CU(cudaMemcpyAsync(e->d_arctl, &ctl, sizeof(ctl), cudaMemcpyHostToDevice, e->st));
    CU(cudaEventRecord(e->ev0, e->st));
    NvtxRange nv("ppsd.ar tokens", 1, max_tokens);
    for (int i = 0; i < max_tokens; ++i) CU(cudaGraphLaunch(e->g_ar, e->st));
    CU(cudaEventRecord(e->ev1, e->st));
    launches += (int64_t)max_tokens * e->ar_launches;
  }
  CU(cudaEventSynchronize(e->ev1));
  if (int rc2 = check_kerr(e)) return rc2;
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
  out->decode_ms = ms;
  out->committed_tokens = max_tokens;
  out->ticks = (int64_t)max_tokens * e->S;  // simulate_autoregressive tick model, pipesim.py:386
  out->rejects = max_tokens;
  out->throughput = 1.0 / e->S;
  out->speedup_vs_ar = 1.0;
  out->gpu_launches = launches;
  if (out_tokens)
    CU(cudaMemcpy(out_tokens, e->d_tokens + n_prompt, sizeof(int32_t) * max_tokens, cudaMemcpyDeviceToHost));
  return PPSD_OK;
}

// ---------------------------------------------------------------------------
// EESD draft-then-verify baseline (pipesim.py:435-551)

static int eesd_graph(ppsd_engine* e, int gamma, cudaGraphExec_t* out, int64_t* nlaunch) {
  auto it = e->eesd_graphs.find(gamma);
  if (it != e->eesd_graphs.end()) {
    *out = it->second.first;
    *nlaunch = it->second.second;
    return PPSD_OK;
  }
  const TickCtx* ctx = e->d_ctx;
  EesdState* es = e->d_eesd;
  const int exit_layer = e->cfg.stage_first[e->cfg.k + 1];
  cudaGraphExec_t g = nullptr;
  int64_t n = 0;
  int rc = capture(
      e,
      [&]() -> int {
        int cnt = 0;
        if (e->md.kind != PPSD_MODEL_TRANSFORMER) {
          if (launch_pdl(eesd_toy_round_kernel, dim3(1), dim3(256), 0, e->st, ctx, es) != cudaSuccess) return -1;
          return 1;
        }
        for (int h = 0; h < gamma; ++h) {  // gamma one-token drafts through the exit layers
          if (launch_pdl(eesd_draft_begin_kernel, dim3(1), dim3(256), 0, e->st, ctx, es) != cudaSuccess) return -1;
          const int m = enqueue_layers(e, e->d_work_ar, exit_layer, false);
          if (m < 0) return -1;
          const int mh = e->hl ? enqueue_head_layer(e, false) : 0;  // exit-head layer on a copy
          if (mh < 0) return -1;
          if (enqueue_gemv(e, e->d_work_ar, 0, kMatHead) != cudaSuccess) return -1;
          if (launch_pdl(eesd_draft_end_kernel, dim3(1), dim3(256), 0, e->st, ctx, es) != cudaSuccess) return -1;
          cnt += m + mh + 3;
        }
        if (launch_pdl(eesd_verify_begin_kernel, dim3(1), dim3(256), 0, e->st, ctx, es) != cudaSuccess) return -1;
        const int m = enqueue_layers(e, e->d_work_ar, e->n_local_layers, true);  // batched verify
        if (m < 0) return -1;
        if (enqueue_gemv(e, e->d_work_ar, 0, kMatHeadV, true) != cudaSuccess) return -1;
        if (launch_pdl(eesd_scan_kernel, dim3(1), dim3(256), 0, e->st, ctx, es) != cudaSuccess) return -1;
        return cnt + m + 3;
      },
      &g, &n);
  if (rc) return rc;
  e->eesd_graphs[gamma] = {g, n};
  *out = g;
  *nlaunch = n;
  return PPSD_OK;
}

static int run_eesd(ppsd_engine* e, int model, int gamma, const int32_t* prompt, int n_prompt, int horizon,
                    double alpha, uint64_t verify_seed, int32_t* out_tokens, int32_t out_cap, ppsd_metrics* out,
                    ppsd_trace_row* trace, int64_t trace_cap, int64_t* trace_len) {
  if (e->lo != 1 || e->hi != e->S) return fail(PPSD_EINVAL, "engine holds a stage subset");
  if (gamma < 1) return fail(PPSD_EINVAL, "gamma must be >= 1");
  if (horizon < 1) return fail(PPSD_EINVAL, "horizon must be >= 1");
  if (model && e->md.kind == PPSD_MODEL_TRANSFORMER && gamma + 1 > kMaxVec)
    return fail(PPSD_EUNSUPPORTED, "gamma + 1 must be <= 16 for the batched verify");
  if (model && (int64_t)n_prompt + horizon + gamma + 2 > e->md.max_ctx)
    return fail(PPSD_EINVAL, "prompt + horizon exceeds the engine's max_ctx");
  memset(out, 0, sizeof(*out));
  CU(cudaSetDevice(e->device));
  cudaGraphExec_t g;
  int64_t per_round = 0;
  int rc = eesd_graph(e, gamma, &g, &per_round);
  if (rc) return rc;
  int64_t launches = 0;
  double pre_ms = 0;
  if (model) {
    rc = upload_prompt(e, prompt, n_prompt);
    if (rc) return rc;
    rc = prefill(e, n_prompt, &pre_ms, &launches);
    if (rc) return rc;
  }
  const int rows_per_round = 2 * gamma + e->S + 1;
  int64_t cap = (int64_t)horizon * rows_per_round + 8;
  if (trace) {
    if (trace_cap < cap) cap = trace_cap;
    rc = ensure_trace(e, cap);
    if (rc) return rc;
  }
  EesdState st{};
  st.gamma = gamma;
  st.k = e->cfg.k;
  st.S = e->S;
  st.per = e->cfg.per;
  st.dt = st.k == 1 ? 1 : st.k * st.per;  // pipesim.py:456
  st.n_prompt = n_prompt;
  st.horizon = horizon;
  st.n_layers = e->md.n_layers;
  st.exit_layer = e->cfg.stage_first[st.k + 1];
  st.model = model;
  st.alpha = alpha;
  st.verify_seed = verify_seed;
  st.len = n_prompt;
  e->h_ctx.trace = trace ? e->d_trace : nullptr;
  e->h_ctx.trace_cap = cap;
  e->h_ctx.inbox = nullptr;
  e->h_ctx.outbox = nullptr;
  CU(cudaMemcpyAsync(e->d_ctx, &e->h_ctx, sizeof(TickCtx), cudaMemcpyHostToDevice, e->st));
  CU(cudaMemcpyAsync(e->d_eesd, &st, sizeof(EesdState), cudaMemcpyHostToDevice, e->st));
  CU(cudaEventRecord(e->ev0, e->st));
  int64_t rounds = 0;
  for (;;) {
    const int64_t n = std::max<int64_t>(1, (horizon - st.committed + gamma) / (gamma + 1));
    NvtxRange nv("ppsd.eesd rounds", 1, n);
    for (int64_t i = 0; i < n; ++i) CU(cudaGraphLaunch(g, e->st));
    rounds += n;
    CU(cudaMemcpyAsync(&st, e->d_eesd, sizeof(EesdState), cudaMemcpyDeviceToHost, e->st));
    CU(cudaStreamSynchronize(e->st));
    if (st.error || st.done) break;
    if (rounds > (int64_t)horizon + 4) return fail(PPSD_ESTATE, "EESD rounds did not converge");
  }
  CU(cudaEventRecord(e->ev1, e->st));
  CU(cudaEventSynchronize(e->ev1));
  if (int rc2 = check_kerr(e)) return rc2;
  if (st.error & kErrTrace) return fail(PPSD_ESTATE, "trace buffer too small");
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
  out->committed_tokens = st.committed;
  out->ticks = st.t;
  out->accepts = st.accepts;
  out->rejects = st.rejects;
  out->alpha_valid = st.drafted > 0;
  out->alpha_all_measured = st.drafted > 0 ? (double)st.accepts / st.drafted : 0.0;  // pipesim.py:272
  out->throughput = st.t > 0 ? (double)st.committed / st.t : 0.0;
  out->speedup_vs_ar = out->throughput * (double)(e->S * e->cfg.per);
  out->decode_ms = ms;
  out->prefill_ms = pre_ms;
  out->gpu_launches = launches + rounds * per_round;
  if (out_tokens && model) {
    const int n = std::min<int>(out_cap, st.committed);
    if (n > 0) CU(cudaMemcpy(out_tokens, e->d_tokens + n_prompt, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  }
  if (trace) {
    const int64_t nr = std::min<int64_t>(st.trace_n, cap);
    if (nr > 0) CU(cudaMemcpy(trace, e->d_trace, sizeof(TraceRow) * nr, cudaMemcpyDeviceToHost));
    if (trace_len) *trace_len = nr;
  } else if (trace_len) {
    *trace_len = 0;
  }
  return PPSD_OK;
}

extern "C" int ppsd_decode_eesd_mode(ppsd_engine* e, int32_t gamma, int32_t greedy, uint64_t rng_seed,
                                     const int32_t* prompt, int32_t n_prompt, int32_t horizon, int32_t* out_tokens,
                                     int32_t out_cap, ppsd_metrics* out, ppsd_trace_row* trace, int64_t trace_cap,
                                     int64_t* trace_len) {
  if (!e || !out) return fail(PPSD_EINVAL, "null argument");
  if (e->md.kind == PPSD_MODEL_BERNOULLI) return fail(PPSD_EINVAL, "Bernoulli engines run ppsd_simulate_eesd");
  int rc = check_prompt(e, prompt, n_prompt);
  if (rc) return rc;
  if (!greedy && gamma > std::max(e->cfg.nslot, (int)kMaxVec))
    return fail(PPSD_EUNSUPPORTED, "sampling-mode EESD keeps each draft's distribution: gamma <= " +
                                       std::to_string(std::max(e->cfg.nslot, (int)kMaxVec)));
  CU(cudaSetDevice(e->device));
  rc = set_mode(e, greedy, rng_seed);
  if (rc) return rc;
  return run_eesd(e, 1, gamma, prompt, n_prompt, horizon, 0.0, greedy ? 0 : e->verify_seed, out_tokens, out_cap,
                  out, trace, trace_cap, trace_len);
}

extern "C" int ppsd_decode_eesd(ppsd_engine* e, int32_t gamma, const int32_t* prompt, int32_t n_prompt,
                                int32_t horizon, int32_t* out_tokens, int32_t out_cap, ppsd_metrics* out,
                                ppsd_trace_row* trace, int64_t trace_cap, int64_t* trace_len) {
  return ppsd_decode_eesd_mode(e, gamma, 1, 0, prompt, n_prompt, horizon, out_tokens, out_cap, out, trace,
                               trace_cap, trace_len);
}

extern "C" int ppsd_simulate_eesd(ppsd_engine* e, int32_t gamma, double alpha, uint64_t verify_seed,
                                  int32_t horizon, ppsd_metrics* out, ppsd_trace_row* trace, int64_t trace_cap,
                                  int64_t* trace_len) {
  if (!e || !out) return fail(PPSD_EINVAL, "null argument");
  if (e->md.kind != PPSD_MODEL_BERNOULLI) return fail(PPSD_EINVAL, "ppsd_simulate_eesd needs a Bernoulli engine");
  if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(PPSD_EINVAL, "BERNOULLI oracle needs alpha in [0, 1]");
  return run_eesd(e, 0, gamma, nullptr, 0, horizon, alpha, verify_seed, nullptr, 0, out, trace, trace_cap,
                  trace_len);
}

// ---------------------------------------------------------------------------
// weight init

extern "C" int ppsd_weight_elems(int32_t tiled, int64_t rows, int64_t cols, int64_t* elems) {
  if (rows <= 0 || cols <= 0 || !elems) return fail(PPSD_EINVAL, "bad weight shape");
  if (!tiled) {
    *elems = rows * cols;
    return PPSD_OK;
  }
  if (rows % 8 || cols % 8 || rows > INT32_MAX || cols > INT32_MAX)
    return fail(PPSD_EUNSUPPORTED, "TC-tiled weights need rows and cols multiples of 8");
  int js, kp;
  tc_layout((int)rows, (int)cols, &js, &kp);
  *elems = rows * kp;
  return PPSD_OK;
}

extern "C" int ppsd_tc_offset(int64_t rows, int64_t cols, int64_t r, int64_t k, int64_t* off) {
  if (rows <= 0 || cols <= 0 || rows % 8 || cols % 8 || r < 0 || r >= rows || k < 0 || !off)
    return fail(PPSD_EINVAL, "bad TC-tiled coordinates");
  int js, kp;
  tc_layout((int)rows, (int)cols, &js, &kp);
  if (k >= kp) return fail(PPSD_EINVAL, "bad TC-tiled coordinates");
  *off = tc_offset((int)rows, (int)cols, r, k);
  return PPSD_OK;
}

extern "C" int ppsd_init_weight(void* dst, int32_t layout, int64_t rows, int64_t cols, uint64_t seed,
                                const uint64_t* tids, const float* scales, int32_t n_heads, int32_t n_kv_heads,
                                int32_t head_dim, void* cuda_stream) {
  if (!dst || !tids || !scales || rows <= 0 || cols <= 0) return fail(PPSD_EINVAL, "bad init arguments");
  const bool tiled = (layout & PPSD_LAYOUT_TC_TILED) != 0;
  layout &= ~PPSD_LAYOUT_TC_TILED;
  if (layout < 0 || layout > 2) return fail(PPSD_EINVAL, "bad weight layout");
  int64_t elems = 0;
  if (int rc = ppsd_weight_elems(tiled, rows, cols, &elems)) return rc;
  const uint64_t salt = 0x5EEDB200C0FFEE01ull;  // oracle/transformer.py INIT_SALT
  uint64_t b[3] = {0, 0, 0};
  float a[3] = {0, 0, 0};
  const int nt = layout == 0 ? 1 : (layout == 1 ? 3 : 2);
  for (int i = 0; i < nt; ++i) {
    b[i] = hmix64(hmix64(seed ^ salt) ^ tids[i]);
    a[i] = scales[i];
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(cuda_stream);
  const long long n = elems;
  long long blocks = (n + 255) / 256;
  if (blocks > 148LL * 64) blocks = 148LL * 64;
  init_weight_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<__nv_bfloat16*>(dst), layout, tiled ? 1 : 0,
                                                     rows, cols, b[0], b[1], b[2], a[0], a[1], a[2], n_heads,
                                                     n_kv_heads, head_dim);
  CU(cudaGetLastError());
  return PPSD_OK;
}

// ---------------------------------------------------------------------------
// multi-rank stepping and the kernel probe: implemented in engine_mr.cu

extern "C" int ppsd_probe_gemv(ppsd_engine* e, int32_t which, int32_t n_groups, int32_t reps, double* avg_ms,
                               double* bytes_per_launch) {
  // n_groups > 0: the decode-tick plan (one vector per group, groups = the
  // first n_groups local stages); n_groups < 0: the batched plan with
  // -n_groups vectors in one group (folded deep batch / EESD verify).
  // Consecutive launches walk the stage's layers so no launch re-reads
  // weights the previous one left in L2.
  if (!e || e->md.kind != PPSD_MODEL_TRANSFORMER) return fail(PPSD_EINVAL, "probe needs a transformer engine");
  if (which < 0 || which > kMatHeadV || reps < 1) return fail(PPSD_EINVAL, "bad probe arguments");
  const int G = e->hi - e->lo + 1;
  const bool batched = n_groups < 0;
  const int nv = batched ? -n_groups : 1;
  const int ng = batched ? 1 : n_groups;
  if (ng < 1 || ng > G || ng > e->cfg.nslot || nv > kMaxVec) return fail(PPSD_EINVAL, "bad n_groups");
  if ((which == kMatHeadV) != batched && which >= kMatHead) return fail(PPSD_EINVAL, "head probe: kMatHead per tick, kMatHeadV batched");
  CU(cudaSetDevice(e->device));
  Work w{};
  w.G = ng;
  int nl = 1 << 30;
  for (int g = 0; g < ng; ++g) {
    w.nv[g] = nv;
    w.slot[g] = g;
    w.pos[g] = 0;
    w.first[g] = e->cfg.stage_first[e->lo + g];
    w.nl[g] = e->cfg.stage_layers[e->lo + g];
    nl = std::min(nl, (int)w.nl[g]);
  }
  w.head_slot[0] = 0;
  w.head_slot[1] = ng > 1 ? 1 : -1;
  CU(cudaMemcpyAsync(e->d_work_ar, &w, sizeof(Work), cudaMemcpyHostToDevice, e->st));
  const bool head = which >= kMatHead;
  e->small_batch = batched && nv <= 5;  // as the folded deep batch runs it
  auto launch = [&](int i) { return enqueue_gemv(e, e->d_work_ar, head ? 0 : i % nl, which, batched); };
  for (int i = 0; i < 3; ++i) CU(launch(i));
  CU(cudaEventRecord(e->ev0, e->st));
  for (int i = 0; i < reps; ++i) CU(launch(i));
  CU(cudaEventRecord(e->ev1, e->st));
  e->small_batch = false;
  CU(cudaEventSynchronize(e->ev1));
  if (int rc = check_kerr(e)) return rc;
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
  const GemvPlan& p = batched ? e->gpb[which] : e->gp[which];
  *avg_ms = ms / reps;
  *bytes_per_launch = (double)p.R * p.K * 2.0 * (head ? 1 : ng);
  return PPSD_OK;
}

// GEMV unit check (parity tests): y_v = W x_v for one O or down projection of
// global layer `layer` through the shipped kernel (residual epilogue into a
// zeroed hidden state), nv vectors in one group, decode-tick (batched = 0,
// nv <= 5) or batched plan. in: host [nv][K] fp32, out: host [nv][R] fp32.
extern "C" int ppsd_debug_matvec(ppsd_engine* e, int32_t which, int32_t layer, int32_t nv, int32_t batched,
                                 const float* in, float* out) {
  if (!e || e->md.kind != PPSD_MODEL_TRANSFORMER) return fail(PPSD_EINVAL, "matvec needs a transformer engine");
  if ((which != kMatO && which != kMatDown) || !in || !out) return fail(PPSD_EINVAL, "matvec: O or down only");
  if (nv < 1 || nv > (batched ? (int)kMaxVec : 5) || nv > e->nbuf) return fail(PPSD_EINVAL, "matvec: bad nv");
  if (layer < e->first_local_layer || layer >= e->first_local_layer + e->n_local_layers)
    return fail(PPSD_EINVAL, "matvec: layer not local");
  CU(cudaSetDevice(e->device));
  const GemvPlan& p = batched ? e->gpb[which] : e->gp[which];
  const int K = p.K, R = p.R;
  Work w{};
  w.G = 1;
  w.slot[0] = 0;
  w.pos[0] = 0;
  w.nv[0] = nv;
  w.first[0] = layer;
  w.nl[0] = 1;
  w.head_slot[0] = w.head_slot[1] = -1;
  CU(cudaMemcpyAsync(e->d_work_ar, &w, sizeof(Work), cudaMemcpyHostToDevice, e->st));
  float* dst_in = which == kMatO ? e->d_o : e->d_h;
  const size_t ld_in = which == kMatO ? (size_t)e->dm.H * e->dm.hd : (size_t)e->dm.ffn;
  for (int v = 0; v < nv; ++v)
    CU(cudaMemcpyAsync(dst_in + v * ld_in, in + (size_t)v * K, sizeof(float) * K, cudaMemcpyHostToDevice, e->st));
  CU(cudaMemsetAsync(e->d_x, 0, sizeof(float) * (size_t)nv * e->dm.d, e->st));
  CU(enqueue_gemv(e, e->d_work_ar, 0, which, batched != 0));
  for (int v = 0; v < nv; ++v)
    CU(cudaMemcpyAsync(out + (size_t)v * R, e->d_x + (size_t)v * e->dm.d, sizeof(float) * R, cudaMemcpyDeviceToHost,
                       e->st));
  CU(cudaStreamSynchronize(e->st));
  return check_kerr(e);
}

namespace ppsd {
int tc_trace_enable(int on);
int tc_trace_read(unsigned long long* out);  // [8][128] + [160][4]
int tc_pass_trace_enable(int on);
int tc_pass_trace_read(unsigned long long* out);  // [8][128]
}
// tensor-core GEMV pipeline timeline of CTA 0 (debugging): on = 1 records the
// next launches, out = [8][128] %globaltimer ns of the last one
extern "C" int ppsd_debug_tc_trace(int32_t on, uint64_t* out) {
  // on / out & 2 (bit 1 of on >= 2): the layer pass's trace instead of the GEMV's;
  // on 4 / 5: attention trace off / on, on -4: read it (uint64 [1024][12])
  if (on == 4 || on == 5) return attn_trace_enable(on & 1) ? fail(PPSD_ECUDA, "trace enable") : PPSD_OK;
  if (on == -4) return out && !attn_trace_read(reinterpret_cast<unsigned long long*>(out)) ? PPSD_OK
                                                                                      : fail(PPSD_ECUDA, "trace read");
  const bool pass = on >= 2 || (on < 0 && out && (on & 2));
  if (on >= 0 && (pass ? tc_pass_trace_enable(on & 1) : tc_trace_enable(on))) return fail(PPSD_ECUDA, "trace enable");
  if (out && (on == -2 ? tc_pass_trace_read(reinterpret_cast<unsigned long long*>(out))
                       : tc_trace_read(reinterpret_cast<unsigned long long*>(out))))
    return fail(PPSD_ECUDA, "trace read");
  return PPSD_OK;
}

extern "C" int ppsd_probe_attn(ppsd_engine* e, int32_t n_vec, int32_t ctx, int32_t reps, double* avg_ms,
                               double* bytes_per_launch) {
  // Decode attention of one group of n_vec vectors whose longest context is
  // ctx positions (positions ctx-n_vec .. ctx-1), walking the local layers
  // so consecutive launches read different KV; the kernel the decode graphs
  // use for that vector count (one vector: the cluster kernel unless
  // PPSD_ATTN_CL=0; more: the folded deep batch's clusters of 4 unless
  // PPSD_ATTN_CLB=0, then split-K).
  if (!e || e->md.kind != PPSD_MODEL_TRANSFORMER) return fail(PPSD_EINVAL, "probe needs a transformer engine");
  if (n_vec < 1 || n_vec > kMaxVec || ctx < n_vec || ctx > e->md.max_ctx || reps < 1)
    return fail(PPSD_EINVAL, "bad attention probe arguments");
  CU(cudaSetDevice(e->device));
  Work w{};
  w.G = 1;
  w.slot[0] = 0;
  w.nv[0] = n_vec;
  w.pos[0] = ctx - n_vec;
  w.first[0] = e->first_local_layer;
  w.nl[0] = e->n_local_layers;
  w.head_slot[0] = w.head_slot[1] = -1;
  CU(cudaMemcpyAsync(e->d_work_ar, &w, sizeof(Work), cudaMemcpyHostToDevice, e->st));
  auto launch = [&](int i) { return enqueue_attn(e, e->d_work_ar, i % e->n_local_layers, n_vec > 1); };
  e->attn_clb_vec = n_vec > 1 ? n_vec : 0;  // a bounded batch (folded deep batch kernel)
  struct Reset {
    ppsd_engine* e;
    ~Reset() { e->attn_clb_vec = 0; }
  } reset{e};
  for (int i = 0; i < 3; ++i) CU(launch(i));
  CU(cudaEventRecord(e->ev0, e->st));
  for (int i = 0; i < reps; ++i) CU(launch(i));
  CU(cudaEventRecord(e->ev1, e->st));
  CU(cudaEventSynchronize(e->ev1));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, e->ev0, e->ev1));
  *avg_ms = ms / reps;
  *bytes_per_launch = 2.0 * ctx * e->dm.KV * e->dm.hd * (e->dm.kv_bf16 ? 2 : 4);  // K + V rows read once
  return PPSD_OK;
}

extern "C" int ppsd_set_logits_tap(ppsd_engine* e, float* dev_tap, int32_t max_pos) {
  if (!e || e->md.kind != PPSD_MODEL_TRANSFORMER) return fail(PPSD_EINVAL, "logits tap needs a transformer engine");
  if (dev_tap && max_pos < 1) return fail(PPSD_EINVAL, "max_pos must be >= 1");
  e->h_ctx.tap = dev_tap;
  e->h_ctx.tap_max = dev_tap ? max_pos : 0;
  CU(cudaSetDevice(e->device));
  CU(cudaMemcpyAsync(e->d_ctx, &e->h_ctx, sizeof(TickCtx), cudaMemcpyHostToDevice, e->st));
  CU(cudaStreamSynchronize(e->st));
  return PPSD_OK;
}

extern "C" int ppsd_read_logits(ppsd_engine* e, int32_t which, float* out) {
  if (!e || e->md.kind != PPSD_MODEL_TRANSFORMER || which < 0 || which > 1 || !out)
    return fail(PPSD_EINVAL, "bad read_logits arguments");
  CU(cudaSetDevice(e->device));
  CU(cudaStreamSynchronize(e->st));
  CU(cudaMemcpy(out, e->d_logits + (size_t)which * e->dm.V, sizeof(float) * e->dm.V, cudaMemcpyDeviceToHost));
  return PPSD_OK;
}

// ---------------------------------------------------------------------------
// multi-rank stepping (one engine per GPU); see include/ppsd.h
//
// Per tick: step_compute = [layers of the local stages, local heads, pack
// outbox]; the caller all-gathers every rank's outbox into every inbox
// (NCCL over NVLink); step_finish = [sched_tick: unpack the arriving
// activation + the owners' head results, verdict/draft/rollback, plan].
// Every rank runs the identical scheduler, so ranks agree on every tick
// without any other message.

// Rank-fold tick graph (sched.h: sched_rfold_plan). The scheduler kernel of
// the previous launch (or step) planned the tick; the first kernel opens the
// IF node when the plan has a deferred batch (the handle resets to 0 at every
// launch). p2p: the scheduler kernel for the next tick closes the graph.
static int build_rf_graph(ppsd_engine* e, bool with_sched, cudaGraphExec_t* out, int64_t* n_launches) {
  const SchedCfg& C = e->cfg;
  const int lo = e->lo, hi = e->hi, k = C.k;
  const int eager = lo <= k ? C.stage_first[k] + C.stage_layers[k] - C.stage_first[lo] : 0;
  const int dlo = sched_rfold_first(&C, lo);
  const int deferred = C.stage_first[hi] + C.stage_layers[hi] - C.stage_first[dlo];
  cudaStream_t main_st = e->st, body_st = nullptr;
  CU(cudaStreamCreateWithFlags(&body_st, cudaStreamNonBlocking));
  cudaGraph_t g = nullptr;
  int n_outer = 0, n_body = 0;
  bool ok = true;
  std::string err;
  auto need = [&](bool cond, const char* what) {
    if (!cond && ok) {
      ok = false;
      const cudaError_t le = g_launch_err != cudaSuccess ? g_launch_err : cudaGetLastError();
      err = std::string(what) + ": " + cudaGetErrorString(le);
    }
  };
  g_launch_err = cudaSuccess;
  cudaError_t ce = cudaStreamBeginCapture(main_st, cudaStreamCaptureModeThreadLocal);
  if (ce != cudaSuccess) {
    cudaStreamDestroy(body_st);
    CU(ce);
  }
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaGraph_t cg = nullptr;
  cudaGraphConditionalHandle h = 0;
  need(cudaStreamGetCaptureInfo(main_st, &cs, nullptr, &cg, &deps, &nd) == cudaSuccess, "capture info");
  if (ok) need(cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault) == cudaSuccess,
               "conditional handle");
  if (ok) need(launch_pdl(rf_cond_kernel, dim3(1), dim3(32), 0, main_st, (const TickCtx*)e->d_ctx,
                          (unsigned long long)h) == cudaSuccess, "IF setter");
  n_outer = 1;
  if (ok && eager > 0) {  // the chain reaching stage lo: stages lo..k, exit head
    e->tick_g1 = true;
    const int m = enqueue_layers(e, e->d_work, eager, false);
    e->tick_g1 = false;
    need(m >= 0, "eager layers");
    n_outer += m;
    need(ok && enqueue_gemv(e, e->d_work, 0, kMatHead) == cudaSuccess, "exit head");
    n_outer += 1;
  }
  cudaGraph_t body = nullptr;
  if (ok) {
    need(cudaStreamGetCaptureInfo(main_st, &cs, nullptr, &cg, &deps, &nd) == cudaSuccess, "capture info");
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode = nullptr;
    if (ok) need(cudaGraphAddNode(&cnode, cg, deps, nd, &cp) == cudaSuccess, "conditional node");
    if (ok) body = cp.conditional.phGraph_out[0];
    if (ok) need(cudaStreamUpdateCaptureDependencies(main_st, &cnode, 1, cudaStreamSetCaptureDependencies) ==
                     cudaSuccess, "capture deps");
  }
  if (ok && body) {  // body: gather, deferred layers (batched plans), final heads
    need(cudaStreamBeginCaptureToGraph(body_st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
             cudaSuccess, "body capture");
    if (ok) {
      e->st = body_st;
      need(launch_pdl(rf_gather_kernel, dim3(1), dim3(256), 0, body_st, (const TickCtx*)e->d_ctx) == cudaSuccess,
           "gather");
      n_body = 1;
      e->small_batch = sched_rfold_width(&C, lo, hi) <= 5;
      e->attn_clb_vec = sched_rfold_width(&C, lo, hi);
      const int m = enqueue_layers(e, e->d_work_deep, deferred, true);
      e->attn_clb_vec = 0;
      need(m >= 0, "deferred layers");
      n_body += m;
      if (ok && hi == e->S) {
        need(enqueue_gemv(e, e->d_work_deep, 0, kMatHeadV, true, e->d_logits + e->dm.V) == cudaSuccess,
             "final heads");
        n_body += 1;
      }
      e->small_batch = false;
      e->st = main_st;
      cudaGraph_t bg = body;
      need(cudaStreamEndCapture(body_st, &bg) == cudaSuccess, "body end capture");
    }
  }
  // after the IF node: plain launches (a programmatic edge needs a kernel predecessor)
  if (ok) {
    pack_outbox_kernel<<<1, 256, 0, main_st>>>((const TickCtx*)e->d_ctx, 0);
    need(cudaGetLastError() == cudaSuccess, "pack");
    n_outer += 1;
  }
  if (ok && with_sched) {
    need(launch_pdl(sched_tick_kernel, dim3(1), dim3(256), 0, main_st, (const TickCtx*)e->d_ctx, 0) ==
             cudaSuccess, "scheduler");
    n_outer += 1;
  }
  e->st = main_st;
  ce = cudaStreamEndCapture(main_st, &g);
  cudaStreamDestroy(body_st);
  if (!ok) {
    if (g) cudaGraphDestroy(g);
    return fail(PPSD_ECUDA, "rank-fold tick graph: " + err);
  }
  CU(ce);
  ce = cudaGraphInstantiate(out, g, 0);
  cudaGraphDestroy(g);
  CU(ce);
  *n_launches = n_outer;
  e->rf_body_launches = n_body;
  return PPSD_OK;
}

static int build_mr_graphs(ppsd_engine* e) {
  if (e->g_compute) return PPSD_OK;
  int rc = capture(
      e,
      [&]() -> int {
        int m = enqueue_layers(e, e->d_work, e->max_local_layers, false);
        if (m < 0) return -1;
        if (e->hl) {  // exit rank: head layer on a copy of the exit chain's state
          const int mh = enqueue_head_layer(e, false);
          if (mh < 0) return -1;
          m += mh;
        }
        if (enqueue_gemv(e, e->d_work, 0, kMatHead) != cudaSuccess) return -1;
        if (launch_pdl(pack_outbox_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx, 0) !=
            cudaSuccess)
          return -1;
        return m + 2;
      },
      &e->g_compute, &e->compute_launches);
  if (rc) return rc;
  rc = capture(
      e,
      [&]() -> int {
        if (launch_pdl(sched_tick_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx, 0) !=
            cudaSuccess)
          return -1;
        return 1;
      },
      &e->g_finish, &e->finish_launches);
  if (rc) return rc;
  return capture(
      e,
      [&]() -> int {
        if (launch_pdl(mr_prefill_begin_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx,
                       e->d_arctl) != cudaSuccess)
          return -1;
        int m;
        if (e->hl) {  // [0, split), head layer on a copy, [split, local end)
          const int split = e->h_ctx.hl_split;
          m = enqueue_prefill_layers(e, e->d_work_ar, split);
          if (m < 0) return -1;
          const int mh = enqueue_head_layer(e, true);
          if (mh < 0) return -1;
          const int m2 = enqueue_prefill_layers(e, e->d_work_p2, e->n_local_layers - split);
          if (m2 < 0) return -1;
          m += mh + m2;
        } else {
          m = enqueue_prefill_layers(e, e->d_work_ar, e->n_local_layers);
          if (m < 0) return -1;
        }
        if (launch_pdl(pack_outbox_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx, 1) !=
            cudaSuccess)
          return -1;
        return m + 2;
      },
      &e->g_mr_prefill, &e->mr_prefill_launches);
}

extern "C" int ppsd_exchange_info(ppsd_engine* e, int64_t* outbox_bytes, void** cuda_stream) {
  if (!e || e->md.kind != PPSD_MODEL_TRANSFORMER) return fail(PPSD_EINVAL, "multi-rank needs a transformer engine");
  if (outbox_bytes) *outbox_bytes = (int64_t)(kBoxHeader + e->dm.d) * 4;
  if (cuda_stream) *cuda_stream = e->st;
  return PPSD_OK;
}

extern "C" int ppsd_step_mode(ppsd_engine* e, int32_t greedy, uint64_t rng_seed) {
  if (!e || e->md.kind != PPSD_MODEL_TRANSFORMER) return fail(PPSD_EINVAL, "multi-rank needs a transformer engine");
  e->mr_greedy = greedy ? 1 : 0;
  e->mr_rng_seed = rng_seed;
  return PPSD_OK;
}

extern "C" int ppsd_step_begin(ppsd_engine* e, const int32_t* prompt, int32_t n_prompt, int32_t max_tokens,
                               int32_t force_reject, const int32_t* stage_owner, int32_t world, int32_t rank,
                               void* outbox, void* inbox) {
  if (!e || e->md.kind != PPSD_MODEL_TRANSFORMER) return fail(PPSD_EINVAL, "multi-rank needs a transformer engine");
  if (!stage_owner || world < 1 || rank < 0 || rank >= world || !outbox || !inbox)
    return fail(PPSD_EINVAL, "bad multi-rank arguments");
  for (int st = e->lo; st <= e->hi; ++st)
    if (stage_owner[st] != rank) return fail(PPSD_EINVAL, "stage_owner disagrees with the engine's stage range");
  int rc = check_prompt(e, prompt, n_prompt);
  if (rc) return rc;
  if (max_tokens < 1) return fail(PPSD_EINVAL, "max_tokens must be >= 1 for stepping");
  if ((int64_t)n_prompt + max_tokens + (int64_t)e->S * e->cfg.per + 2 > e->md.max_ctx)
    return fail(PPSD_EINVAL, "prompt + max_tokens exceeds the engine's max_ctx");
  CU(cudaSetDevice(e->device));
  rc = build_mr_graphs(e);
  if (rc) return rc;
  rc = upload_prompt(e, prompt, n_prompt);
  if (rc) return rc;
  const int64_t max_ticks = (int64_t)max_tokens * e->S * e->cfg.per + (int64_t)e->S * e->cfg.per + 8;
  rc = ensure_trace(e, max_ticks * (e->S + 2));
  if (rc) return rc;
  TickCtx& c = e->h_ctx;
  c.fold = 0;
  c.trace = e->d_trace;
  c.trace_cap = e->trace_cap;
  c.outbox = reinterpret_cast<float*>(outbox);
  c.inbox = reinterpret_cast<const float*>(inbox);
  c.box_words = kBoxHeader + e->dm.d;
  c.greedy = e->mr_greedy;
  c.box_logits = e->mr_greedy ? 0 : 1;
  if (!e->mr_greedy) {
    c.box_words += 2 * e->dm.V;
    c.draft_seed = derive_seed_str(e->mr_rng_seed, "draft");
    c.commit_seed = derive_seed_str(e->mr_rng_seed, "commit");
  }
  c.box_used = c.box_words;
  c.rank = rank;
  c.world = world;
  c.owner_k = stage_owner[e->cfg.k];
  c.owner_S = stage_owner[e->S];
  c.owner_prev = e->lo > 1 ? stage_owner[e->lo - 1] : -1;
  c.n_prompt = n_prompt;
  // greedy decodes fold this rank's stages where they can (ppsd_get_schedule)
  e->mr_rf = e->rfold_ok && e->mr_greedy && e->schedule != PPSD_SCHEDULE_PIPELINED;
  if (e->mr_rf && !e->g_compute_rf) {
    rc = build_rf_graph(e, false, &e->g_compute_rf, &e->compute_rf_launches);
    if (rc) return rc;
  }
  c.rfold = e->mr_rf ? 1 : 0;
  c.has_cond = 0;
  Sched& s = *e->h_sched;
  memset(&s, 0, sizeof(Sched));
  s.c = e->cfg;
  s.c.fold = 0;  // the single-device fold needs every stage; ranks fold their own range (rfold)
  s.c.rfold = e->mr_rf ? 1 : 0;
  s.c.rf_lo = e->lo;
  s.c.rf_hi = e->hi;
  s.c.model = 1;
  s.c.force_reject = force_reject;
  s.c.stop = max_tokens;
  s.c.n_prompt = n_prompt;
  s.c.verify_seed = e->mr_greedy ? 0 : derive_seed_str(e->mr_rng_seed, "verify");
  sched_reset(&s);
  ArCtl ctl{0, e->first_local_layer, e->n_local_layers, 0};
  CU(cudaMemcpyAsync(e->d_arctl, &ctl, sizeof(ctl), cudaMemcpyHostToDevice, e->st));
  CU(cudaMemcpyAsync(e->d_ctx, &c, sizeof(TickCtx), cudaMemcpyHostToDevice, e->st));
  CU(cudaMemcpyAsync(e->d_sched, &s, sizeof(Sched), cudaMemcpyHostToDevice, e->st));
  sched_tick_kernel<<<1, 256, 0, e->st>>>(e->d_ctx, 1);  // plan tick 1 (+ embed on rank 0)
  CU(cudaGetLastError());
  e->mr_world = world;
  e->mr_rank = rank;
  e->mr_stop = max_tokens;
  e->mr_n_prompt = n_prompt;
  e->mr_launches = 1;
  e->mr_ticks_launched = 0;
  CU(cudaEventRecord(e->ev0, e->st));
  return PPSD_OK;
}

extern "C" int ppsd_prefill_steps(ppsd_engine* e, int32_t* n_steps) {
  if (!e || !n_steps) return fail(PPSD_EINVAL, "null argument");
  *n_steps = e->mr_n_prompt >= 2 ? (e->mr_n_prompt - 1) + (e->mr_world - 1) : 0;
  return PPSD_OK;
}

extern "C" int ppsd_prefill_compute(ppsd_engine* e) {
  if (!e || !e->g_mr_prefill) return fail(PPSD_ESTATE, "call ppsd_step_begin first");
  CU(cudaGraphLaunch(e->g_mr_prefill, e->st));
  e->mr_launches += e->mr_prefill_launches;
  return PPSD_OK;
}

extern "C" int ppsd_step_compute(ppsd_engine* e) {
  if (!e || !e->g_compute) return fail(PPSD_ESTATE, "call ppsd_step_begin first");
  if (e->mr_ticks_launched == 0) CU(cudaEventRecord(e->ev2, e->st));  // decode starts (prefill done)
  CU(cudaGraphLaunch(e->mr_rf ? e->g_compute_rf : e->g_compute, e->st));
  e->mr_launches += e->mr_rf ? e->compute_rf_launches : e->compute_launches;
  return PPSD_OK;
}

extern "C" int ppsd_step_finish(ppsd_engine* e) {
  if (!e || !e->g_finish) return fail(PPSD_ESTATE, "call ppsd_step_begin first");
  CU(cudaGraphLaunch(e->g_finish, e->st));
  e->mr_launches += e->finish_launches;
  e->mr_ticks_launched += 1;
  return PPSD_OK;
}

extern "C" int ppsd_step_poll(ppsd_engine* e, int32_t* done, int64_t* committed, int64_t* ticks) {
  if (!e) return fail(PPSD_EINVAL, "null argument");
  Sched& s = *e->h_sched;
  const size_t off = offsetof(Sched, t);
  const size_t len = offsetof(Sched, verify_counter) - off;
  CU(cudaMemcpyAsync(reinterpret_cast<char*>(&s) + off, reinterpret_cast<char*>(e->d_sched) + off, len,
                     cudaMemcpyDeviceToHost, e->st));
  CU(cudaStreamSynchronize(e->st));
  if (s.error) return fail(PPSD_ESTATE, "scheduler error flags " + std::to_string(s.error));
  if (done) *done = s.done;
  if (committed) *committed = s.committed;
  if (ticks) *ticks = s.t;
  return PPSD_OK;
}

extern "C" int ppsd_step_end(ppsd_engine* e, int32_t* out_tokens, ppsd_metrics* out, ppsd_trace_row* trace,
                             int64_t trace_cap, int64_t* trace_len) {
  if (!e || !out) return fail(PPSD_EINVAL, "null argument");
  CU(cudaEventRecord(e->ev1, e->st));
  Sched& s = *e->h_sched;
  CU(cudaMemcpyAsync(&s, e->d_sched, sizeof(Sched), cudaMemcpyDeviceToHost, e->st));
  CU(cudaStreamSynchronize(e->st));
  if (!s.done) return fail(PPSD_ESTATE, "decode not finished");
  if (s.error) return fail(PPSD_ESTATE, "scheduler error flags " + std::to_string(s.error));
  float ms = 0, pre = 0;
  CU(cudaEventElapsedTime(&ms, e->ev2, e->ev1));
  CU(cudaEventElapsedTime(&pre, e->ev0, e->ev2));
  memset(out, 0, sizeof(*out));
  fill_metrics(e, s, out);
  out->decode_ms = ms;    // decode ticks on this rank's stream (CUDA events)
  out->prefill_ms = pre;  // pipelined prefill steps
  out->gpu_launches = e->mr_launches + (e->mr_rf ? (int64_t)s.fold_batches * e->rf_body_launches : 0);
  out->schedule = e->mr_rf ? PPSD_SCHEDULE_FOLDED : PPSD_SCHEDULE_PIPELINED;
  if (e->mr_rf) {  // this rank's deferred batches (sched_rfold_plan)
    out->deep_batches = s.fold_batches;
    out->deep_vectors = s.fold_vectors;
    out->deep_pos_sum = s.fold_pos_sum;
  }
  if (out_tokens)
    CU(cudaMemcpy(out_tokens, e->d_tokens + e->mr_n_prompt, sizeof(int32_t) * e->mr_stop, cudaMemcpyDeviceToHost));
  if (trace) {
    const int64_t n = std::min<int64_t>(s.trace_n, trace_cap);
    if (n > 0) CU(cudaMemcpy(trace, e->d_trace, sizeof(TraceRow) * n, cudaMemcpyDeviceToHost));
    if (trace_len) *trace_len = n;
  } else if (trace_len) {
    *trace_len = 0;
  }
  e->h_ctx.inbox = nullptr;
  e->h_ctx.outbox = nullptr;
  CU(cudaMemcpy(e->d_ctx, &e->h_ctx, sizeof(TickCtx), cudaMemcpyHostToDevice));
  return PPSD_OK;
}

// ---------------------------------------------------------------------------
// NVLink peer-store transport (p2p.cuh): no host work per tick — a whole tick
// (local stages, local heads, box peer-stores + release flags, acquire-wait,
// replicated scheduler) is one graph, launched back to back like single-GPU.

// pinned staging: [TickCtx][ArCtl][prompt int32 x max_ctx][xerr int32]
static size_t p2p_pin_bytes(const ppsd_engine* e) {
  return sizeof(TickCtx) + sizeof(ArCtl) + sizeof(int32_t) * ((size_t)e->md.max_ctx + 1);
}

extern "C" int ppsd_p2p_prepare(ppsd_engine* e, int32_t world, void* ipc_handle, void** xbuf) {
  if (!e || e->md.kind != PPSD_MODEL_TRANSFORMER) return fail(PPSD_EINVAL, "p2p needs a transformer engine");
  if (world < 1 || world > e->S) return fail(PPSD_EINVAL, "bad world size");
  CU(cudaSetDevice(e->device));
  const int box = kBoxHeader + e->dm.d + 2 * e->dm.V;  // stride: room for sampling's logits
  if (!e->d_xbuf || e->p2p_world != world) {
    if (e->d_xbuf) CU(cudaFree(e->d_xbuf));
    size_t bytes = sizeof(float) * 2 * (size_t)world * box + sizeof(uint64_t) * world;
#ifdef PPSD_P2P_DEBUG
    bytes += sizeof(uint64_t) * (1 + 500 * 8);
#endif
    CU(dalloc(&e->d_xbuf, bytes));  // flags start at 0; exchange numbers start at 1
    e->p2p_world = world;
  }
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, e->d_xbuf));
    memcpy(ipc_handle, &h, sizeof(h));
  }
  if (xbuf) *xbuf = e->d_xbuf;
  return PPSD_OK;
}

extern "C" int ppsd_p2p_connect(ppsd_engine* e, int32_t rank, const void* ipc_handles, void* const* local_xbufs,
                                const int32_t* stage_owner) {
  if (!e || !e->d_xbuf) return fail(PPSD_ESTATE, "call ppsd_p2p_prepare first");
  const int world = e->p2p_world;
  if (rank < 0 || rank >= world || !stage_owner || (!ipc_handles && !local_xbufs))
    return fail(PPSD_EINVAL, "bad p2p_connect arguments");
  for (int st = e->lo; st <= e->hi; ++st)
    if (stage_owner[st] != rank) return fail(PPSD_EINVAL, "stage_owner disagrees with the engine's stage range");
  CU(cudaSetDevice(e->device));
  std::vector<float*> peers(world);
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      peers[r] = e->d_xbuf;
    } else if (local_xbufs) {
      peers[r] = reinterpret_cast<float*>(local_xbufs[r]);
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, static_cast<const char*>(ipc_handles) + r * sizeof(h), sizeof(h));
      void* p = nullptr;
      CU(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      e->ipc_opened.push_back(p);
      peers[r] = reinterpret_cast<float*>(p);
    }
  }
  if (!e->d_peer_xbuf) CU(dalloc(&e->d_peer_xbuf, sizeof(float*) * kMaxStages));
  CU(cudaMemcpy(e->d_peer_xbuf, peers.data(), sizeof(float*) * world, cudaMemcpyHostToDevice));
  if (!e->d_p2p_outbox) CU(dalloc(&e->d_p2p_outbox, sizeof(float) * (kBoxHeader + e->dm.d + 2 * e->dm.V)));
  if (!e->d_xcount) CU(dalloc(&e->d_xcount, sizeof(uint64_t)));
  if (!e->d_xerr) CU(dalloc(&e->d_xerr, sizeof(int32_t)));
  {  // everything a decode up to max_ctx can need, allocated now
    const int64_t max_ticks = (int64_t)e->md.max_ctx * e->S * e->cfg.per + (int64_t)e->S * e->cfg.per + 8;
    int rc0 = ensure_trace(e, max_ticks * (e->S + 2));
    if (rc0) return rc0;
    if (!e->h_p2p_pin) {
      const size_t pin = p2p_pin_bytes(e);
      CU(cudaMallocHost(reinterpret_cast<void**>(&e->h_p2p_pin), pin));
      e->h_p2p_out = reinterpret_cast<int32_t*>(e->h_p2p_pin + pin) - 1;  // xerr word
    }
  }
  TickCtx& c = e->h_ctx;
  c.fold = 0;
  c.p2p = 1;
  c.peer_xbuf = e->d_peer_xbuf;
  c.my_xbuf = e->d_xbuf;
  c.xcount = e->d_xcount;
  c.xerr = e->d_xerr;
  c.outbox = e->d_p2p_outbox;
  c.inbox = nullptr;
  c.box_words = kBoxHeader + e->dm.d + 2 * e->dm.V;
  c.box_used = kBoxHeader + e->dm.d;
  c.rank = rank;
  c.world = world;
  c.owner_k = stage_owner[e->cfg.k];
  c.owner_S = stage_owner[e->S];
  c.owner_prev = e->lo > 1 ? stage_owner[e->lo - 1] : -1;
  CU(cudaMemcpy(e->d_ctx, &c, sizeof(TickCtx), cudaMemcpyHostToDevice));
  // Load every kernel a decode launches outside a graph now: with lazy module
  // loading the first launch of a kernel waits for the device to drain, which
  // never happens while a peer engine on the same device spins on our flags.
  cudaFuncAttributes fa;
  CU(cudaFuncGetAttributes(&fa, sched_tick_kernel));
  CU(cudaFuncGetAttributes(&fa, p2p_wait_kernel));
  int rc = build_mr_graphs(e);
  if (rc) return rc;
  if (!e->g_p2p_tick) {
    rc = capture(
        e,
        [&]() -> int {
          int m = enqueue_layers(e, e->d_work, e->max_local_layers, false);
          if (m < 0) return -1;
          if (e->hl) {
            const int mh = enqueue_head_layer(e, false);
            if (mh < 0) return -1;
            m += mh;
          }
          if (enqueue_gemv(e, e->d_work, 0, kMatHead) != cudaSuccess) return -1;
          if (launch_pdl(pack_outbox_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx, 0) !=
              cudaSuccess)
            return -1;
          if (launch_pdl(sched_tick_kernel, dim3(1), dim3(256), 0, e->st, (const TickCtx*)e->d_ctx, 0) !=
              cudaSuccess)
            return -1;
          return m + 3;
        },
        &e->g_p2p_tick, &e->p2p_tick_launches);
    if (rc) return rc;
  }
  if (e->rfold_ok && !e->g_p2p_tick_rf) {
    CU(cudaFuncGetAttributes(&fa, rf_cond_kernel));
    CU(cudaFuncGetAttributes(&fa, rf_gather_kernel));
    rc = build_rf_graph(e, true, &e->g_p2p_tick_rf, &e->p2p_tick_rf_launches);
    if (rc) return rc;
  }
  return PPSD_OK;
}

extern "C" int ppsd_p2p_decode(ppsd_engine* e, const int32_t* prompt, int32_t n_prompt, int32_t max_tokens,
                               int32_t force_reject, int32_t* out_tokens, ppsd_metrics* out, ppsd_trace_row* trace,
                               int64_t trace_cap, int64_t* trace_len) {
  if (!e || !e->g_p2p_tick) return fail(PPSD_ESTATE, "call ppsd_p2p_connect first");
  int rc = check_prompt(e, prompt, n_prompt);
  if (rc) return rc;
  if (max_tokens < 1) return fail(PPSD_EINVAL, "max_tokens must be >= 1");
  if ((int64_t)n_prompt + max_tokens + (int64_t)e->S * e->cfg.per + 2 > e->md.max_ctx)
    return fail(PPSD_EINVAL, "prompt + max_tokens exceeds the engine's max_ctx");
  CU(cudaSetDevice(e->device));
  // No allocation and no pageable copy from here on (see h_p2p_pin): with
  // several engines on one device either can wait for a peer's spinning wait.
  const int64_t max_ticks = (int64_t)max_tokens * e->S * e->cfg.per + (int64_t)e->S * e->cfg.per + 8;
  if (max_ticks * (e->S + 2) > e->trace_cap) return fail(PPSD_ESTATE, "p2p trace reservation too small");
  TickCtx& c = e->h_ctx;
  e->mr_rf = e->rfold_ok && e->mr_greedy && e->schedule != PPSD_SCHEDULE_PIPELINED && e->g_p2p_tick_rf;
  c.fold = 0;
  c.rfold = e->mr_rf ? 1 : 0;
  c.has_cond = 0;
  c.trace = e->d_trace;
  c.trace_cap = e->trace_cap;
  c.n_prompt = n_prompt;
  c.greedy = e->mr_greedy;
  c.box_logits = e->mr_greedy ? 0 : 1;
  c.box_used = kBoxHeader + e->dm.d + (e->mr_greedy ? 0 : 2 * e->dm.V);
  if (!e->mr_greedy) {
    c.draft_seed = derive_seed_str(e->mr_rng_seed, "draft");
    c.commit_seed = derive_seed_str(e->mr_rng_seed, "commit");
  }
  Sched& s = *e->h_sched;
  memset(&s, 0, sizeof(Sched));
  s.c = e->cfg;
  s.c.fold = 0;
  s.c.rfold = e->mr_rf ? 1 : 0;
  s.c.rf_lo = e->lo;
  s.c.rf_hi = e->hi;
  s.c.model = 1;
  s.c.force_reject = force_reject;
  s.c.stop = max_tokens;
  s.c.n_prompt = n_prompt;
  s.c.verify_seed = e->mr_greedy ? 0 : derive_seed_str(e->mr_rng_seed, "verify");
  sched_reset(&s);
  char* pin = e->h_p2p_pin;
  TickCtx* pin_ctx = reinterpret_cast<TickCtx*>(pin);
  ArCtl* pin_ctl = reinterpret_cast<ArCtl*>(pin + sizeof(TickCtx));
  int32_t* pin_prompt = reinterpret_cast<int32_t*>(pin + sizeof(TickCtx) + sizeof(ArCtl));
  *pin_ctx = c;
  *pin_ctl = ArCtl{0, e->first_local_layer, e->n_local_layers, 0};
  memcpy(pin_prompt, prompt, sizeof(int32_t) * n_prompt);
  CU(cudaMemcpyAsync(e->d_tokens, pin_prompt, sizeof(int32_t) * n_prompt, cudaMemcpyHostToDevice, e->st));
  CU(cudaMemcpyAsync(e->d_arctl, pin_ctl, sizeof(ArCtl), cudaMemcpyHostToDevice, e->st));
  CU(cudaMemcpyAsync(e->d_ctx, pin_ctx, sizeof(TickCtx), cudaMemcpyHostToDevice, e->st));
  CU(cudaMemcpyAsync(e->d_sched, &s, sizeof(Sched), cudaMemcpyHostToDevice, e->st));
  sched_tick_kernel<<<1, 256, 0, e->st>>>(e->d_ctx, 1);  // plan tick 1 (+ embed on rank 0)
  CU(cudaGetLastError());
  int64_t launches = 1;
  CU(cudaEventRecord(e->ev0, e->st));
  const int steps = n_prompt >= 2 ? (n_prompt - 1) + (e->p2p_world - 1) : 0;  // pipelined prefill
  for (int i = 0; i < steps; ++i) CU(cudaGraphLaunch(e->g_mr_prefill, e->st));
  launches += (int64_t)steps * e->mr_prefill_launches;
  if (steps > 0) {
    p2p_wait_kernel<<<1, 32, 0, e->st>>>(e->d_ctx);
    CU(cudaGetLastError());
    launches += 1;
  }
  CU(cudaEventRecord(e->ev2, e->st));
  int64_t ticks_launched = 0;
  const size_t off = offsetof(Sched, t);
  const size_t len = offsetof(Sched, verify_counter) - off;
  for (;;) {  // replicated state: every rank launches the same number of ticks
    const int64_t n = std::max<int64_t>(1, (int64_t)max_tokens - s.committed);
    NvtxRange nv("ppsd.p2p ticks", 1, n);
    cudaGraphExec_t tick = e->mr_rf ? e->g_p2p_tick_rf : e->g_p2p_tick;
    for (int64_t i = 0; i < n; ++i) CU(cudaGraphLaunch(tick, e->st));
    ticks_launched += n;
    CU(cudaMemcpyAsync(reinterpret_cast<char*>(&s) + off, reinterpret_cast<char*>(e->d_sched) + off, len,
                       cudaMemcpyDeviceToHost, e->st));
    CU(cudaStreamSynchronize(e->st));
    if (s.error || s.done) break;
    if (ticks_launched > max_ticks + 4) return fail(PPSD_ESTATE, "tick machine did not converge");
  }
  CU(cudaEventRecord(e->ev1, e->st));
  CU(cudaMemcpyAsync(&s, e->d_sched, sizeof(Sched), cudaMemcpyDeviceToHost, e->st));
  CU(cudaMemcpyAsync(e->h_p2p_out, e->d_xerr, sizeof(int32_t), cudaMemcpyDeviceToHost, e->st));
  CU(cudaStreamSynchronize(e->st));
  const int32_t xerr = *e->h_p2p_out;
  if (s.error && !xerr) return fail(PPSD_ESTATE, "scheduler error flags " + std::to_string(s.error));
  float ms = 0, pre = 0;
  CU(cudaEventElapsedTime(&ms, e->ev2, e->ev1));
  CU(cudaEventElapsedTime(&pre, e->ev0, e->ev2));
  memset(out, 0, sizeof(*out));
  fill_metrics(e, s, out);
  out->decode_ms = ms;
  out->prefill_ms = pre;
  out->gpu_launches = launches + ticks_launched * (e->mr_rf ? e->p2p_tick_rf_launches : e->p2p_tick_launches) +
                      (e->mr_rf ? (int64_t)s.fold_batches * e->rf_body_launches : 0);
  out->schedule = e->mr_rf ? PPSD_SCHEDULE_FOLDED : PPSD_SCHEDULE_PIPELINED;
  if (e->mr_rf) {
    out->deep_batches = s.fold_batches;
    out->deep_vectors = s.fold_vectors;
    out->deep_pos_sum = s.fold_pos_sum;
  }
  if (out_tokens) CU(cudaMemcpy(out_tokens, e->d_tokens + n_prompt, sizeof(int32_t) * max_tokens, cudaMemcpyDeviceToHost));
  if (trace) {
    const int64_t nr = std::min<int64_t>(s.trace_n, trace_cap);
    if (nr > 0) CU(cudaMemcpy(trace, e->d_trace, sizeof(TraceRow) * nr, cudaMemcpyDeviceToHost));
    if (trace_len) *trace_len = nr;
  } else if (trace_len) {
    *trace_len = 0;
  }
  // outputs are filled either way so a failed exchange can be inspected
  if (xerr) return fail(PPSD_ECUDA, "p2p exchange timed out waiting for a peer rank");
  return PPSD_OK;
}
