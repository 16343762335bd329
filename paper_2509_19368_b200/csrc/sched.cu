// sched.cu — the device-resident tick machine and the per-tick bookkeeping
// kernels. One CTA: the scheduler state (~14 KB) is staged into shared memory
// by all threads, thread 0 runs sched_finish(t) + sched_plan(t+1) from
// sched.h, the local work descriptor is written for the layer kernels, and
// the chain launched at stage 1 gets its input (embedding row / ToyLM prefix
// digest). No host round trip per tick: the host only enqueues tick graphs.
#include "engine_dev.cuh"
#include "p2p.cuh"
#include "sample.cuh"

namespace ppsd {

// Exit-head layer (md.exit_head_layer): one decoder layer (global index
// c.hl_layer, its own KV) run on copies of rows [src, src + nv) placed at
// c.head_row; src < 0 plans no work. Thread 0 only.
__device__ void plan_head_layer(const TickCtx& c, Work* wh, int src, int pos, int nv) {
  wh->G = 1;
  wh->slot[0] = src >= 0 ? c.head_row : -1;
  wh->src_slot = src;
  wh->pos[0] = src >= 0 ? pos : 0;
  wh->first[0] = c.hl_layer;
  wh->nl[0] = 1;
  wh->nv[0] = nv;
  wh->head_slot[0] = wh->head_slot[1] = -1;
}

// Prefill with the exit-head layer: w runs layers [first, first + split),
// the head layer runs on copies of its rows, w2 runs the rest. Thread 0 only.
__device__ void split_prefill(const TickCtx& c, const ArCtl* ctl, Work* w, bool active, int pos, int nv) {
  w->nl[0] = c.hl_split;
  plan_head_layer(c, c.work_head_pf, active ? 0 : -1, pos, nv);
  Work* w2 = c.work_p2;
  *w2 = *w;
  w2->first[0] = ctl->first_layer + c.hl_split;
  w2->nl[0] = ctl->n_layers - c.hl_split;
}

// Sampling mode, run by the whole block before sched_finish (pipesim.py:346-365):
// the draft for this tick's exit chain is drawn from p = softmax(exit logits)
// (p kept per chain for its verdict), and the verdict for the chain at stage S
// runs accept_draft / the residual resample against q = softmax(final logits).
__device__ void sampling_tick(const TickCtx& c, Sched& s, int* exit_tok, int* final_ok, int* final_tok) {
  const int V = c.vocab;
  const bool exact = V <= kExactVocab;
  const double* l64 = c.logits64;
  const float* l32 = c.logits32;
  if (s.final_slot >= 0) {  // verdict first: its draws do not interleave with the draft stream
    // folded: the final logits of the deep batch sit in rows 1.. (position order)
    const float* q32 = !l32 ? nullptr
                       : c.fold ? l32 + (size_t)(1 + s.ch_pos[s.final_slot] - s.fold_base) * V
                                : l32 + V;
    block_softmax(l64 ? l64 + V : nullptr, q32, V, c.qbuf, exact);
    const double* p = c.pdist + (size_t)s.final_slot * V;
    const int d = s.ch_tok[s.final_slot];
    __shared__ int s_ok;
    __shared__ double s_u;
    if (threadIdx.x == 0) {
      if (s.c.force_reject) {
        s_ok = 0;  // full_model_token: sample q with the commit stream
        s_u = counter_uniform(c.commit_seed, s.commit_counter++);
      } else {
        const double r = counter_uniform(s.c.verify_seed, s.verify_counter++);
        const double pt = p[d], qt = c.qbuf[d];
        s_ok = (qt != 0.0) && r <= fmin(1.0, __ddiv_rn(qt, pt));  // speccore.py:90-101
        if (!s_ok) s_u = counter_uniform(c.commit_seed, s.commit_counter++);
      }
    }
    __syncthreads();
    const int ok = s_ok;
    int tok = d;
    if (!ok) {
      const double* dist = c.qbuf;
      if (!s.c.force_reject) {  // residual max(q - p, 0) / Z (speccore.py:104-113)
        for (int i = threadIdx.x; i < V; i += blockDim.x) c.wbuf[i] = fmax(__dsub_rn(c.qbuf[i], p[i]), 0.0);
        __syncthreads();
        const double z = block_sum(c.wbuf, V, exact);
        if (z <= 1e-12 && threadIdx.x == 0) s.error |= kErrResidual;
        for (int i = threadIdx.x; i < V; i += blockDim.x) c.wbuf[i] = __ddiv_rn(c.wbuf[i], z);
        __syncthreads();
        dist = c.wbuf;
      }
      tok = block_sample(dist, V, s_u, exact);
    }
    *final_ok = ok;
    *final_tok = tok;
  }
  if (s.exit_slot >= 0) {  // the draft: sample_token(p, draft_stream)
    double* p = c.pdist + (size_t)s.exit_slot * V;
    block_softmax(l64, l32, V, p, exact);
    __shared__ double s_ud;
    if (threadIdx.x == 0) s_ud = counter_uniform(c.draft_seed, s.draft_counter++);
    __syncthreads();
    *exit_tok = block_sample(p, V, s_ud, exact);
  }
}

// block copy with all loads of a thread issued before its stores (one
// memory round trip instead of a dependent chain per element)
__device__ void copy_words(void* dst, const void* src, int bytes) {
  const int n16 = bytes / 16;
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  constexpr int U = 4;
  for (int base = 0; base < n16; base += U * blockDim.x) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * blockDim.x + threadIdx.x;
      if (i < n16) v[u] = s[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * blockDim.x + threadIdx.x;
      if (i < n16) d[i] = v[u];
    }
  }
  const int tail = bytes - n16 * 16;  // Sched is 4-byte aligned
  if ((int)threadIdx.x < tail / 4)
    reinterpret_cast<int*>(dst)[n16 * 4 + threadIdx.x] = reinterpret_cast<const int*>(src)[n16 * 4 + threadIdx.x];
}

__device__ void embed_row(const TickCtx& c, int slot, int tok) {
  const uint4* row = reinterpret_cast<const uint4*>(c.embed + (size_t)tok * c.d);  // 8 bf16 per vector
  float4* x = reinterpret_cast<float4*>(c.x + (size_t)slot * c.d);
  const int nv = c.d / 8;
  constexpr int U = 4;
  for (int base = 0; base < nv; base += U * blockDim.x) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * blockDim.x + threadIdx.x;
      if (i < nv) v[u] = row[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * blockDim.x + threadIdx.x;
      if (i < nv) {
        x[2 * i] = make_float4(bf16lo(v[u].x), bf16hi(v[u].x), bf16lo(v[u].y), bf16hi(v[u].y));
        x[2 * i + 1] = make_float4(bf16lo(v[u].z), bf16hi(v[u].z), bf16lo(v[u].w), bf16hi(v[u].w));
      }
    }
  }
}

__global__ void __launch_bounds__(256) sched_tick_kernel(const TickCtx* ctxp, int begin) {
  __shared__ __align__(16) Sched s;
  __shared__ int s_launch_slot, s_launch_pos;
  pdl_wait();  // head results of this tick
  pdl_trigger();
  const TickCtx c = *ctxp;
  copy_words(&s, c.sched, sizeof(Sched));
  __syncthreads();
  // multi-rank: this tick's boxes — all-gathered by the caller, or peer-stored (p2p)
  const float* inbox = c.inbox;
  if (!begin && c.p2p) inbox = p2p_wait_latest(c);
  if (!begin && inbox && c.owner_prev >= 0) {
    // the chain stage lo-1 (another rank) ran this tick arrives with its activation
    const int prev = s.work[c.lo - 1];
    if (prev >= 0) {
      const float* box = inbox + (size_t)c.owner_prev * c.box_words;
      float* x = c.x + (size_t)prev * c.d;
      for (int i = threadIdx.x; i < c.d; i += blockDim.x) x[i] = box[kBoxHeader + i];
    }
  }
  __shared__ int s_exit_tok, s_final_ok, s_final_tok;
  if (threadIdx.x == 0) {
    s_exit_tok = c.work->head_out[0];
    s_final_tok = c.work->head_out[1];
    s_final_ok = -1;  // greedy verdict inside sched_finish
  }
  __syncthreads();
  if (!begin && !c.greedy && s.c.model != 0) {
    if (inbox && c.box_logits) {
      // replicated sampling: every rank draws from the owners' logits, so the
      // draft / verify / commit streams advance identically everywhere
      float* l = const_cast<float*>(c.logits32);
      const float* ex = inbox + (size_t)c.owner_k * c.box_words + kBoxHeader + c.d;
      const float* fi = inbox + (size_t)c.owner_S * c.box_words + kBoxHeader + c.d + c.vocab;
      for (int i = threadIdx.x; i < c.vocab; i += blockDim.x) {
        l[i] = ex[i];
        l[c.vocab + i] = fi[i];
      }
      __syncthreads();
    }
    int e = -1, ok = -1, f = -1;
    sampling_tick(c, s, &e, &ok, &f);
    if (threadIdx.x == 0) {
      s_exit_tok = e;
      s_final_ok = ok;
      s_final_tok = f;
    }
    __syncthreads();
  }
  if (!begin && c.tap && c.logits32 && !inbox) {  // logits tap, before sched_finish moves the chains
    __shared__ int s_tp[2], s_trow[2];
    if (threadIdx.x == 0) {
      // exit head: folded, the chain launched last tick (eager shallow stages);
      // pipelined, the chain at the exit stage. Final head: the chain at
      // stage S (folded: its row of the deep batch).
      const int es = c.fold ? (s.launched ? s.work[1] : -1) : s.exit_slot;
      s_tp[0] = es >= 0 ? s.ch_pos[es] : -1;
      s_trow[0] = 0;
      s_tp[1] = s.final_slot >= 0 ? s.ch_pos[s.final_slot] : -1;
      s_trow[1] = c.fold ? 1 + s_tp[1] - s.fold_base : 1;
    }
    __syncthreads();
    for (int wh = 0; wh < 2; ++wh) {
      const int p = s_tp[wh];
      if (p < 1 || p > c.tap_max) continue;
      const float* src = c.logits32 + (size_t)s_trow[wh] * c.vocab;
      float* dst = c.tap + ((size_t)p * 2 + wh) * c.vocab;
      for (int i = threadIdx.x; i < c.vocab; i += blockDim.x) dst[i] = src[i];
    }
  }
  if (threadIdx.x == 0) {
    int exit_tok = s_exit_tok, final_tok = s_final_tok;
    if (inbox && c.greedy) {  // replicated scheduler: head results come from their owners' boxes
      exit_tok = reinterpret_cast<const int32_t*>(inbox + (size_t)c.owner_k * c.box_words)[0];
      final_tok = reinterpret_cast<const int32_t*>(inbox + (size_t)c.owner_S * c.box_words)[1];
    }
    if (c.fold && !begin) {
      // the chain launched last tick ran its shallow stages and exit head
      // eagerly (with a deep batch and fold_comb: inside the final-head launch)
      if (s.launched)
        s.ch_draft[s.work[1]] = c.fold_comb && s.fold_nb > 0 ? c.work_deep->head_out[0] : c.work->head_out[0];
      if (c.greedy) exit_tok = s.exit_slot >= 0 ? s.ch_draft[s.exit_slot] : -1;
      final_tok = (c.greedy && s.final_slot >= 0)
                      ? c.work_deep->vec_out[s.ch_pos[s.final_slot] - s.fold_base] : final_tok;
    }
    // rank fold: the chain that ran its eager stages last tick keeps its
    // draft until the machine emits it at stage k
    if (c.rfold && !begin && c.work->slot[0] >= 0 && c.work->head_slot[0] >= 0)
      s.ch_draft[c.work->slot[0]] = c.work->head_out[0];
    if (!begin)
      sched_finish(&s, exit_tok, final_tok, c.tokens, c.pdig, c.trace, c.trace_cap, s_final_ok);
    sched_plan(&s);
    Work* w = c.work;
    if (c.fold) {  // sched.h: sched_fold_plan
      sched_fold_plan(&s);
      const int row = s.fold_row;
      w->G = 1;
      w->slot[0] = row;
      w->pos[0] = row >= 0 ? s.c.n_prompt + s.ch_pos[s.work[1]] - 2 : 0;
      w->first[0] = 0;
      w->nl[0] = s.c.shallow_layers;
      w->nv[0] = 1;
      w->head_slot[0] = row;
      w->head_slot[1] = -1;
      Work* wd = c.work_deep;
      wd->G = 1;
      wd->slot[0] = s.fold_nb > 0 ? 0 : -1;
      wd->pos[0] = s.c.n_prompt + s.fold_base - 2;
      wd->first[0] = s.c.shallow_layers;
      wd->nl[0] = s.c.n_layers - s.c.shallow_layers;
      wd->nv[0] = s.fold_nb > 0 ? s.fold_nb : 1;
      wd->head_slot[0] = wd->head_slot[1] = -1;
      wd->head_exit = -1;
      if (c.fold_comb && s.fold_nb > 0 && row >= 0) {  // exit head inside the final-head launch
        wd->head_exit = c.comb_row;
        wd->src_slot = row;
        w->head_slot[0] = -1;
        s.fold_comb += 1;
      }
      if (s.fold_nb > 0 && c.has_cond) cudaGraphSetConditional(c.cond, 1u);
      if (c.hl) {  // exit-head layer on a copy of the launched chain's exit state
        plan_head_layer(c, c.work_head, row, w->pos[0], 1);
        w->head_slot[0] = row >= 0 ? c.head_row : -1;
      }
      s_launch_slot = row;
      s_launch_pos = row >= 0 ? s.ch_pos[s.work[1]] : 0;
    } else if (c.rfold) {  // sched.h: sched_rfold_plan
      sched_rfold_plan(&s);
      const int lo = c.lo, hi = c.hi, k = s.c.k;
      const int a = s.work[lo];
      const bool eager = lo <= k;  // the rank owns the exit stage: stages lo..k + exit head on arrival
      w->G = 1;
      w->slot[0] = eager ? a : -1;
      w->pos[0] = a >= 0 ? s.c.n_prompt + s.ch_pos[a] - 2 : 0;
      w->first[0] = s.c.stage_first[lo];
      w->nl[0] = eager ? s.c.stage_first[k] + s.c.stage_layers[k] - s.c.stage_first[lo] : 1;
      w->nv[0] = 1;
      w->head_slot[0] = eager ? a : -1;
      w->head_slot[1] = -1;
      const int ex = s.exit_slot;
      w->exit_tok = !eager || ex < 0 ? -1 : k == lo ? -2 : s.ch_draft[ex];
      Work* wd = c.work_deep;
      const int dlo = sched_rfold_first(&s.c, lo);
      wd->G = 1;
      wd->slot[0] = s.fold_nb > 0 ? c.rf_row0 : -1;
      wd->pos[0] = s.c.n_prompt + s.fold_base - 2;
      wd->first[0] = s.c.stage_first[dlo];
      wd->nl[0] = s.c.stage_first[hi] + s.c.stage_layers[hi] - s.c.stage_first[dlo];
      wd->nv[0] = s.fold_nb > 0 ? s.fold_nb : 1;
      wd->head_slot[0] = wd->head_slot[1] = -1;
      for (int j = 0; j < s.fold_nb; ++j) wd->rf_src[j] = (s.fold_base + j) % s.c.nslot;
      // this tick's box: the chain due at stage hi (its row of the latest batch)
      const int due = s.work[hi];
      const int di = due >= 0 ? s.ch_pos[due] - s.fold_base : -1;
      w->out_row = due >= 0 && hi < s.c.S ? c.rf_row0 + di : -1;
      w->out_slot = due;
      w->out_pos = due >= 0 ? s.c.n_prompt + s.ch_pos[due] - 2 : -1;
      w->final_idx = due >= 0 && hi == s.c.S ? di : -1;
      if (s.fold_nb > 0 && c.has_cond) cudaGraphSetConditional(c.cond, 1u);
      s_launch_slot = (s.launched && lo == 1) ? s.work[1] : -1;
      s_launch_pos = s_launch_slot >= 0 ? s.ch_pos[s_launch_slot] : 0;
    } else {
      w->G = c.hi - c.lo + 1;
      for (int g = 0; g < w->G; ++g) {
        const int st = c.lo + g;
        const int slot = s.work[st];
        w->slot[g] = slot;
        w->pos[g] = slot >= 0 ? s.c.n_prompt + s.ch_pos[slot] - 2 : 0;
        w->first[g] = s.c.stage_first[st];
        w->nl[g] = s.c.stage_layers[st];
        w->nv[g] = 1;
      }
      w->head_slot[0] = (s.c.k >= c.lo && s.c.k <= c.hi) ? s.exit_slot : -1;
      w->head_slot[1] = (s.c.S >= c.lo && s.c.S <= c.hi) ? s.final_slot : -1;
      if (c.hl) {  // exit-head layer on a copy of the exit chain's state (exit stage's rank)
        const int ex = w->head_slot[0];
        plan_head_layer(c, c.work_head, ex, ex >= 0 ? s.c.n_prompt + s.ch_pos[ex] - 2 : 0, 1);
        w->head_slot[0] = ex >= 0 ? c.head_row : -1;
      }
      s_launch_slot = (s.launched && c.lo == 1) ? s.work[1] : -1;
      s_launch_pos = s_launch_slot >= 0 ? s.ch_pos[s_launch_slot] : 0;
    }
  }
  __syncthreads();
  const int slot = s_launch_slot;
  if (slot >= 0) {
    const int idx = s.c.n_prompt + s_launch_pos - 2;  // last token of the chain's prefix
    if (c.model == PPSD_MODEL_TRANSFORMER) {
      embed_row(c, slot, c.tokens[idx]);
    } else if (c.model == PPSD_MODEL_TOYLM && threadIdx.x == 0) {
      c.chain_dig[slot] = c.pdig[idx + 1];  // prefix digest (pipesim.py:768)
    }
  }
  copy_words(c.sched, &s, sizeof(Sched));
}

// Multi-rank: publish this rank's head results and the activation leaving
// its last local stage (decode tick), or the prefill activation.
__global__ void __launch_bounds__(256) pack_outbox_kernel(const TickCtx* ctxp, int prefill) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  int32_t* hdr = reinterpret_cast<int32_t*>(c.outbox);
  const Work* w = prefill ? c.work_ar : c.work;
  const bool rf = c.rfold && !prefill;  // rank fold: the due chain's row of the latest batch
  const int slot = rf ? w->out_slot : w->slot[w->G - 1];
  const int row = rf ? w->out_row : slot;
  const bool send = row >= 0 && (prefill || c.hi < c.model_stages);
  if (threadIdx.x == 0) {
    if (rf) {
      hdr[0] = w->exit_tok == -2 ? w->head_out[0] : w->exit_tok;
      hdr[1] = w->final_idx >= 0 ? c.work_deep->vec_out[w->final_idx] : -1;
    } else {
      hdr[0] = w->head_slot[0] >= 0 ? w->head_out[0] : -1;
      hdr[1] = w->head_slot[1] >= 0 ? w->head_out[1] : -1;
    }
    hdr[2] = send ? slot : -1;
    hdr[3] = send ? (rf ? w->out_pos : w->pos[w->G - 1]) : -1;
  }
  if (send) {
    const float* x = c.x + (size_t)row * c.d;
    for (int i = threadIdx.x; i < c.d; i += blockDim.x) c.outbox[kBoxHeader + i] = x[i];
  }
  if (c.box_logits && !prefill) {  // sampling: the exit / final logits of the heads this rank owns
    float* dst = c.outbox + kBoxHeader + c.d;
    if (w->head_slot[0] >= 0)
      for (int i = threadIdx.x; i < c.vocab; i += blockDim.x) dst[i] = c.logits32[i];
    if (w->head_slot[1] >= 0)
      for (int i = threadIdx.x; i < c.vocab; i += blockDim.x) dst[c.vocab + i] = c.logits32[c.vocab + i];
  }
  if (c.p2p) {  // NVLink peer stores into every rank's exchange buffer + release flags
    __syncthreads();
    p2p_publish(c);
  }
}

// Folded tick with a deep batch (fold_comb): the launched chain's exit state
// into row comb_row before the deep layers advance its own row.
__global__ void __launch_bounds__(256) fold_exit_copy_kernel(const TickCtx* ctxp) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  const Work* wd = c.work_deep;
  if (wd->head_exit < 0) return;
  const float4* src = reinterpret_cast<const float4*>(c.x + (size_t)wd->src_slot * c.d);
  float4* dst = reinterpret_cast<float4*>(c.x + (size_t)wd->head_exit * c.d);
  for (int i = threadIdx.x; i < c.d / 4; i += blockDim.x) dst[i] = src[i];
}

// Rank fold: open the deferred batch's graph IF node for this launch (the
// scheduler kernel planned the tick at the end of the previous launch).
__global__ void rf_cond_kernel(const TickCtx* ctxp, unsigned long long handle) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0 && ctxp->work_deep->slot[0] >= 0) cudaGraphSetConditional(handle, 1u);
}

// Rank fold: the batch chains' activations (stage-lo inputs, or the eager
// stages' outputs) from their slots into the consecutive batch rows.
__global__ void __launch_bounds__(256) rf_gather_kernel(const TickCtx* ctxp) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  const Work* wd = c.work_deep;
  if (wd->slot[0] < 0) return;
  const int nv = wd->nv[0], d4 = c.d / 4;
  for (int j = 0; j < nv; ++j) {
    const float4* src = reinterpret_cast<const float4*>(c.x + (size_t)wd->rf_src[j] * c.d);
    float4* dst = reinterpret_cast<float4*>(c.x + (size_t)(wd->slot[0] + j) * c.d);
    for (int i = threadIdx.x; i < d4; i += blockDim.x) dst[i] = src[i];
  }
}

// p2p: wait until every rank published the latest exchange (orders the first
// decode tick after every rank finished reading the last prefill box)
__global__ void __launch_bounds__(32) p2p_wait_kernel(const TickCtx* ctxp) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  if (c.p2p) p2p_wait_latest(c);
}

// Multi-rank pipelined prefill: at step p rank r runs its layers on prompt
// token p - r; its input is the embedding (rank 0) or rank r-1's box.
__global__ void __launch_bounds__(256) mr_prefill_begin_kernel(const TickCtx* ctxp, ArCtl* ctl) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  const int p = ctl->j;
  const int j = p - c.rank;
  const bool active = j >= 0 && j < c.n_prompt - 1;
  const float* inbox = c.inbox;
  if (c.p2p && p > 0) inbox = p2p_wait_latest(c);  // every rank, every step: lockstep
  __syncthreads();
  if (threadIdx.x == 0) {
    Work* w = c.work_ar;
    w->G = 1;
    w->slot[0] = active ? 0 : -1;
    w->nv[0] = 1;
    w->pos[0] = active ? j : 0;
    w->first[0] = ctl->first_layer;
    w->nl[0] = ctl->n_layers;
    w->head_slot[0] = w->head_slot[1] = -1;
    if (c.hl) {  // exit rank: [0, split) -> head layer on a copy -> [split, local end)
      split_prefill(c, ctl, w, active, j, 1);
    }
    ctl->j = p + 1;
  }
  if (!active) return;
  if (c.rank == 0) {
    embed_row(c, 0, c.tokens[j]);
  } else {
    const float* box = inbox + (size_t)(c.rank - 1) * c.box_words;
    for (int i = threadIdx.x; i < c.d; i += blockDim.x) c.x[i] = box[kBoxHeader + i];
  }
}

// Batched prefill: the next chunk of up to kMaxVec prompt tokens goes through
// the layers as ONE group of nv vectors (ceil(nv/m) weight passes per matrix
// instead of nv), positions j0..j0+nv-1.
__global__ void __launch_bounds__(256) prefill_chunk_kernel(const TickCtx* ctxp, ArCtl* ctl) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  __shared__ int s_j0, s_n;
  if (threadIdx.x == 0) {
    const int j0 = ctl->j;
    const int n = min(c.prefill_chunk, ctl->end - j0);
    Work* w = c.work_ar;
    w->G = 1;
    w->slot[0] = n > 0 ? 0 : -1;
    w->nv[0] = n > 0 ? n : 1;
    w->pos[0] = j0;
    w->first[0] = ctl->first_layer;
    w->nl[0] = ctl->n_layers;
    w->head_slot[0] = w->head_slot[1] = -1;
    if (c.hl) {  // [0, split) -> head layer on copies -> [split, N)
      split_prefill(c, ctl, w, n > 0, j0, n > 0 ? n : 1);
    }
    ctl->j = j0 + (n > 0 ? n : 0);
    s_j0 = j0;
    s_n = n;
  }
  __syncthreads();
  for (int v = 0; v < s_n; ++v) embed_row(c, v, c.tokens[s_j0 + v]);
}

// ---- autoregressive / prefill control (decode_autoregressive, pipesim.py:390-409)
__global__ void __launch_bounds__(256) ar_begin_kernel(const TickCtx* ctxp, ArCtl* ctl, int with_head) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  const int j = ctl->j;
  if (threadIdx.x == 0) {
    Work* w = c.work_ar;
    w->G = 1;
    w->slot[0] = 0;
    w->nv[0] = 1;
    w->pos[0] = j;
    w->first[0] = ctl->first_layer;
    w->nl[0] = ctl->n_layers;
    w->head_slot[0] = -1;
    w->head_slot[1] = with_head ? 0 : -1;
  }
  embed_row(c, 0, c.tokens[j]);
}

__global__ void ar_end_kernel(const TickCtx* ctxp, ArCtl* ctl, int with_head) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  const int j = ctl->j;
  int tok = c.work_ar->head_out[1];
  if (with_head && !c.greedy) {  // sample_token(q, commit_stream), one draw per token
    const int V = c.vocab;
    const bool exact = V <= kExactVocab;
    block_softmax(nullptr, c.logits32 + V, V, c.qbuf, exact);
    tok = block_sample(c.qbuf, V, counter_uniform(c.commit_seed, (uint64_t)(j - ctl->end)), exact);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (with_head) c.tokens[j + 1] = tok;
    ctl->j = j + 1;
  }
}

// Exit-head layer input: rows slot[0] .. +nv of `wh` = rows src_slot .. (the
// exit-layer state of the drafting chain(s)); the head layer then runs on the
// copies in place and the chains' own rows continue unchanged.
__global__ void __launch_bounds__(256) head_copy_kernel(const TickCtx* ctxp, const Work* wh) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  const int dst = wh->slot[0], src = wh->src_slot, nv = wh->nv[0];
  if (dst < 0 || src < 0) return;
  for (int v = 0; v < nv; ++v) {
    const float4* a = reinterpret_cast<const float4*>(c.x + (size_t)(src + v) * c.d);
    float4* b = reinterpret_cast<float4*>(c.x + (size_t)(dst + v) * c.d);
    for (int i = threadIdx.x; i < c.d / 4; i += blockDim.x) b[i] = a[i];
  }
}

}  // namespace ppsd
