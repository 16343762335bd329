// eesd.cu — the draft-then-verify baseline (EESD, pkg/src/specpipe/pipesim.py:435-551)
// on the device: per round gamma one-token drafts through the first
// exit_layer layers + exit head, then ONE batched verify of the gamma+1
// positions through all N layers (kMatHeadV gives every position's final
// argmax), then the acceptance scan. eesd_account restates the scan,
// bonus / truncate and tick accounting with trace rows in the reference's
// append order. The batched verify reuses the batch-invariant GEMVs, so
// verify logits equal the autoregressive ones bit-for-bit and greedy EESD
// stays lossless.
#include <float.h>
#include <limits.h>

#include "engine_dev.cuh"

namespace ppsd {

__device__ void eesd_trace(EesdState* s, TraceRow* tr, int64_t cap, int tick, int st, int kind, int pos,
                           int tok, int verdict) {
  if (!tr) return;
  if (s->trace_n >= cap) {
    s->error |= kErrTrace;
    return;
  }
  TraceRow r;
  r.tick = tick;
  r.stage = st;
  r.kind = kind;
  r.position = pos;
  r.token = tok;
  r.verdict = verdict;
  tr[s->trace_n++] = r;
}

// One round's bookkeeping. model: top[h-1] = final-head argmax after the
// prefix holding drafts 1..h-1 (h = 1..gamma+1); the drafts already sit in
// tokens[n_prompt+base .. +gamma). Bernoulli: verdicts from the stream.
__device__ void eesd_account(EesdState* s, const int32_t* top, int32_t* tokens, uint64_t* pdig, TraceRow* tr,
                             int64_t cap) {
  const int g = s->gamma, S = s->S, per = s->per, dt = s->dt, k = s->k;
  const int base = s->committed, t = s->t;
  const int vt = t + g * dt + (S - 1) * per + 1;
  const int np = s->n_prompt;
  for (int h = 1; h <= g; ++h)  // pipesim.py:486-491
    eesd_trace(s, tr, cap, t + h * dt, k, kKindDraft, base + h, s->model ? tokens[np + base + h - 1] : kNone,
               kVerdictNone);
  for (int st = 1; st < S; ++st)  // pipesim.py:492-498
    eesd_trace(s, tr, cap, t + g * dt + (st - 1) * per + 1, st, kKindAct, base + 1, kNone, kVerdictNone);
  int n_acc = 0, corrected = kNone;
  for (int h = 1; h <= g; ++h) {  // pipesim.py:501-529
    bool ok;
    int tok = kNone, ctok = kNone;
    if (s->model) {
      tok = tokens[np + base + h - 1];
      ok = tok == top[h - 1];
      ctok = ok ? tok : top[h - 1];
    } else {
      ok = counter_uniform(s->verify_seed, s->verify_counter++) < s->alpha;
    }
    if (ok) {
      n_acc += 1;
      eesd_trace(s, tr, cap, vt, S, kKindFinal, base + h, tok, kVerdictAccept);
    } else {
      corrected = ctok;
      eesd_trace(s, tr, cap, vt, S, kKindCheck, base + h, ctok, kVerdictReject);
      break;
    }
  }
  if (n_acc == g) {  // pipesim.py:531-541
    const int bonus = s->model ? top[g] : kNone;
    if (s->model) {
      tokens[np + base + g] = bonus;
      if (pdig) pdig[np + base + g + 1] = toy_extend(pdig[np + base + g], bonus);
    }
    s->len = np + base + g + 1;
    eesd_trace(s, tr, cap, vt, S, kKindFinal, base + g + 1, bonus, kVerdictNone);
  } else if (s->model) {  // pipesim.py:542-543
    const int idx = np + base + n_acc;
    tokens[idx] = corrected;
    if (pdig) pdig[idx + 1] = toy_extend(pdig[idx], corrected);
    s->len = idx + 1;
  }
  s->drafted += g;
  s->accepts += n_acc;
  s->rejects += 1;
  s->committed += n_acc + 1;
  s->t += g * dt + S * per;
  if (s->committed >= s->horizon) s->done = 1;
}

// ---- transformer rounds: drafts through the first exit_layer layers -------
__global__ void eesd_draft_begin_kernel(const TickCtx* ctxp, EesdState* es) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  __shared__ int s_j, s_done;
  if (threadIdx.x == 0) {
    Work* w = c.work_ar;
    s_done = es->done;
    s_j = es->len - 1;
    w->G = 1;
    w->slot[0] = s_done ? -1 : 0;
    w->nv[0] = 1;
    w->pos[0] = s_j;
    w->first[0] = 0;
    w->nl[0] = es->exit_layer;
    w->head_slot[0] = s_done ? -1 : 0;
    w->head_slot[1] = -1;
  }
  __syncthreads();
  if (s_done) return;
  const int tok = c.tokens[s_j];
  const uint4* row = reinterpret_cast<const uint4*>(c.embed + (size_t)tok * c.d);
  for (int i = threadIdx.x; i < c.d / 8; i += blockDim.x) {
    const uint4 v = row[i];
    float* x = c.x + (size_t)i * 8;
    x[0] = bf16lo(v.x); x[1] = bf16hi(v.x); x[2] = bf16lo(v.y); x[3] = bf16hi(v.y);
    x[4] = bf16lo(v.z); x[5] = bf16hi(v.z); x[6] = bf16lo(v.w); x[7] = bf16hi(v.w);
  }
}

__global__ void eesd_draft_end_kernel(const TickCtx* ctxp, EesdState* es) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  if (threadIdx.x == 0 && !es->done) {
    c.tokens[es->len] = c.work_ar->head_out[0];  // draft = exit-head argmax (pipesim.py:475-483)
    es->len += 1;
  }
}

__global__ void eesd_verify_begin_kernel(const TickCtx* ctxp, EesdState* es) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  __shared__ int s_j0, s_nv, s_done;
  if (threadIdx.x == 0) {
    Work* w = c.work_ar;
    s_done = es->done;
    s_j0 = es->n_prompt + es->committed - 1;  // last committed token: verifies draft 1
    s_nv = es->gamma + 1;
    w->G = 1;
    w->slot[0] = s_done ? -1 : 0;
    w->nv[0] = s_nv;
    w->pos[0] = s_j0;
    w->first[0] = 0;
    w->nl[0] = es->n_layers;
    w->head_slot[0] = w->head_slot[1] = -1;
  }
  __syncthreads();
  if (s_done) return;
  for (int v = 0; v < s_nv; ++v) {
    const int tok = c.tokens[s_j0 + v];
    const uint4* row = reinterpret_cast<const uint4*>(c.embed + (size_t)tok * c.d);
    float* x = c.x + (size_t)v * c.d;
    for (int i = threadIdx.x; i < c.d / 8; i += blockDim.x) {
      const uint4 q = row[i];
      float* xx = x + (size_t)i * 8;
      xx[0] = bf16lo(q.x); xx[1] = bf16hi(q.x); xx[2] = bf16lo(q.y); xx[3] = bf16hi(q.y);
      xx[4] = bf16lo(q.z); xx[5] = bf16hi(q.z); xx[6] = bf16lo(q.w); xx[7] = bf16hi(q.w);
    }
  }
}

__global__ void eesd_scan_kernel(const TickCtx* ctxp, EesdState* es) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  if (threadIdx.x == 0 && !es->done) eesd_account(es, c.work_ar->vec_out, c.tokens, nullptr, c.trace, c.trace_cap);
}

// ---- ToyLM / Bernoulli rounds: one block per round ---------------------------
__device__ double eesd_toy_unit(uint64_t digest, uint64_t salt, int v) {
  const uint64_t keyed = (digest ^ ((uint64_t)v * (kTokenSalt | 1ull))) + salt;
  return __dmul_rn((double)(hmix64(keyed) >> 11), 0x1p-53);
}

template <class F>
__device__ int eesd_block_argmax(int V, F f) {
  __shared__ double s_v[32];
  __shared__ int s_i[32];
  double bv = -DBL_MAX;
  int bi = INT_MAX;
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const double z = f(v);
    if (z > bv) { bv = z; bi = v; }
  }
  for (int off = 16; off > 0; off >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s_v[warp] = bv; s_i[warp] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (s_v[w] > bv || (s_v[w] == bv && s_i[w] < bi)) { bv = s_v[w]; bi = s_i[w]; }
    s_i[0] = bi;
  }
  __syncthreads();
  const int r = s_i[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) eesd_toy_round_kernel(const TickCtx* ctxp, EesdState* es) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  __shared__ int s_top[kMaxVec + 1];
  __shared__ int s_done;
  if (threadIdx.x == 0) s_done = es->done;
  __syncthreads();
  if (s_done) return;
  const int g = es->gamma;
  if (es->model) {
    const double beta = c.beta;
    for (int h = 0; h < g; ++h) {  // drafts (pipesim.py:475-483)
      const int len = es->len;
      const uint64_t d0 = c.pdig[len];
      const uint64_t fin = toy_advance(d0, 0, c.n_layers);
      const uint64_t ex = toy_advance(d0, 0, es->exit_layer);
      const int tok = eesd_block_argmax(c.vocab, [&](int v) {
        double z = __dmul_rn(__dsub_rn(eesd_toy_unit(fin, kLogitSalt, v), 0.5), 8.0);
        if (beta != 0.0)
          z = __dadd_rn(z, __dmul_rn(beta, __dsub_rn(__dmul_rn(2.0, eesd_toy_unit(ex, kNoiseSalt, v)), 1.0)));
        return z;
      });
      if (threadIdx.x == 0) {
        c.tokens[len] = tok;
        c.pdig[len + 1] = toy_extend(d0, tok);
        es->len = len + 1;
      }
      __syncthreads();
    }
    for (int h = 0; h <= g; ++h) {  // final-head argmax after each draft prefix (pipesim.py:505-509, 533-534)
      const uint64_t fin = toy_advance(c.pdig[es->n_prompt + es->committed + h], 0, c.n_layers);
      const int top = eesd_block_argmax(c.vocab, [&](int v) {
        return __dmul_rn(__dsub_rn(eesd_toy_unit(fin, kLogitSalt, v), 0.5), 8.0);
      });
      if (threadIdx.x == 0) s_top[h] = top;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) eesd_account(es, s_top, c.tokens, c.pdig, c.trace, c.trace_cap);
}

}  // namespace ppsd
