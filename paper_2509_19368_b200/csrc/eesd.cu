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
#include "sample.cuh"

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

// One round's bookkeeping. The verdicts are given: n_acc leading drafts
// accepted, then (n_acc < gamma) the rejected draft's committed token
// `corrected`, or (n_acc == gamma) the bonus token. The drafts already sit in
// tokens[n_prompt+base .. +gamma).
__device__ void eesd_account_verdicts(EesdState* s, int n_acc, int corrected, int bonus, int32_t* tokens,
                                      uint64_t* pdig, TraceRow* tr, int64_t cap) {
  const int g = s->gamma, S = s->S, per = s->per, dt = s->dt, k = s->k;
  const int base = s->committed, t = s->t;
  const int vt = t + g * dt + (S - 1) * per + 1;
  const int np = s->n_prompt;
  for (int h = 1; h <= g; ++h)  // pipesim.py:486-491
    eesd_trace(s, tr, cap, t + h * dt, k, kKindDraft, base + h, s->model ? tokens[np + base + h - 1] : kNone,
               kVerdictNone);
  for (int st = 1; st < S; ++st)  // pipesim.py:492-498
    eesd_trace(s, tr, cap, t + g * dt + (st - 1) * per + 1, st, kKindAct, base + 1, kNone, kVerdictNone);
  for (int h = 1; h <= n_acc; ++h)  // pipesim.py:501-529
    eesd_trace(s, tr, cap, vt, S, kKindFinal, base + h, s->model ? tokens[np + base + h - 1] : kNone,
               kVerdictAccept);
  if (n_acc < g) eesd_trace(s, tr, cap, vt, S, kKindCheck, base + n_acc + 1, corrected, kVerdictReject);
  if (n_acc == g) {  // pipesim.py:531-541
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

// Greedy / Bernoulli verdicts (thread 0). model: top[h-1] = final-head argmax
// after the prefix holding drafts 1..h-1 (h = 1..gamma+1).
__device__ void eesd_account(EesdState* s, const int32_t* top, int32_t* tokens, uint64_t* pdig, TraceRow* tr,
                             int64_t cap) {
  const int g = s->gamma, np = s->n_prompt, base = s->committed;
  int n_acc = 0, corrected = kNone;
  for (int h = 1; h <= g; ++h) {  // pipesim.py:501-529
    bool ok;
    if (s->model) {
      ok = tokens[np + base + h - 1] == top[h - 1];  // greedy_match
      if (!ok) corrected = top[h - 1];
    } else {
      ok = counter_uniform(s->verify_seed, s->verify_counter++) < s->alpha;
    }
    if (!ok) break;
    n_acc += 1;
  }
  eesd_account_verdicts(s, n_acc, corrected, s->model ? top[g] : kNone, tokens, pdig, tr, cap);
}

// Sampling verdicts, block-wide (pipesim.py:501-541 with _ToyVerifier,
// :346-365): draft h's p sits in pdist row h-1; q_h = softmax of the final
// logits after drafts 1..h-1 (fill_q(h, out) writes them). accept_draft draws
// from the verify stream, a rejection resamples the residual max(q - p, 0)
// with the commit stream, a clean sweep samples the bonus from q_{gamma+1}.
template <class FillQ>
__device__ void eesd_sampling_round(const TickCtx& c, EesdState* es, FillQ fill_q) {
  const int V = c.vocab, g = es->gamma;
  const bool exact = V <= kExactVocab;
  __shared__ int s_stop, s_ok, s_tok;
  __shared__ double s_u;
  int n_acc = 0, corrected = kNone, bonus = kNone;
  for (int h = 1; h <= g + 1; ++h) {
    fill_q(h, c.qbuf);  // q_h
    __syncthreads();
    block_softmax(c.qbuf, nullptr, V, c.qbuf, exact);
    if (h == g + 1) {  // bonus: full_model_token(q)
      if (threadIdx.x == 0) s_u = counter_uniform(c.commit_seed, es->commit_counter++);
      __syncthreads();
      bonus = block_sample(c.qbuf, V, s_u, exact);
      break;
    }
    const double* p = c.pdist + (size_t)(h - 1) * V;
    if (threadIdx.x == 0) {
      const int d = c.tokens[es->n_prompt + es->committed + h - 1];
      const double r = counter_uniform(es->verify_seed, es->verify_counter++);
      const double pt = p[d], qt = c.qbuf[d];
      s_ok = (qt != 0.0) && r <= fmin(1.0, __ddiv_rn(qt, pt));  // speccore.py:90-101
      if (!s_ok) s_u = counter_uniform(c.commit_seed, es->commit_counter++);
    }
    __syncthreads();
    if (s_ok) {
      ++n_acc;
      continue;
    }
    for (int i = threadIdx.x; i < V; i += blockDim.x) c.wbuf[i] = fmax(__dsub_rn(c.qbuf[i], p[i]), 0.0);
    __syncthreads();
    const double z = block_sum(c.wbuf, V, exact);
    if (z <= 1e-12 && threadIdx.x == 0) es->error |= kErrResidual;
    for (int i = threadIdx.x; i < V; i += blockDim.x) c.wbuf[i] = __ddiv_rn(c.wbuf[i], z);
    __syncthreads();
    corrected = block_sample(c.wbuf, V, s_u, exact);
    break;
  }
  (void)s_stop;
  (void)s_tok;
  if (threadIdx.x == 0) eesd_account_verdicts(es, n_acc, corrected, bonus, c.tokens, c.pdig, c.trace, c.trace_cap);
  __syncthreads();
}

// draft sample (sampling mode): p = softmax(exit logits) -> pdist row h,
// token = sample_token(p, draft_stream)
__device__ int eesd_sample_draft(const TickCtx& c, EesdState* es, int h, const double* l64, const float* l32) {
  const int V = c.vocab;
  const bool exact = V <= kExactVocab;
  double* p = c.pdist + (size_t)h * V;
  block_softmax(l64, l32, V, p, exact);
  __shared__ double s_ud;
  if (threadIdx.x == 0) s_ud = counter_uniform(c.draft_seed, es->draft_counter++);
  __syncthreads();
  return block_sample(p, V, s_ud, exact);
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
    if (c.hl) {  // exit-head layer on a copy of the draft's exit state
      Work* wh = c.work_head;
      wh->G = 1;
      wh->slot[0] = s_done ? -1 : c.head_row;
      wh->src_slot = 0;
      wh->pos[0] = s_j;
      wh->first[0] = c.hl_layer;
      wh->nl[0] = 1;
      wh->nv[0] = 1;
      wh->head_slot[0] = wh->head_slot[1] = -1;
      w->head_slot[0] = s_done ? -1 : c.head_row;
    }
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
  __shared__ int s_done;
  if (threadIdx.x == 0) s_done = es->done;
  __syncthreads();
  if (s_done) return;
  int tok = c.work_ar->head_out[0];  // greedy: draft = exit-head argmax (pipesim.py:475-483)
  if (!c.greedy)  // draft h of the round: sample p = softmax(exit logits, row 0)
    tok = eesd_sample_draft(c, es, es->len - (es->n_prompt + es->committed), nullptr, c.logits32);
  if (threadIdx.x == 0) {
    c.tokens[es->len] = tok;
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
  __shared__ int s_done;
  if (threadIdx.x == 0) s_done = es->done;
  __syncthreads();
  if (s_done) return;
  if (c.greedy) {
    if (threadIdx.x == 0) eesd_account(es, c.work_ar->vec_out, c.tokens, nullptr, c.trace, c.trace_cap);
    return;
  }
  // sampling: q_h from the batched verify's final logits, row h-1 (kMatHeadV)
  const int V = c.vocab;
  eesd_sampling_round(c, es, [&](int h, double* out) {
    for (int v = threadIdx.x; v < V; v += blockDim.x) out[v] = (double)c.logits32[(size_t)(h - 1) * V + v];
  });
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
  if (es->model && !c.greedy) {  // sampling mode (_ToyVerifier, pipesim.py:346-365)
    const double beta = c.beta;
    const int V = c.vocab;
    for (int h = 0; h < g; ++h) {
      const int len = es->len;
      const uint64_t d0 = c.pdig[len];
      const uint64_t fin = toy_advance(d0, 0, c.n_layers);
      const uint64_t ex = toy_advance(d0, 0, es->exit_layer);
      for (int v = threadIdx.x; v < V; v += blockDim.x) {
        double z = __dmul_rn(__dsub_rn(eesd_toy_unit(fin, kLogitSalt, v), 0.5), 8.0);
        if (beta != 0.0)
          z = __dadd_rn(z, __dmul_rn(beta, __dsub_rn(__dmul_rn(2.0, eesd_toy_unit(ex, kNoiseSalt, v)), 1.0)));
        c.logits64[v] = z;
      }
      __syncthreads();
      const int tok = eesd_sample_draft(c, es, h, c.logits64, nullptr);
      if (threadIdx.x == 0) {
        c.tokens[len] = tok;
        c.pdig[len + 1] = toy_extend(d0, tok);
        es->len = len + 1;
      }
      __syncthreads();
    }
    eesd_sampling_round(c, es, [&](int h, double* out) {  // q_h: prefix holding drafts 1..h-1
      const uint64_t fin = toy_advance(c.pdig[es->n_prompt + es->committed + h - 1], 0, c.n_layers);
      for (int v = threadIdx.x; v < V; v += blockDim.x)
        out[v] = __dmul_rn(__dsub_rn(eesd_toy_unit(fin, kLogitSalt, v), 0.5), 8.0);
    });
    return;
  }
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
