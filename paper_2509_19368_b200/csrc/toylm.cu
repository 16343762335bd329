// toylm.cu — the reference ToyLM (pkg/src/specpipe/toylm.py:72-130) on the
// GPU, bit-exact: the digest chain is integer splitmix64, the logits are
// formed with explicitly rounded fp64 ops in numpy's evaluation order
// (no FMA contraction), and argmax keeps the lowest index among maxima like
// np.argmax. The reference takes argmax of softmax(logits); softmax is
// monotone, so argmax over the logits is the same token unless exp() maps
// two distinct logits to one double (logits live on a 2^-50 grid, see
// DESIGN.md §ToyLM).
#include <float.h>
#include <limits.h>

#include "engine_dev.cuh"
#include "sample.cuh"

namespace ppsd {

__device__ __forceinline__ double toy_unit(uint64_t digest, uint64_t salt, int v) {
  const uint64_t keyed = (digest ^ ((uint64_t)v * (kTokenSalt | 1ull))) + salt;  // toylm.py:109-112
  return __dmul_rn((double)(hmix64(keyed) >> 11), 0x1p-53);                    // toylm.py:51-52
}
__device__ __forceinline__ double toy_logit(uint64_t fin, int v) {  // toylm.py:114-116
  return __dmul_rn(__dsub_rn(toy_unit(fin, kLogitSalt, v), 0.5), 8.0);
}
__device__ __forceinline__ double toy_exit_logit(uint64_t fin, uint64_t ex, double beta, int v) {
  double z = toy_logit(fin, v);
  if (beta != 0.0) {  // toylm.py:118-130: logits + beta * (2u - 1)
    const double noise = __dsub_rn(__dmul_rn(2.0, toy_unit(ex, kNoiseSalt, v)), 1.0);
    z = __dadd_rn(z, __dmul_rn(beta, noise));
  }
  return z;
}

// block-wide first-index argmax of f(v) over v in [0, V)
template <class F>
__device__ int block_argmax(int V, F f) {
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

// One tick of stage compute for every local stage plus both heads.
__global__ void __launch_bounds__(256) toy_tick_kernel(const TickCtx* ctxp) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  Work* w = c.work;
  __shared__ uint64_t s_dig[kMaxStages];
  __shared__ int s_after[kMaxStages];
  if (threadIdx.x == 0) {
    for (int g = 0; g < w->G; ++g) {
      const int slot = w->slot[g];
      if (slot < 0) continue;
      const uint64_t d = toy_advance(c.chain_dig[slot], w->first[g], w->first[g] + w->nl[g]);
      s_dig[g] = d;
      s_after[g] = w->first[g] + w->nl[g];
      c.chain_dig[slot] = d;
    }
  }
  __syncthreads();
  for (int m = 0; m < 2; ++m) {
    const int slot = w->head_slot[m];
    if (slot < 0) continue;
    int g = 0;
    while (w->slot[g] != slot) ++g;
    const uint64_t d = s_dig[g];
    int tok;
    double* out64 = c.greedy ? nullptr : c.logits64 + (size_t)m * c.vocab;  // sampling: full logits
    if (m == 0) {  // exit head: final digest + noise keyed by the exit state (pipesim.py:711-715)
      const uint64_t fin = toy_advance(d, s_after[g], c.n_layers);
      const double beta = c.beta;
      tok = block_argmax(c.vocab, [&](int v) {
        const double z = toy_exit_logit(fin, d, beta, v);
        if (out64) out64[v] = z;
        return z;
      });
    } else {
      tok = block_argmax(c.vocab, [&](int v) {
        const double z = toy_logit(d, v);
        if (out64) out64[v] = z;
        return z;
      });
    }
    if (threadIdx.x == 0) w->head_out[m] = tok;
  }
}

// decode_autoregressive on the ToyLM (pipesim.py:390-409), one block.
__global__ void __launch_bounds__(256) toy_ar_kernel(const TickCtx* ctxp, int n_prompt, int max_tokens) {
  const TickCtx c = *ctxp;
  for (int i = 0; i < max_tokens; ++i) {
    const int len = n_prompt + i;
    const uint64_t d0 = c.pdig[len];
    const uint64_t fin = toy_advance(d0, 0, c.n_layers);
    int tok;
    if (c.greedy) {
      tok = block_argmax(c.vocab, [&](int v) { return toy_logit(fin, v); });
    } else {  // sample_token(q, commit_stream) (pipesim.py:403-406)
      for (int v = threadIdx.x; v < c.vocab; v += blockDim.x) c.logits64[v] = toy_logit(fin, v);
      __syncthreads();
      const bool exact = c.vocab <= kExactVocab;
      block_softmax(c.logits64, nullptr, c.vocab, c.qbuf, exact);
      tok = block_sample(c.qbuf, c.vocab, counter_uniform(c.commit_seed, (uint64_t)i), exact);
    }
    if (threadIdx.x == 0) {
      c.tokens[len] = tok;
      c.pdig[len + 1] = toy_extend(d0, tok);
    }
    __syncthreads();
  }
}

// Measured alignment of the exit head (toylm.py:160-192): for prefix i
// (sequence digest pdig[i]) p = softmax(exit logits at layer E), q =
// softmax(final logits); minsum[i] = sum(min(p, q)) in numpy's pairwise
// order, agree[i] = argmax p == argmax q (first index among maxima). One CTA
// per prefix; scratch = 4 * V doubles per prefix.
__global__ void __launch_bounds__(256) toy_alignment_kernel(const uint64_t* pdig, int n_layers, int exit_depth,
                                                            int vocab, uint64_t toy_seed, double beta,
                                                            double* scratch, double* minsum, int* agree) {
  (void)toy_seed;
  const int i = blockIdx.x, V = vocab;
  const bool exact = V <= kExactVocab;
  double* zl = scratch + (size_t)i * 4 * V;
  double* q = zl + V;
  double* p = q + V;
  double* w = p + V;
  const uint64_t d0 = pdig[i];
  const uint64_t fin = toy_advance(d0, 0, n_layers);
  const uint64_t ex = toy_advance(d0, 0, exit_depth);
  for (int v = threadIdx.x; v < V; v += blockDim.x) zl[v] = toy_logit(fin, v);
  __syncthreads();
  block_softmax(zl, nullptr, V, q, exact);
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x) zl[v] = toy_exit_logit(fin, ex, beta, v);
  __syncthreads();
  block_softmax(zl, nullptr, V, p, exact);
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x) w[v] = fmin(p[v], q[v]);
  __syncthreads();
  const double ms = block_sum(w, V, exact);
  const int ap = block_argmax(V, [&](int v) { return p[v]; });
  const int aq = block_argmax(V, [&](int v) { return q[v]; });
  if (threadIdx.x == 0) {
    minsum[i] = ms;
    agree[i] = ap == aq;
  }
}

}  // namespace ppsd
