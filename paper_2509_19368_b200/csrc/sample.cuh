// sample.cuh — sampling-mode verification on the device:
// softmax in float64 with numpy's summation order, the inverse-CDF draw of
// speccore.sample_token (speccore.py:76-87), accept_draft's r <= min(1, q/p)
// (speccore.py:90-101) and the residual resample (speccore.py:104-113),
// driven by the three counter streams of _ToyVerifier (pipesim.py:339-344).
//
// Exact mode (vocab <= kExactVocab, the ToyLM parity configs): the softmax
// normaliser and the residual mass use numpy's pairwise summation
// (0 + pairwise(a): 8-accumulator leaves of <= 128, split at n/2 rounded down
// to a multiple of 8) and the CDF is a left-to-right fold, as np.cumsum. Only
// exp() can differ from numpy's by an ulp, which moves a sample only if the
// uniform draw lands within ~1e-16 of a CDF boundary. Large vocabularies
// (transformer heads, fp32 logits) use block-parallel sums instead.
#pragma once
#include <float.h>

#include "engine_dev.cuh"

namespace ppsd {

constexpr int kExactVocab = 4096;

__device__ inline double np_pairwise(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(a, n2), np_pairwise(a + n2, n - n2));
}

// block-wide: sum of a[0..n) — numpy order (thread 0) or a fixed tree
__device__ inline double block_sum(const double* a, int n, bool exact) {
  __shared__ double s_part[32];
  __shared__ double s_res;
  if (exact) {
    if (threadIdx.x == 0) s_res = __dadd_rn(0.0, np_pairwise(a, n));
  } else {
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v += a[i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_part[w];
      s_res = t;
    }
  }
  __syncthreads();
  const double r = s_res;
  __syncthreads();
  return r;
}

// out = softmax(logits) in float64 (toylm.py:45-48); logits in fp64 or fp32
__device__ inline void block_softmax(const double* l64, const float* l32, int V, double* out, bool exact) {
  __shared__ double s_max[32];
  __shared__ double s_m;
  double m = -DBL_MAX;
  for (int i = threadIdx.x; i < V; i += blockDim.x) m = fmax(m, l64 ? l64[i] : (double)l32[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = s_max[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, s_max[w]);
    s_m = t;
  }
  __syncthreads();
  const double mx = s_m;
  for (int i = threadIdx.x; i < V; i += blockDim.x) out[i] = exp(__dsub_rn(l64 ? l64[i] : (double)l32[i], mx));
  __syncthreads();
  const double z = block_sum(out, V, exact);
  for (int i = threadIdx.x; i < V; i += blockDim.x) out[i] = __ddiv_rn(out[i], z);
  __syncthreads();
}

// inverse CDF: first index whose running sum exceeds u (np.searchsorted side=right)
__device__ inline int block_sample(const double* p, int V, double u, bool exact) {
  __shared__ int s_idx;
  __shared__ double s_tot[256];
  if (exact) {
    if (threadIdx.x == 0) {
      double cum = 0.0;
      int idx = V;
      for (int i = 0; i < V; ++i) {
        cum = __dadd_rn(cum, p[i]);
        if (cum > u) { idx = i; break; }
      }
      s_idx = idx < V ? idx : V - 1;
    }
  } else {  // chunked scan: deterministic, not numpy's rounding
    const int nt = blockDim.x;
    const int per = (V + nt - 1) / nt;
    const int lo = threadIdx.x * per, hi = min(V, lo + per);
    double t = 0.0;
    for (int i = lo; i < hi; ++i) t += p[i];
    s_tot[threadIdx.x] = t;
    if (threadIdx.x == 0) s_idx = V;
    __syncthreads();
    double base = 0.0;
    for (int j = 0; j < (int)threadIdx.x; ++j) base += s_tot[j];
    double cum = base;
    for (int i = lo; i < hi; ++i) {
      cum += p[i];
      if (cum > u) { atomicMin(&s_idx, i); break; }
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_idx >= V) s_idx = V - 1;
  }
  __syncthreads();
  const int r = s_idx;
  __syncthreads();
  return r;
}

}  // namespace ppsd
