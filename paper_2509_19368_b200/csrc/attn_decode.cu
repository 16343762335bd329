// attn_decode.cu — latency-first decode attention over the paged KV cache.
//
// The decode step attends 1..16 query vectors per (stage group, kv head) row
// to a context of <= 2048 positions; at the Llama-2-7B shape that is ~10 MB
// of K/V per layer (1.5 us at HBM speed) but the split-K kernel in
// attn_core.cuh spent ~8.7 us per launch on dependent global round trips:
// per-page partials to global, an atomic arrival ticket, and a serial merge
// by the last CTA. This kernel keeps the same per-page arithmetic and the
// same page-order merge (so results are bit-identical to attn_core.cuh and
// the two kernels are interchangeable) but:
//
//   * one thread-block CLUSTER of C CTAs per row (group g, kv head h); CTA r
//     of the cluster owns KV pages r, r + C, r + 2C, ... of the row;
//   * every CTA issues the bulk copies (UBLKCP, one mbarrier per ring slot)
//     of its first pages BEFORE griddepcontrol.wait when they hold no
//     position this layer's QKV kernel writes, so the K/V fetch overlaps the
//     previous kernel's tail; the row's newest page follows the wait;
//   * all query vectors of the group (nv consecutive positions, a folded
//     deep batch or an EESD verify) are scored against each K/V page while
//     it is in shared memory: K/V cross HBM once per row, not once per vector;
//   * per-page partials (m, l, o[hd]) stay in the owning CTA's shared memory;
//     after one cluster barrier each CTA merges rows r = cluster rank, +C,
//     ... reading the peers' partials over DSMEM in page order (no global
//     partials, no atomics), and writes o;
//   * the grid is sized to the rows (rows x C CTAs), not to the SM count.
//
// Per-page arithmetic (must match attn_core.cuh bit for bit):
//   scores  : LPT lanes per token, fmaf over the lane's 16-byte K vector in
//             element order, xor-butterfly over the LPT lanes, x scale;
//   softmax : warp max, p = expf(s - max), per-lane sums over tokens lane,
//             lane+32 then warp_sum;
//   PV      : acc = sum over tokens in order of fmaf(p, v, acc);
//   merge   : M = max_c m_c, e_c = expf(m_c - M), L = warp_sum of per-lane
//             fmaf(l_c, e_c, 0), O = sum over pages in order of
//             fmaf(o_c, e_c, O), o = O / L.
#include <cooperative_groups.h>

#include <algorithm>
#include <type_traits>

#include "attn_core.cuh"

namespace cg = cooperative_groups;

namespace ppsd {

constexpr int kDecRowsChunk = 16;  // query rows scored together (registers)
constexpr int kDecMaxWorkers = 4;  // 128-thread page workers per CTA (128 registers per thread)

struct DecLayout {  // dynamic shared memory carve-up, identical on host and device
  size_t ring, sc, qs, part, se, total;
};

// W workers per CTA, C CTAs per cluster (pages C*W), qmax query rows
template <int HD, typename KVT>
__host__ __device__ inline DecLayout dec_layout(int W, int C, int qmax) {
  DecLayout L;
  const size_t page = 2 * (size_t)kPage * HD * sizeof(KVT);  // K block + V block
  const int rc = qmax < kDecRowsChunk ? qmax : kDecRowsChunk;
  L.ring = 0;
  L.sc = L.ring + (size_t)W * page;
  L.qs = L.sc + (size_t)W * rc * kPage * sizeof(float);
  L.part = L.qs + (size_t)qmax * HD * sizeof(float);
  L.se = L.part + (size_t)C * W * qmax * (HD + 2) * sizeof(float);
  L.total = L.se + (size_t)qmax * (kMergePages + 1) * sizeof(float);
  return L;
}

// One worker (128 threads, named barrier `wbar`) runs rows r0 .. r0+RC
// (RC <= RCT) of its page: scores, chunk-local softmax, PV, and pushes the
// partials (o[HD], m, l) of the rows whose context reaches the page into the
// cluster leader's shared memory `pdst` ([page][qmax][HD + 2]). Row q's
// context in the page is nq[q] tokens (attn_core.cuh arithmetic per row).
template <int HD, typename KVT, int RCT>
__device__ __forceinline__ void page_rows(const KVT* ks, const KVT* vs, const float* qs, float* sc, float* s_m,
                                          float* s_l, float* pdst, int r0, int RC, int nmax, const int (&nq)[RCT],
                                          const int* s_nq, int wt, int lane, int wbar, float scale) {
  constexpr int EPV = 16 / (int)sizeof(KVT);
  constexpr int LPT = HD / EPV;
  constexpr int TPW = 32 / LPT;
  const int wwarp = wt >> 5;
  const int li = lane % LPT, tw = lane / LPT;
  for (int base = wwarp * TPW; base < nmax; base += 4 * TPW) {
    const int tt = base + tw;
    float kf[EPV];
    if (tt < nmax) unpack16<KVT>(lds128(ks + (size_t)tt * HD + li * EPV), kf);
    float prt[RCT];
#pragma unroll
    for (int q = 0; q < RCT; ++q) {
      prt[q] = 0.f;
      if (q < RC && tt < nmax) {
        const float* qr = qs + (size_t)(r0 + q) * HD + li * EPV;
#pragma unroll
        for (int e = 0; e < EPV; ++e) prt[q] = fmaf(kf[e], qr[e], prt[q]);
      }
    }
#pragma unroll
    for (int off = LPT / 2; off > 0; off >>= 1)
#pragma unroll
      for (int q = 0; q < RCT; ++q) prt[q] += __shfl_xor_sync(0xffffffffu, prt[q], off);
    if (li == 0)
#pragma unroll
      for (int q = 0; q < RCT; ++q)
        if (tt < nq[q]) sc[q * kPage + tt] = prt[q] * scale;
  }
  named_bar_sync(wbar, kAttnThreads);
  for (int q = wwarp; q < RC; q += 4) {  // chunk-local softmax statistics
    const int n = s_nq[q];
    float* sr = sc + q * kPage;
    if (n <= 0) continue;  // the page is past this vector's context
    float mx = -FLT_MAX;
    for (int tt = lane; tt < n; tt += 32) mx = fmaxf(mx, sr[tt]);
    mx = warp_max(mx);
    float l = 0.f;
    for (int tt = lane; tt < n; tt += 32) {
      const float p = expf(sr[tt] - mx);
      sr[tt] = p;
      l += p;
    }
    l = warp_sum(l);
    if (lane == 0) { s_m[q] = mx; s_l[q] = l; }
  }
  named_bar_sync(wbar, kAttnThreads);
  // PV: thread wt owns dim d of every row; the rows' accumulators advance
  // together (ILP), each over its tokens in order
  for (int d = wt; d < HD; d += kAttnThreads) {
    float acc[RCT];
#pragma unroll
    for (int q = 0; q < RCT; ++q) acc[q] = 0.f;
#pragma unroll 4
    for (int tt = 0; tt < nmax; ++tt) {
      const float vv = tof(vs[(size_t)tt * HD + d]);
#pragma unroll
      for (int q = 0; q < RCT; ++q)
        if (tt < nq[q]) acc[q] = fmaf(sc[q * kPage + tt], vv, acc[q]);
    }
#pragma unroll
    for (int q = 0; q < RCT; ++q)
      if (nq[q] > 0) pdst[(size_t)(r0 + q) * (HD + 2) + d] = acc[q];
  }
  if (wt < RC && s_nq[wt] > 0) {
    pdst[(size_t)(r0 + wt) * (HD + 2) + HD] = s_m[wt];
    pdst[(size_t)(r0 + wt) * (HD + 2) + HD + 1] = s_l[wt];
  }
  named_bar_sync(wbar, kAttnThreads);
}

template <int HD, typename KVT, int RCT, class NF>
__device__ __forceinline__ void page_chunk(const KVT* ks, const KVT* vs, const float* qs, float* sc, float* s_m,
                                           float* s_l, int* s_nq, float* pdst, int r0, int RC, int nmax, NF nrow,
                                           int wt, int lane, int wbar, float scale) {
  int nq[RCT];
#pragma unroll
  for (int q = 0; q < RCT; ++q) nq[q] = q < RC ? nrow(r0 + q) : 0;
  if (wt < RC) s_nq[wt] = nrow(r0 + wt);  // read after the worker barrier below
  page_rows<HD, KVT, RCT>(ks, vs, qs, sc, s_m, s_l, pdst, r0, RC, nmax, nq, s_nq, wt, lane, wbar, scale);
}

template <int HD, typename KVT, int QPK>
__global__ void __launch_bounds__(kAttnThreads* kDecMaxWorkers) attn_decode_kernel(const AttnArgs a) {
  constexpr int BLK = kPage * HD;  // elements per K (or V) page block
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar[kDecMaxWorkers];
  __shared__ float s_m[kDecMaxWorkers][kDecRowsChunk], s_l[kDecMaxWorkers][kDecRowsChunk];
  __shared__ int s_nq[kDecMaxWorkers][kDecRowsChunk];

  cg::cluster_group cluster = cg::this_cluster();
  const int C = a.dec_c, W = a.dec_w, qmax = a.dec_qmax;
  const DecLayout lay = dec_layout<HD, KVT>(W, C, qmax);
  const int rcmax = qmax < kDecRowsChunk ? qmax : kDecRowsChunk;

  const int tid = threadIdx.x, lane = tid & 31;
  const int wk = tid >> 7, wt = tid & 127;  // page worker and its thread
  const int cr = (int)cluster.block_rank();
  const int row = (int)blockIdx.x / C;
  const int H = a.dm.H, KVh = a.dm.KV;
  const float scale = 1.0f / sqrtf((float)HD);
  const Work* w = a.work;

  // ---- row -> (group, kv head); the descriptor was written >= 2 kernels ago
  int g = -1, kvh = 0, r = row;
  for (int gg = 0; gg < w->G; ++gg) {
    if (w->slot[gg] < 0 || a.layer_i >= w->nl[gg]) continue;
    if (r < KVh) {
      g = gg;
      kvh = r;
      break;
    }
    r -= KVh;
  }
  if (g < 0) {  // idle row: the whole cluster leaves together
    pdl_wait();
    pdl_trigger();
    return;
  }
  const int pos0 = w->pos[g], nv = w->nv[g], slot0 = w->slot[g];
  const int Q = nv * QPK;
  const int nch = (pos0 + nv - 1 + kPage) / kPage;  // pages of the longest context
  const int c = wk * C + cr;                        // this worker's page
  const bool active = c < nch;
  const int nmax = active ? min(kPage, pos0 + nv - c * kPage) : 0;  // rows of the page, longest context
  auto nrow = [&](int q) { return min(kPage, pos0 + q / QPK + 1 - c * kPage); };
  const int gl = w->first[g] + a.layer_i;
  const int lloc = gl == a.hl_global ? a.hl_local : gl - a.first_local;
  const char* kvl = static_cast<const char*>(a.kv_base) + a.kv_layer_bytes * (2 * (size_t)lloc);
  KVT* ks = reinterpret_cast<KVT*>(smem + lay.ring) + (size_t)wk * 2 * BLK;
  const KVT* vs = ks + BLK;
  float* sc = reinterpret_cast<float*>(smem + lay.sc) + (size_t)wk * rcmax * kPage;
  float* qs = reinterpret_cast<float*>(smem + lay.qs);  // [Q][HD]
  // partials live in the cluster leader's shared memory: [page][qmax][HD + 2]
  float* part0 = cluster.map_shared_rank(reinterpret_cast<float*>(smem + lay.part), 0);

  if (wt == 0) {
    mbar_init(&bar[wk], 1);
    fence_mbar_init();
  }
  // DSMEM may be touched only once every CTA of the cluster runs: arrive now,
  // wait before the first push into the leader's shared memory
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  named_bar_sync(1 + wk, kAttnThreads);
  auto issue = [&]() {  // worker thread 0: the page's K and V blocks, one mbarrier
    const size_t blk = ((size_t)a.page_table[c] * KVh + kvh) * BLK;
    const uint32_t bytes = (uint32_t)(nmax * HD * sizeof(KVT));
    mbar_expect_tx(&bar[wk], 2 * bytes);
    bulk_g2s(ks, reinterpret_cast<const KVT*>(kvl) + blk, bytes, &bar[wk]);
    bulk_g2s(ks + BLK, reinterpret_cast<const KVT*>(kvl + a.kv_layer_bytes) + blk, bytes, &bar[wk]);
  };
  // a page entirely below the first position this layer's QKV kernel writes
  // is final: fetch it while the previous kernel drains
  const bool early = active && (c + 1) * kPage <= pos0;
  if (early && wt == 0) issue();
  pdl_wait();     // q and this layer's new K/V rows are visible from here on
  pdl_trigger();  // the O projection may start streaming its weights
  if (active && !early && wt == 0) issue();
  for (int i = tid; i < Q * HD; i += blockDim.x) {
    const int v = i / (QPK * HD), rem = i - v * QPK * HD;
    qs[i] = a.q[(size_t)(slot0 + v) * H * HD + (size_t)kvh * QPK * HD + rem];
  }
  __syncthreads();
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");

  if (active) {
    mbar_wait(&bar[wk], 0);
    float* pdst = part0 + (size_t)c * qmax * (HD + 2);
    for (int r0 = 0; r0 < Q; r0 += kDecRowsChunk) {
      const int RC = min(kDecRowsChunk, Q - r0);
      float* sm = s_m[wk];
      float* sl = s_l[wk];
      if (RC == 1) page_chunk<HD, KVT, 1>(ks, vs, qs, sc, sm, sl, s_nq[wk], pdst, r0, RC, nmax, nrow, wt, lane, 1 + wk, scale);
      else if (RC <= 2) page_chunk<HD, KVT, 2>(ks, vs, qs, sc, sm, sl, s_nq[wk], pdst, r0, RC, nmax, nrow, wt, lane, 1 + wk, scale);
      else if (RC <= 4) page_chunk<HD, KVT, 4>(ks, vs, qs, sc, sm, sl, s_nq[wk], pdst, r0, RC, nmax, nrow, wt, lane, 1 + wk, scale);
      else if (RC <= 8) page_chunk<HD, KVT, 8>(ks, vs, qs, sc, sm, sl, s_nq[wk], pdst, r0, RC, nmax, nrow, wt, lane, 1 + wk, scale);
      else page_chunk<HD, KVT, 16>(ks, vs, qs, sc, sm, sl, s_nq[wk], pdst, r0, RC, nmax, nrow, wt, lane, 1 + wk, scale);
    }
  }

  cluster.sync();  // every page partial of the row is in the leader's shared memory
  if (cr != 0) return;

  // ---- leader: merge each row over its pages in page order
  const float* part = reinterpret_cast<const float*>(smem + lay.part);
  float* se = reinterpret_cast<float*>(smem + lay.se);  // [Q][kMergePages] page weights, then [Q] sums
  const int nwarps = blockDim.x >> 5, warp = tid >> 5;
  for (int q = warp; q < Q; q += nwarps) {
    const int nq = (pos0 + q / QPK + kPage) / kPage;
    float mv = -FLT_MAX;
    for (int cc = lane; cc < nq; cc += 32) mv = fmaxf(mv, part[((size_t)cc * qmax + q) * (HD + 2) + HD]);
    mv = warp_max(mv);
    float Ls = 0.f;
    for (int cc = lane; cc < nq; cc += 32) {
      const float* pp = part + ((size_t)cc * qmax + q) * (HD + 2);
      const float e = expf(pp[HD] - mv);
      se[q * kMergePages + cc] = e;  // page weight
      Ls = fmaf(pp[HD + 1], e, Ls);
    }
    Ls = warp_sum(Ls);
    if (lane == 0) se[qmax * kMergePages + q] = Ls;
  }
  __syncthreads();
  for (int idx = tid; idx < Q * HD; idx += blockDim.x) {
    const int q = idx / HD, d = idx - q * HD;
    const int v = q / QPK, i = q - v * QPK;
    const int nq = (pos0 + v + kPage) / kPage;
    float O = 0.f;
    for (int cc = 0; cc < nq; ++cc) O = fmaf(part[((size_t)cc * qmax + q) * (HD + 2) + d], se[q * kMergePages + cc], O);
    a.o[(size_t)(slot0 + v) * H * HD + ((size_t)kvh * QPK + i) * HD + d] = O / se[qmax * kMergePages + q];
  }
}

namespace {
template <int HD, typename KVT, int QPK>
cudaError_t dec_launch_k(const AttnArgs& a, int rows, cudaStream_t st, bool attrs, size_t smem) {
  auto fn = attn_decode_kernel<HD, KVT, QPK>;
  if (attrs) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rows * a.dec_c);
  cfg.blockDim = dim3(kAttnThreads * a.dec_w);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = a.dec_c;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, fn, a);
}
template <int HD, typename KVT>
cudaError_t dec_launch_q(const AttnArgs& a, int rows, cudaStream_t st, bool attrs, size_t smem) {
  switch (a.dm.H / a.dm.KV) {
    case 1: return dec_launch_k<HD, KVT, 1>(a, rows, st, attrs, smem);
    case 2: return dec_launch_k<HD, KVT, 2>(a, rows, st, attrs, smem);
    case 4: return dec_launch_k<HD, KVT, 4>(a, rows, st, attrs, smem);
    case 8: return dec_launch_k<HD, KVT, 8>(a, rows, st, attrs, smem);
  }
  return cudaErrorInvalidValue;
}
template <int HD>
cudaError_t dec_launch_h(const AttnArgs& a, int rows, cudaStream_t st, bool attrs, size_t smem) {
  return a.dm.kv_bf16 ? dec_launch_q<HD, __nv_bfloat16>(a, rows, st, attrs, smem)
                      : dec_launch_q<HD, float>(a, rows, st, attrs, smem);
}
cudaError_t dec_dispatch(const AttnArgs& a, int rows, cudaStream_t st, bool attrs, size_t smem) {
  switch (a.dm.hd) {
    case 16: return dec_launch_h<16>(a, rows, st, attrs, smem);
    case 32: return dec_launch_h<32>(a, rows, st, attrs, smem);
    case 64: return dec_launch_h<64>(a, rows, st, attrs, smem);
    case 128: return dec_launch_h<128>(a, rows, st, attrs, smem);
  }
  return cudaErrorInvalidValue;
}
size_t dec_smem(const AttnArgs& a) {
  const int hd = a.dm.hd;
  auto f = [&](auto hdc, auto kvt) {
    constexpr int HDc = decltype(hdc)::value;
    using KVT = decltype(kvt);
    return dec_layout<HDc, KVT>(a.dec_w, a.dec_c, a.dec_qmax).total;
  };
  using I16 = std::integral_constant<int, 16>;
  using I32 = std::integral_constant<int, 32>;
  using I64 = std::integral_constant<int, 64>;
  using I128 = std::integral_constant<int, 128>;
  const bool b = a.dm.kv_bf16;
  switch (hd) {
    case 16: return b ? f(I16{}, __nv_bfloat16{}) : f(I16{}, 0.f);
    case 32: return b ? f(I32{}, __nv_bfloat16{}) : f(I32{}, 0.f);
    case 64: return b ? f(I64{}, __nv_bfloat16{}) : f(I64{}, 0.f);
    case 128: return b ? f(I128{}, __nv_bfloat16{}) : f(I128{}, 0.f);
  }
  return 0;
}
}  // namespace

// Plan a decode-attention launch for gmax * KV rows of up to nvmax query
// vectors each: one cluster of C CTAs per row, W 128-thread page workers per
// CTA, C * W >= the engine's pages. C is the largest power of two <= 8 with
// rows * C <= 2 CTAs per SM. Returns false when the plan does not fit (the
// caller then launches the split-K kernel, attn_core.cuh: same arithmetic).
bool attn_decode_plan(AttnArgs* a, int gmax, int nvmax, int num_sms) {
  const int rows = gmax * a->dm.KV;
  const int qpk = a->dm.H / a->dm.KV;
  if (nvmax < 1 || a->max_pages > kMergePages || a->max_pages < 1) return false;
  int C = 8;
  while (C > 1 && (rows * C > 2 * num_sms || C > a->max_pages)) C >>= 1;
  const int W = (a->max_pages + C - 1) / C;
  if (W > kDecMaxWorkers) return false;
  a->dec_c = C;
  a->dec_w = W;
  a->dec_qmax = nvmax * qpk;
  return dec_smem(*a) <= 220 * 1024;
}

// the dynamic shared-memory ceiling every plan stays under (attn_decode_plan)
cudaError_t attn_decode_set_attrs(const AttnArgs& a) { return dec_dispatch(a, 0, 0, true, 220 * 1024); }

cudaError_t attn_decode_launch(const AttnArgs& a, int rows, cudaStream_t st) {
  return dec_dispatch(a, rows, st, false, dec_smem(a));
}

}  // namespace ppsd
