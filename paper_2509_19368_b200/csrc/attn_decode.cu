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

struct DecLayout {  // dynamic shared memory carve-up, identical on host and device
  size_t ring, part, qs, sc, total;
};

template <int HD, typename KVT>
__host__ __device__ inline DecLayout dec_layout(int nb, int ppc, int qmax) {
  DecLayout L;
  const size_t page = 2 * (size_t)kPage * HD * sizeof(KVT);  // K block + V block
  L.ring = 0;
  L.part = L.ring + (size_t)nb * page;
  L.qs = L.part + (size_t)ppc * qmax * (HD + 2) * sizeof(float);
  L.sc = L.qs + (size_t)qmax * HD * sizeof(float);
  L.total = L.sc + (size_t)kDecRowsChunk * kPage * sizeof(float);
  return L;
}

template <int HD, typename KVT, int QPK>
__global__ void __launch_bounds__(kAttnThreads) attn_decode_kernel(const AttnArgs a) {
  constexpr int EPV = 16 / (int)sizeof(KVT);  // elements per 16-byte vector
  constexpr int LPT = HD / EPV;                // lanes per token
  constexpr int TPW = 32 / LPT;                // tokens per warp pass
  constexpr int BLK = kPage * HD;              // elements per K (or V) page block
  static_assert(LPT >= 1 && LPT <= 32 && (32 % LPT) == 0, "head_dim / dtype combination");
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar[4];
  __shared__ float s_m[kDecRowsChunk], s_l[kDecRowsChunk];
  __shared__ float s_e[kMergePages];
  __shared__ float s_L;

  cg::cluster_group cluster = cg::this_cluster();
  const int C = a.dec_c, nb = a.dec_nb, ppc = a.dec_ppc, qmax = a.dec_qmax;
  const DecLayout lay = dec_layout<HD, KVT>(nb, ppc, qmax);
  KVT* ring = reinterpret_cast<KVT*>(smem + lay.ring);
  float* part = reinterpret_cast<float*>(smem + lay.part);  // [ppc][qmax][HD + 2]
  float* qs = reinterpret_cast<float*>(smem + lay.qs);      // [qmax][HD]
  float* sc = reinterpret_cast<float*>(smem + lay.sc);      // [kDecRowsChunk][kPage]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
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
  const int my_n = cr < nch ? (nch - 1 - cr) / C + 1 : 0;  // pages this CTA owns
  const int gl = w->first[g] + a.layer_i;
  const int lloc = gl == a.hl_global ? a.hl_local : gl - a.first_local;
  const char* kvl = static_cast<const char*>(a.kv_base) + a.kv_layer_bytes * (2 * (size_t)lloc);

  if (tid == 0) {
    for (int i = 0; i < nb; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // page j of this CTA (global page cr + j*C), into ring slot j % nb
  auto issue = [&](int j) {
    const int c = cr + j * C;
    const int n = min(kPage, pos0 + nv - c * kPage);  // rows of the page in the longest context
    const int page = a.page_table[c];
    const size_t blk = ((size_t)page * KVh + kvh) * BLK;
    const uint32_t bytes = (uint32_t)(n * HD * sizeof(KVT));
    KVT* ks = ring + (size_t)(j % nb) * 2 * BLK;
    mbar_expect_tx(&bar[j % nb], 2 * bytes);
    bulk_g2s(ks, reinterpret_cast<const KVT*>(kvl) + blk, bytes, &bar[j % nb]);
    bulk_g2s(ks + BLK, reinterpret_cast<const KVT*>(kvl + a.kv_layer_bytes) + blk, bytes, &bar[j % nb]);
  };
  // a page entirely below the first position this layer's QKV kernel writes is final
  int issued = 0;
  if (tid == 0)
    while (issued < min(my_n, nb) && (cr + issued * C + 1) * kPage <= pos0) issue(issued++);
  pdl_wait();     // q and this layer's new K/V rows are visible from here on
  pdl_trigger();  // the O projection may start streaming its weights
  if (tid == 0)
    while (issued < min(my_n, nb)) issue(issued++);
  for (int i = tid; i < Q * HD; i += kAttnThreads) {
    const int v = i / (QPK * HD), rem = i - v * QPK * HD;
    qs[i] = a.q[(size_t)(slot0 + v) * H * HD + (size_t)kvh * QPK * HD + rem];
  }
  __syncthreads();

  const int li = lane % LPT, tw = lane / LPT;
  for (int j = 0; j < my_n; ++j) {
    const int c = cr + j * C;
    mbar_wait(&bar[j % nb], (j / nb) & 1);
    const KVT* ks = ring + (size_t)(j % nb) * 2 * BLK;
    const KVT* vs = ks + BLK;
    float* pj = part + (size_t)j * qmax * (HD + 2);
    for (int r0 = 0; r0 < Q; r0 += kDecRowsChunk) {
      const int RC = min(kDecRowsChunk, Q - r0);
      const int nmax = min(kPage, pos0 + nv - c * kPage);
      // scores (rows r0 .. r0+RC of this chunk; row r = vector r / QPK)
      for (int base = warp * TPW; base < nmax; base += 4 * TPW) {
        const int tt = base + tw;
        float kf[EPV];
        if (tt < nmax) unpack16<KVT>(lds128(ks + (size_t)tt * HD + li * EPV), kf);
        float prt[kDecRowsChunk];
#pragma unroll
        for (int q = 0; q < kDecRowsChunk; ++q) {
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
          for (int q = 0; q < kDecRowsChunk; ++q) prt[q] += __shfl_xor_sync(0xffffffffu, prt[q], off);
        if (li == 0)
#pragma unroll
          for (int q = 0; q < kDecRowsChunk; ++q) {
            if (q >= RC) break;
            const int n = min(kPage, pos0 + (r0 + q) / QPK + 1 - c * kPage);
            if (tt < n) sc[q * kPage + tt] = prt[q] * scale;
          }
      }
      __syncthreads();
      for (int q = warp; q < RC; q += 4) {  // chunk-local softmax statistics
        const int n = min(kPage, pos0 + (r0 + q) / QPK + 1 - c * kPage);
        float* sr = sc + q * kPage;
        if (n <= 0) {
          if (lane == 0) { s_m[q] = -FLT_MAX; s_l[q] = 0.f; }
          continue;
        }
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
      __syncthreads();
      for (int idx = tid; idx < RC * HD; idx += kAttnThreads) {
        const int q = idx / HD, d = idx - q * HD;
        const int n = min(kPage, pos0 + (r0 + q) / QPK + 1 - c * kPage);
        float acc = 0.f;
#pragma unroll 8
        for (int tt = 0; tt < n; ++tt) acc = fmaf(sc[q * kPage + tt], tof(vs[(size_t)tt * HD + d]), acc);
        pj[(size_t)(r0 + q) * (HD + 2) + d] = acc;
      }
      if (tid < RC) {
        pj[(size_t)(r0 + tid) * (HD + 2) + HD] = s_m[tid];
        pj[(size_t)(r0 + tid) * (HD + 2) + HD + 1] = s_l[tid];
      }
      __syncthreads();
    }
    // refill this ring slot with the page nb ahead (its reads are done)
    if (tid == 0 && j + nb < my_n) issue(j + nb);
  }

  cluster.sync();  // every page partial of the row is in some CTA's shared memory

  // ---- merge rows cr, cr + C, ... in page order over DSMEM
  for (int q = cr; q < Q; q += C) {
    const int v = q / QPK, i = q - v * QPK;
    const int nq = (pos0 + v + kPage) / kPage;  // pages of this vector's context
    auto pptr = [&](int cc) {                    // partial row of page cc (peer smem)
      float* base = cluster.map_shared_rank(part, cc % C);
      return base + ((size_t)(cc / C) * qmax + q) * (HD + 2);
    };
    if (warp == 0) {
      float mv = -FLT_MAX;
      for (int cc = lane; cc < nq; cc += 32) mv = fmaxf(mv, pptr(cc)[HD]);
      mv = warp_max(mv);
      float Ls = 0.f;
      for (int cc = lane; cc < nq; cc += 32) {
        const float* pp = pptr(cc);
        const float e = expf(pp[HD] - mv);
        s_e[cc] = e;  // page weight
        Ls = fmaf(pp[HD + 1], e, Ls);
      }
      Ls = warp_sum(Ls);
      if (lane == 0) s_L = Ls;
    }
    __syncthreads();
    for (int d = tid; d < HD; d += kAttnThreads) {
      float pv[kMergePages];
#pragma unroll
      for (int cc = 0; cc < kMergePages; ++cc)
        if (cc < nq) pv[cc] = pptr(cc)[d];
      float O = 0.f;
#pragma unroll
      for (int cc = 0; cc < kMergePages; ++cc)
        if (cc < nq) O = fmaf(pv[cc], s_e[cc], O);
      a.o[(size_t)(slot0 + v) * H * HD + ((size_t)kvh * QPK + i) * HD + d] = O / s_L;
    }
    __syncthreads();
  }
  cluster.sync();  // peers may still read this CTA's partials
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
  cfg.blockDim = dim3(kAttnThreads);
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
    return dec_layout<HDc, KVT>(a.dec_nb, a.dec_ppc, a.dec_qmax).total;
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

// Plan a decode-attention launch for rows = gmax * KV rows of up to nvmax
// query vectors each: cluster size C (largest power of two <= 8 keeping
// rows * C within two CTAs per SM and C <= pages), pages per CTA, ring depth.
// Returns false when the plan does not fit shared memory (the caller then
// launches the split-K kernel, attn_core.cuh: same arithmetic).
bool attn_decode_plan(AttnArgs* a, int gmax, int nvmax, int num_sms) {
  const int rows = gmax * a->dm.KV;
  const int qpk = a->dm.H / a->dm.KV;
  if (nvmax < 1 || a->max_pages > kMergePages || a->max_pages < 1) return false;
  int C = 8;
  while (C > 1 && (rows * C > 2 * num_sms || C > a->max_pages)) C >>= 1;
  a->dec_c = C;
  a->dec_ppc = (a->max_pages + C - 1) / C;
  a->dec_qmax = nvmax * qpk;
  for (int nb = std::min(a->dec_ppc, 3); nb >= 1; --nb) {
    a->dec_nb = nb;
    if (dec_smem(*a) <= 220 * 1024) return true;
  }
  return false;
}

// the dynamic shared-memory ceiling every plan stays under (attn_decode_plan)
cudaError_t attn_decode_set_attrs(const AttnArgs& a) { return dec_dispatch(a, 0, 0, true, 220 * 1024); }

cudaError_t attn_decode_launch(const AttnArgs& a, int rows, cudaStream_t st) {
  return dec_dispatch(a, rows, st, false, dec_smem(a));
}

}  // namespace ppsd
