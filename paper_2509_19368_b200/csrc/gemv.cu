// gemv.cu — weight-streaming GEMV for bs=1 decode on sm_100a.
//
// Every decode-step matmul is y = W x with W bf16 [R][K] streamed from HBM
// exactly once and x a handful of fp32 vectors; the roofline is HBM bytes.
// One persistent CTA per SM (grid = #SMs, ~200 KB smem):
//
//   warp 8 (producer, one lane): cp.async.bulk (UBLKCP) of up to SUB
//       tiles of TR contiguous weight rows (48-96 KB per copy — measured: the
//       per-SM bulk-copy engine needs few, large copies in flight; a stage
//       never spans two problems) into an NS-deep smem ring, completion
//       counted on per-stage mbarriers (expect_tx), L2 evict_first. TR is
//       what the consumers' registers allow (fewer rows when M vectors'
//       input slices live there too); SUB restores the copy size.
//   warps 0-7 (consumers, 256 threads): thread t owns the 16-byte column
//       vectors t, t+256, ... of every row; its slice of the normalised input
//       vector lives in registers for the whole kernel. Per stage it issues
//       all TR x VPT ld.shared.v4 at once, releases the stage back to the
//       producer immediately (early release keeps the ring full), then does
//       the FMAs and ONE transpose-butterfly that reduces all M x TR row
//       partials of the warp in N-1+5-log2(N) shuffles.
//
// Programmatic dependent launch: the producer starts streaming weights
// before the previous kernel of the step has finished (weights never depend
// on it); consumers wait (griddepcontrol.wait) before touching activations.
// The per-tick work descriptor is read early except by the first layer
// kernel after the scheduler (desc_early == 0).
//
// The tile space of ALL active problems of one launch (the same layer slot of
// every pipeline stage with a chain this tick — the grouped launch through
// which the stages on one GPU share the SMs) is split into contiguous ranges,
// one per CTA. Row results never depend on the split, the group count or M,
// so PPSD and autoregressive decoding produce bit-identical hidden states.
//
// Fused epilogues (the op that follows each matmul in the decoder layer):
//   kMatQKV  : RMSNorm prologue; RoPE on (q,k) row pairs; q -> scratch,
//              k,v -> paged KV cache at the chain's position.
//   kMatGU   : RMSNorm prologue; SwiGLU on (gate,up) row pairs -> h.
//   kMatO / kMatDown : residual add into the chain's fp32 hidden state.
//   kMatHead : per-vector RMSNorm prologue (exit norm | final norm); M=2
//              vectors share one pass over the tied LM head; fp32 logits and
//              a deterministic first-index argmax across CTAs.
#include <float.h>
#include <limits.h>

#include "kernels.cuh"

namespace ppsd {

__device__ __forceinline__ bool better(float v, int i, float bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

// d = a * b on both lanes (mul.rn.f32x2, sm_100: FMUL2)
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mul.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// d = a * b + c on both lanes (fma.rn.f32x2, sm_100: FFMA2)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
      " mov.b64 rc, {%6, %7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// Reduce N per-lane values across the warp. Afterwards lane L holds the
// warp total of value index L >> (5 - log2 N). Fixed shuffle tree: the
// result is deterministic.
template <int N>
__device__ __forceinline__ float transpose_reduce(float (&v)[N], int lane) {
  static_assert((N & (N - 1)) == 0 && N <= 32, "N must be a power of two <= 32");
  int cnt = N;
  int off = 16;
#pragma unroll
  for (int step = 0; step < ilog2(N); ++step) {
    const int half = cnt >> 1;
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      if (i < half) {
        const float keep = upper ? v[i + half] : v[i];
        const float send = upper ? v[i] : v[i + half];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    cnt = half;
    off >>= 1;
  }
  float s = v[0];
#pragma unroll
  for (int o = 16 >> ilog2(N); o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Consumer warps per CTA. A matrix must use the same NW (and so the same
// per-row reduction tree) in every plan. Measured: 16 warps at K <= 8192
// (VPT 1-2) did not beat 8 warps with twice the columns per thread (the
// batched plans got slower: fewer rows per tile fit in 120 registers), so
// every plan uses 8.
constexpr int nw_for(int /*vpt*/) { return 8; }

// Register boost for the batched plans of wide-K matrices (VPT >= 3: K >
// 4096): their M=4 input slices need ~170-230 registers per thread, but 9
// warps cap every thread at 168 (allocation granularity is 4 warps). Those
// instantiations run a 4-warp producer warpgroup that hands its registers
// to the consumers (setmaxnreg). Measured: the boost made the K = 4096
// (VPT 2) batched plans slower, so they keep 9 warps; without it the 13B
// (K = 5120) and 70B (K = 8192) 4-vector plans spilled 100-480 bytes, the
// 70B split down projection's 2-vector plans (K/2 = 14336) 260-400.
template <int VPT, int M, int EPI = -1>
constexpr bool reg_boost() { return (VPT >= 3 && M >= 4) || (VPT >= 7 && M >= 2); }
template <int VPT, int M, int EPI = -1>
constexpr int gemv_threads() { return (nw_for(VPT) + (reg_boost<VPT, M, EPI>() ? 4 : 1)) * 32; }

template <int VPT, int TR, int M, int EPI>
__global__ void __launch_bounds__(gemv_threads<VPT, M, EPI>(), 1) gemv_kernel(const GemvArgs a) {
  constexpr int NW = nw_for(VPT);  // consumer warps
  constexpr int NC = NW * 32;      // consumer threads
  constexpr bool kHead2 = EPI == kMatHead;   // PPSD tick: exit (m=0) + final (m=1) head
  constexpr bool kHeadV = EPI == kMatHeadV;  // final head on the vectors of group 0
  constexpr bool kHead = kHead2 || kHeadV;
  constexpr bool kDown = EPI == kMatDown || EPI == kMatDownS;
  constexpr bool ksplit = EPI == kMatDownS;  // K split across the grid halves
  // M = 1 and the tick head: all loads of a tile first, release the stage,
  // then the math (the ring refills during it). Batched plans: weights are
  // loaded as the FMAs need them, so no register copy of the tile bounds TR,
  // and the stage is released after its last tile (SUB >= 2 keeps the ring
  // deep enough).
  constexpr bool kLoadsFirst = M == 1 || kHead2;
  // batched plans pair vectors (m, m+1) in FFMA2s; their partials are kept
  // pair-adjacent: value index of (vector m, row r) in acc / red
  constexpr bool kPairs = M >= 2 && !kHead2;
  auto vidx = [](int m, int r) { return kPairs ? ((m >> 1) * TR + r) * 2 + (m & 1) : m * TR + r; };
  constexpr int NV = M * TR;                 // row partials per thread per stage
  constexpr int CHT = ((NW == 16 ? 64 : 128) / TR) < 1 ? 1 : ((NW == 16 ? 64 : 128) / TR);  // tiles per epilogue
  constexpr int kMaxProb = 128;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ int s_pg[kMaxProb], s_pv[kMaxProb];  // problem = (group, first vector)
  __shared__ int s_np;
  __shared__ float s_ss[NW][M];
  __shared__ float s_bv[NW][M];
  __shared__ int s_bi[NW][M];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = a.K, R = a.R, NS = a.nstage, SUB = a.sub;
  const int tile_bytes = TR * K * 2;
  const int stage_bytes = SUB * tile_bytes;
  unsigned char* ring = smem;
  float* red = reinterpret_cast<float*>(smem + (size_t)NS * stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(red + CHT * NW * NV);
  uint64_t* empty = full + NS;
  const Work* work = a.work;

  if (!a.desc_early) pdl_wait();
  if (tid == 0) {
    int np = 0;
    if (kHead2) {
      if (work->head_slot[0] >= 0 || work->head_slot[1] >= 0) { s_pg[0] = -1; s_pv[0] = 0; np = 1; }
    } else if (kHeadV) {
      if (work->G >= 1 && work->slot[0] >= 0)
        for (int v0 = 0; v0 < work->nv[0] && np < kMaxProb; v0 += M) { s_pg[np] = 0; s_pv[np++] = v0; }
    } else {
      for (int g = 0; g < work->G; ++g)
        if (work->slot[g] >= 0 && a.layer_i < work->nl[g])
          for (int v0 = 0; v0 < work->nv[g] && np < kMaxProb; v0 += M) { s_pg[np] = g; s_pv[np++] = v0; }
    }
    s_np = np;
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int np = s_np;
  if (np == 0) {
    pdl_wait();
    pdl_trigger();
    return;
  }
  const int tpp = R / TR;
  // K split: CTA kb of each grid half takes the same tiles, column half kh.
  // The publishing half (kh = 1) has the LOW block indices so it is
  // dispatched first: a waiting CTA's partner is then already resident.
  const int kG = ksplit ? (int)gridDim.x / 2 : (int)gridDim.x;
  const int kh = ksplit && (int)blockIdx.x < kG ? 1 : 0;
  const int kb = ksplit ? (int)blockIdx.x - (kh ? 0 : kG) : (int)blockIdx.x;
  long long t0, t1;
  int hv_p = 0, hv_c0 = 0, hv_c1 = 0;  // kHeadV: this CTA's problem and its CTA span
  if (kHeadV) {
    // CTAs are split between problems so no CTA spans two vector chunks
    const int G = gridDim.x, b = blockIdx.x;
    while (hv_p + 1 < np && (hv_p + 1) * G / np <= b) ++hv_p;
    hv_c0 = hv_p * G / np;
    hv_c1 = (hv_p + 1) * G / np;
    const int nc = hv_c1 - hv_c0, bl = b - hv_c0;
    t0 = (long long)hv_p * tpp + (long long)tpp * bl / nc;
    t1 = (long long)hv_p * tpp + (long long)tpp * (bl + 1) / nc;
  } else {
    const long long T = (long long)np * tpp;
    t0 = T * kb / kG;
    t1 = T * (kb + 1) / kG;
  }
  const int ntiles = (int)(t1 - t0);

  if (warp >= NW) {  // ---------------- producer ----------------
    if constexpr (reg_boost<VPT, M, EPI>()) setmaxnreg_dec<40>();
    if (warp == NW && lane == 0 && ntiles > 0) {
      const uint64_t pol = policy_evict_first();
      int cur_p = -1;
      const unsigned char* wb = nullptr;
      for (int n = 0, j = 0; n < ntiles; ++j) {
        const long long t = t0 + n;
        const int p = (int)(t / tpp);
        const int tile = (int)(t - (long long)p * tpp);
        const int cnt = min(SUB, min(ntiles - n, tpp - tile));  // stage = tiles of one problem
        if (p != cur_p) {
          const __nv_bfloat16* w;
          if (kHead) {
            w = a.head_w;
          } else {
            const LayerW& L = a.layers[work->first[s_pg[p]] + a.layer_i];
            w = EPI == kMatQKV ? L.qkv : EPI == kMatO ? L.o : EPI == kMatGU ? L.gu : L.down;  // kDown
          }
          wb = reinterpret_cast<const unsigned char*>(w);
          cur_p = p;
        }
        const int st = j % NS;
        if (j >= NS) mbar_wait(&empty[st], ((j / NS) & 1) ^ 1);
        mbar_expect_tx(&full[st], cnt * tile_bytes);
        if (ksplit) {  // this half's columns of each row: one copy per row
          const unsigned char* src = wb + ((size_t)tile * TR * a.k_ld + (size_t)kh * K) * 2;
          for (int r = 0; r < cnt * TR; ++r)
            bulk_g2s(ring + (size_t)st * stage_bytes + (size_t)r * K * 2, src + (size_t)r * a.k_ld * 2, K * 2,
                     &full[st], pol);
        } else {
          bulk_g2s(ring + (size_t)st * stage_bytes, wb + (size_t)tile * tile_bytes, cnt * tile_bytes, &full[st],
                   pol);
        }
        n += cnt;
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  if constexpr (reg_boost<VPT, M, EPI>()) setmaxnreg_inc<232>();
  pdl_wait();     // activations of the previous kernel are visible from here on
  pdl_trigger();  // ...so the next kernel may start streaming its weights
  float bestv[M];
  int besti[M];
  bool mact[M];
  int vslot[M], vpos[M];  // per vector of the current problem
#pragma unroll
  for (int m = 0; m < M; ++m) {
    bestv[m] = -FLT_MAX;
    besti[m] = INT_MAX;
    mact[m] = false;
    vslot[m] = vpos[m] = 0;
  }
  int cur_v0 = 0;
  int chunk_n0 = 0;  // first tile of the current (not yet flushed) epilogue chunk
  int sj = -1, s_off = 0, s_cnt = 0;  // ring stage, tile within it, its tile count
  int nchunk = 0;                     // K split: epilogue chunks so far (flag index)

  if (ntiles > 0) {
    const int nvec = K >> 3;
    // shared-memory addressing, fixed per thread: column vector tid + u*256
    const uint32_t ring_s = smem_u32(ring);
    const int K2 = K * 2;
    uint32_t colb[VPT];
    bool cvalid[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      colb[u] = (uint32_t)(tid + u * NC) * 16u;
      cvalid[u] = tid + u * NC < nvec;
    }
    // input slices: vectors (m, m+1) share a float2 so the FMAs of a vector
    // pair issue as one FFMA2 (fma.rn.f32x2: two independent fma.rn.f32,
    // bit-identical to the scalar sequence)
    float2 xr2[(M + 1) / 2][VPT][8];
#define XR(m, u, e) (((m) & 1) ? xr2[(m) >> 1][u][e].y : xr2[(m) >> 1][u][e].x)
    int cur_p = -1;
    int p = (int)(t0 / tpp);                 // problem of the current tile
    int tip = (int)(t0 - (long long)p * tpp);  // tile index inside it
    for (int n = 0; n < ntiles; ++n) {
      if (p != cur_p) {  // load + normalise this problem's input vectors
        cur_p = p;
        const float* nw[M];
        const float* src[M];
        const int g = s_pg[p];
        cur_v0 = s_pv[p];
#pragma unroll
        for (int m = 0; m < M; ++m) {
          nw[m] = nullptr;
          src[m] = nullptr;
          if (kHead2) {
            const int s = work->head_slot[m];
            mact[m] = s >= 0;
            vslot[m] = s;
            nw[m] = m == 0 ? a.head_norm0 : a.head_norm1;
            src[m] = s >= 0 ? a.x + (size_t)s * a.dm.d : nullptr;
          } else {
            mact[m] = cur_v0 + m < work->nv[g];
            vslot[m] = work->slot[g] + cur_v0 + m;
            vpos[m] = work->pos[g] + cur_v0 + m;
            if (!mact[m]) continue;
            const int s = vslot[m];
            if (kHeadV) {
              src[m] = a.x + (size_t)s * a.dm.d;
              nw[m] = a.head_norm1;
            } else {
              const LayerW& L = a.layers[work->first[g] + a.layer_i];
              if (EPI == kMatQKV) { src[m] = a.x + (size_t)s * a.dm.d; nw[m] = L.attn_norm; }
              if (EPI == kMatGU) { src[m] = a.x + (size_t)s * a.dm.d; nw[m] = L.mlp_norm; }
              if (EPI == kMatO) src[m] = a.o + (size_t)s * a.dm.H * a.dm.hd;
              if (kDown) src[m] = a.h + (size_t)s * a.dm.ffn + (size_t)kh * K;
            }
          }
        }
#pragma unroll
        for (int m = 0; m < M; ++m) {
          float ss = 0.f;
#pragma unroll
          for (int u = 0; u < VPT; ++u) {
            const int v = tid + u * NC;
            if (src[m] && v < nvec) {
              const float4 lo = *reinterpret_cast<const float4*>(src[m] + v * 8);
              const float4 hi = *reinterpret_cast<const float4*>(src[m] + v * 8 + 4);
              XR(m, u, 0) = lo.x; XR(m, u, 1) = lo.y; XR(m, u, 2) = lo.z; XR(m, u, 3) = lo.w;
              XR(m, u, 4) = hi.x; XR(m, u, 5) = hi.y; XR(m, u, 6) = hi.z; XR(m, u, 7) = hi.w;
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) XR(m, u, e) = 0.f;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) ss = fmaf(XR(m, u, e), XR(m, u, e), ss);
          }
          ss = warp_sum(ss);
          if (lane == 0) s_ss[warp][m] = ss;
        }
        named_bar_sync(1, NC);
#pragma unroll
        for (int m = 0; m < M; ++m) {
          if (!nw[m]) continue;
          float tot = 0.f;
#pragma unroll
          for (int w = 0; w < NW; ++w) tot += s_ss[w][m];
          const float rstd = 1.0f / sqrtf(tot / (float)K + a.dm.eps);
#pragma unroll
          for (int u = 0; u < VPT; ++u) {
            const int v = tid + u * NC;
            if (v < nvec) {
              const float4 w0 = *reinterpret_cast<const float4*>(nw[m] + v * 8);
              const float4 w1 = *reinterpret_cast<const float4*>(nw[m] + v * 8 + 4);
              const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
              for (int e = 0; e < 8; ++e) XR(m, u, e) = (XR(m, u, e) * rstd) * wv[e];
            }
          }
        }
        named_bar_sync(1, NC);
      }

      // ---- tile: all shared loads first, release the stage after its last
      // tile's loads, then math ----
      if (s_off == s_cnt) {  // next ring stage (same partition rule as the producer)
        ++sj;
        s_off = 0;
        s_cnt = min(SUB, min(ntiles - n, tpp - tip));
        mbar_wait(&full[sj % NS], (sj / NS) & 1);
      }
      const int st = sj % NS;
      const uint32_t tb_s = ring_s + (uint32_t)(st * stage_bytes + s_off * tile_bytes);
      auto wload = [&](int r, int u) {
        return cvalid[u] ? lds128s(tb_s + (uint32_t)(r * K2) + colb[u]) : make_uint4(0, 0, 0, 0);
      };
      uint4 wv[kLoadsFirst ? TR : 1][VPT];
      if constexpr (kLoadsFirst) {
#pragma unroll
        for (int r = 0; r < TR; ++r)
#pragma unroll
          for (int u = 0; u < VPT; ++u) wv[r][u] = wload(r, u);
        __syncwarp();
        if (++s_off == s_cnt && lane == 0) mbar_arrive(&empty[st]);
      }
      // Every accumulator starts with the product of its first (u, e) term
      // and adds the rest in (u, e) order in all three forms below, so row
      // results do not depend on M, TR or the form.
      float acc[NV];
      if constexpr (kPairs) {  // vector pairs: one FFMA2 per weight and pair
        float2 ap[M / 2][TR];
#pragma unroll
        for (int r = 0; r < TR; ++r) {
#pragma unroll
          for (int u = 0; u < VPT; ++u) {
            const uint4 w = kLoadsFirst ? wv[kLoadsFirst ? r : 0][u] : wload(r, u);
            const float wf[8] = {bf16lo(w.x), bf16hi(w.x), bf16lo(w.y), bf16hi(w.y),
                                 bf16lo(w.z), bf16hi(w.z), bf16lo(w.w), bf16hi(w.w)};
#pragma unroll
            for (int mp = 0; mp < M / 2; ++mp) {
              if (!mact[2 * mp]) {  // batched plans: active vectors are a prefix
                if (u == 0) ap[mp][r] = make_float2(0.f, 0.f);
                continue;
              }
#pragma unroll
              for (int e = 0; e < 8; ++e)
                ap[mp][r] = (u == 0 && e == 0) ? fmul2(make_float2(wf[e], wf[e]), xr2[mp][u][e])
                                               : ffma2(make_float2(wf[e], wf[e]), xr2[mp][u][e], ap[mp][r]);
            }
          }
        }
        if constexpr (!kLoadsFirst) {
          __syncwarp();
          if (++s_off == s_cnt && lane == 0) mbar_arrive(&empty[st]);
        }
#pragma unroll
        for (int mp = 0; mp < M / 2; ++mp)
#pragma unroll
          for (int r = 0; r < TR; ++r) {
            acc[vidx(2 * mp, r)] = ap[mp][r].x;
            acc[vidx(2 * mp + 1, r)] = ap[mp][r].y;
          }
      } else if constexpr (M == 1 && TR % 2 == 0) {  // one vector: row pairs share an FFMA2
        float2 ap[TR / 2];
#pragma unroll
        for (int rp = 0; rp < TR / 2; ++rp) {
#pragma unroll
          for (int u = 0; u < VPT; ++u) {
            const uint4 w0 = wv[2 * rp][u], w1 = wv[2 * rp + 1][u];
            const float2 wf[8] = {
                make_float2(bf16lo(w0.x), bf16lo(w1.x)), make_float2(bf16hi(w0.x), bf16hi(w1.x)),
                make_float2(bf16lo(w0.y), bf16lo(w1.y)), make_float2(bf16hi(w0.y), bf16hi(w1.y)),
                make_float2(bf16lo(w0.z), bf16lo(w1.z)), make_float2(bf16hi(w0.z), bf16hi(w1.z)),
                make_float2(bf16lo(w0.w), bf16lo(w1.w)), make_float2(bf16hi(w0.w), bf16hi(w1.w))};
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const float xv = xr2[0][u][e].x;
              ap[rp] = (u == 0 && e == 0) ? fmul2(wf[e], make_float2(xv, xv))
                                          : ffma2(wf[e], make_float2(xv, xv), ap[rp]);
            }
          }
        }
#pragma unroll
        for (int rp = 0; rp < TR / 2; ++rp) {
          acc[2 * rp] = ap[rp].x;
          acc[2 * rp + 1] = ap[rp].y;
        }
      } else {  // scalar: TR = 1 rows, and the tick head (either vector may be idle)
#pragma unroll
        for (int r = 0; r < TR; ++r) {
#pragma unroll
          for (int u = 0; u < VPT; ++u) {
            const uint4 w = wv[kLoadsFirst ? r : 0][u];
            const float wf[8] = {bf16lo(w.x), bf16hi(w.x), bf16lo(w.y), bf16hi(w.y),
                                 bf16lo(w.z), bf16hi(w.z), bf16lo(w.w), bf16hi(w.w)};
#pragma unroll
            for (int m = 0; m < M; ++m) {
              if (!mact[m]) {
                if (u == 0) acc[m * TR + r] = 0.f;
                continue;
              }
#pragma unroll
              for (int e = 0; e < 8; ++e)
                acc[m * TR + r] = (u == 0 && e == 0) ? __fmul_rn(wf[e], XR(m, u, e))
                                                     : fmaf(wf[e], XR(m, u, e), acc[m * TR + r]);
            }
          }
        }
      }
      const int ct = n - chunk_n0;
      const float s = transpose_reduce<NV>(acc, lane);
      constexpr int kShift = 5 - ilog2(NV);
      if ((lane & ((1 << kShift) - 1)) == 0) red[(ct * NW + warp) * NV + (lane >> kShift)] = s;

      // deferred epilogue over CHT tiles (or at a problem boundary: the
      // per-vector state above belongs to the current problem)
      const bool last_of_problem = (n == ntiles - 1) || (tip + 1 == tpp);
      if (ct == CHT - 1 || last_of_problem) {
        named_bar_sync(1, NC);
        // K split: publication / consumption counts of this chunk slot
        int* kpub = ksplit ? a.part_flag + (size_t)kb * kSplitChunks + (nchunk++ % kSplitChunks) : nullptr;
        int* kcons = ksplit ? kpub + (size_t)gridDim.x * kSplitChunks : nullptr;
        if (ksplit && kh == 0) {  // wait for the second half's row sums of this chunk
          if (tid == 0) {
            const int want = *kcons + 1;  // only this CTA writes its consumption count
            const uint64_t tw = globaltimer();
            while ((int)((unsigned)ld_acquire_gpu(kpub) - (unsigned)want) < 0)
              if (globaltimer() - tw > 2000000000ull) {  // 2 s: sticky error, never a hang
                atomicOr(a.err, kGemvErrSplitTimeout);
                break;
              }
            *kcons = want;  // consumed (a late publication then pairs with this chunk, not the next)
          }
          named_bar_sync(1, NC);
        }
        const int n0 = chunk_n0;
        chunk_n0 = n + 1;
        const int nrows = (ct + 1) * TR;
        auto rowsum = [&](int rl, int m) {
          const int tt = rl / TR, r = rl % TR;
          float s = 0.f;
#pragma unroll
          for (int w = 0; w < NW; ++w) s += red[(tt * NW + w) * NV + vidx(m, r)];
          return s;
        };
        if (EPI == kMatQKV || EPI == kMatGU) {
          for (int pr = tid; pr < nrows / 2; pr += NC) {
            const int rl = pr * 2;
            const long long tg = t0 + n0 + rl / TR;
            const int rr = (int)(tg - (long long)p * tpp) * TR + rl % TR;
#pragma unroll
            for (int m = 0; m < M; ++m) {
              if (!mact[m]) continue;
              const float y0 = rowsum(rl, m), y1 = rowsum(rl + 1, m);
              const int slot = vslot[m], pos = vpos[m];
              if (EPI == kMatGU) {
                a.h[(size_t)slot * a.dm.ffn + (rr >> 1)] = y0 / (1.0f + expf(-y0)) * y1;
              } else {
                const int H = a.dm.H, KVh = a.dm.KV, hd = a.dm.hd;
                const LayerW& L = a.layers[work->first[s_pg[p]] + a.layer_i];
                const int head = rr / hd, w = rr - head * hd;
                float o0 = y0, o1 = y1;
                void* cache = nullptr;
                int kvh = 0;
                if (head < H + KVh) {
                  const int half = hd >> 1;
                  const float c = a.rope_cos[(size_t)pos * half + (w >> 1)];
                  const float sn = a.rope_sin[(size_t)pos * half + (w >> 1)];
                  o0 = y0 * c - y1 * sn;
                  o1 = y1 * c + y0 * sn;
                  if (head < H) {
                    float* q = a.q + (size_t)slot * H * hd + head * hd + w;
                    q[0] = o0;
                    q[1] = o1;
                  } else {
                    cache = L.kc;
                    kvh = head - H;
                  }
                } else {
                  cache = L.vc;
                  kvh = head - H - KVh;
                }
                if (cache) {
                  const int page = a.page_table[pos / kPage];
                  const size_t off = (((size_t)page * KVh + kvh) * kPage + (pos % kPage)) * hd + w;
                  if (a.dm.kv_bf16) {
                    *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(cache) + off) =
                        __floats2bfloat162_rn(o0, o1);
                  } else {
                    float* cp = reinterpret_cast<float*>(cache) + off;
                    cp[0] = o0;
                    cp[1] = o1;
                  }
                }
              }
            }
          }
        } else {
          for (int rl = tid; rl < nrows; rl += NC) {
            const long long tg = t0 + n0 + rl / TR;
            const int rr = (int)(tg - (long long)p * tpp) * TR + rl % TR;
#pragma unroll
            for (int m = 0; m < M; ++m) {
              if (!mact[m]) continue;
              const float y = rowsum(rl, m);
              if (kHead) {
                const int vi = kHead2 ? m : cur_v0 + m;
                a.logits[(size_t)vi * a.dm.V + rr] = y;
                if (y > bestv[m]) {  // rows ascend per thread: strict > keeps first index
                  bestv[m] = y;
                  besti[m] = rr;
                }
              } else if (ksplit) {
                float* pb = a.part_buf + (size_t)vslot[m] * a.dm.d + rr;
                if (kh) *pb = y;
                else a.x[(size_t)vslot[m] * a.dm.d + rr] += y + __ldcg(pb);
              } else {
                a.x[(size_t)vslot[m] * a.dm.d + rr] += y;
              }
            }
          }
        }
        if (ksplit && kh == 1) __threadfence();  // row sums before the flag
        named_bar_sync(1, NC);
        if (ksplit && kh == 1 && tid == 0) red_release_gpu_add(kpub, 1);  // publish
      }
      if (++tip == tpp) {
        tip = 0;
        ++p;
      }
    }
#undef XR
  }

  if (kHead) {  // deterministic first-index argmax across the CTAs of each problem
#pragma unroll
    for (int m = 0; m < M; ++m) {
      float v = bestv[m];
      int i = besti[m];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, v, off);
        const int oi = __shfl_xor_sync(0xffffffffu, i, off);
        if (better(ov, oi, v, i)) { v = ov; i = oi; }
      }
      if (lane == 0) { s_bv[warp][m] = v; s_bi[warp][m] = i; }
    }
    named_bar_sync(1, NC);
    // kHead2: one problem over the whole grid; kHeadV: this CTA's problem span
    const int v0 = kHeadV ? s_pv[hv_p] : 0;
    const int c0 = kHeadV ? hv_c0 : 0, c1 = kHeadV ? hv_c1 : (int)gridDim.x;
    int* ticket = a.head_cnt + (kHeadV ? hv_p : 0);
    __shared__ int s_last;
    if (tid == 0) {
      for (int m = 0; m < M; ++m) {
        float v = s_bv[0][m];
        int i = s_bi[0][m];
        for (int w = 1; w < NW; ++w)
          if (better(s_bv[w][m], s_bi[w][m], v, i)) { v = s_bv[w][m]; i = s_bi[w][m]; }
        a.head_part[((size_t)blockIdx.x * kMaxVec + v0 + m) * 2 + 0] = v;
        a.head_part[((size_t)blockIdx.x * kMaxVec + v0 + m) * 2 + 1] = __int_as_float(i);
      }
      __threadfence();
      s_last = atomicAdd(ticket, 1) == c1 - c0 - 1;
    }
    named_bar_sync(1, NC);
    if (s_last) {  // the last CTA merges the per-CTA partials, all loads in parallel
      __threadfence();
#pragma unroll
      for (int m = 0; m < M; ++m) {
        float v = -FLT_MAX;
        int i = INT_MAX;
        for (int b = c0 + tid; b < c1; b += NC) {
          const float bv = __ldcg(&a.head_part[((size_t)b * kMaxVec + v0 + m) * 2 + 0]);
          const int bi = __float_as_int(__ldcg(&a.head_part[((size_t)b * kMaxVec + v0 + m) * 2 + 1]));
          if (better(bv, bi, v, i)) { v = bv; i = bi; }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, v, off);
          const int oi = __shfl_xor_sync(0xffffffffu, i, off);
          if (better(ov, oi, v, i)) { v = ov; i = oi; }
        }
        if (lane == 0) { s_bv[warp][m] = v; s_bi[warp][m] = i; }
      }
      named_bar_sync(1, NC);
      if (tid == 0) {
        Work* wk = const_cast<Work*>(work);
        const int nv0 = kHeadV ? work->nv[0] : 0;
        for (int m = 0; m < M; ++m) {
          float v = s_bv[0][m];
          int i = s_bi[0][m];
          for (int w = 1; w < NW; ++w)
            if (better(s_bv[w][m], s_bi[w][m], v, i)) { v = s_bv[w][m]; i = s_bi[w][m]; }
          if (kHead2) wk->head_out[m] = work->head_slot[m] >= 0 ? i : -1;
          else if (v0 + m < nv0) wk->vec_out[v0 + m] = i;
        }
        *ticket = 0;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host-side dispatch

namespace {
constexpr int kVpts[] = {1, 2, 3, 4, 6, 7, 8, 14};
constexpr size_t kRingBudget = 212 * 1024;
constexpr size_t kMinCopy = 64 * 1024;  // bulk-copy bytes per stage to aim for

// rows per stage: ~64-96 KB bulk copies at M=1 (tools/stream_bench.cu);
// fewer rows when M vectors' input slices must also live in registers
// M >= 2 loads weights as the FMAs need them (gemv_kernel), so its rows per
// tile are bounded by the accumulators + input slices only.
constexpr int tr_for(int vpt, int m, int epi = -1) {
  if (m == 1) return vpt == 1 ? 16 : vpt <= 3 ? 8 : vpt <= 6 ? 4 : vpt <= 8 ? 2 : 1;
  if (m == 2 && epi == kMatHead) return vpt <= 2 ? 8 : 4;  // loads-first (kLoadsFirst)
  if (m == 2) return vpt <= 4 ? 4 : vpt <= 8 ? 2 : 1;
  if (epi == kMatHeadV) return vpt <= 2 ? 4 : 2;  // + the argmax state
  if (vpt >= 5) return 2;  // m == 4, register boost
  return vpt <= 2 ? 8 : 4;  // m == 4
}
// vectors per weight pass of the batched (prefill / EESD) plans
constexpr int m_batched(int vpt) { return vpt <= 6 ? 4 : vpt <= 8 ? 2 : 1; }

template <int VPT, int M, int EPI>
cudaError_t launch_one(const GemvArgs& a, size_t smem, int grid, cudaStream_t st, bool attrs_only) {
  constexpr int TR = tr_for(VPT, M, EPI);
  auto fn = gemv_kernel<VPT, TR, M, EPI>;
  if (attrs_only) return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return launch_pdl(fn, dim3(grid), dim3(gemv_threads<VPT, M, EPI>()), smem, st, a);
}

template <int VPT, int M>
cudaError_t launch_vm(const GemvArgs& a, size_t smem, int grid, cudaStream_t st, bool attrs_only, int mat) {
  if constexpr (M == 2 && VPT <= 4) {  // the PPSD tick head (exit + final)
    if (mat == kMatHead) return launch_one<VPT, 2, kMatHead>(a, smem, grid, st, attrs_only);
  }
  if constexpr ((M == 1) || (M == m_batched(VPT))) {
    if (mat == kMatO) return launch_one<VPT, M, kMatO>(a, smem, grid, st, attrs_only);
    if (mat == kMatDown) return launch_one<VPT, M, kMatDown>(a, smem, grid, st, attrs_only);
    if (mat == kMatDownS) return launch_one<VPT, M, kMatDownS>(a, smem, grid, st, attrs_only);
    if constexpr (tr_for(VPT, M) >= 2) {  // row-pair epilogues
      if (mat == kMatQKV) return launch_one<VPT, M, kMatQKV>(a, smem, grid, st, attrs_only);
      if (mat == kMatGU) return launch_one<VPT, M, kMatGU>(a, smem, grid, st, attrs_only);
    }
    if constexpr (M == 4) {
      if (mat == kMatHeadV) return launch_one<VPT, 4, kMatHeadV>(a, smem, grid, st, attrs_only);
    }
  }
  return cudaErrorInvalidValue;
}

template <int VPT>
cudaError_t launch_vpt(const GemvArgs& a, int m, size_t smem, int grid, cudaStream_t st, bool attrs_only,
                       int mat) {
  switch (m) {
    case 1: return launch_vm<VPT, 1>(a, smem, grid, st, attrs_only, mat);
    case 2: return launch_vm<VPT, 2>(a, smem, grid, st, attrs_only, mat);
    case 4: return launch_vm<VPT, 4>(a, smem, grid, st, attrs_only, mat);
  }
  return cudaErrorInvalidValue;
}

cudaError_t dispatch(const GemvArgs& a, int vpt, int m, size_t smem, int grid, cudaStream_t st, bool attrs_only,
                     int mat) {
  switch (vpt) {
    case 1: return launch_vpt<1>(a, m, smem, grid, st, attrs_only, mat);
    case 2: return launch_vpt<2>(a, m, smem, grid, st, attrs_only, mat);
    case 3: return launch_vpt<3>(a, m, smem, grid, st, attrs_only, mat);
    case 4: return launch_vpt<4>(a, m, smem, grid, st, attrs_only, mat);
    case 6: return launch_vpt<6>(a, m, smem, grid, st, attrs_only, mat);
    case 7: return launch_vpt<7>(a, m, smem, grid, st, attrs_only, mat);
    case 8: return launch_vpt<8>(a, m, smem, grid, st, attrs_only, mat);
    case 14: return launch_vpt<14>(a, m, smem, grid, st, attrs_only, mat);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

// Choose the (VPT, TR, M, NS) instantiation for a [R][K] matrix; 0 on success.
int gemv_pick(int K, int R, int mat, int batched, int* vpt, int* tr, int* m, int* nstage, int* sub,
              size_t* smem) {
  if (K % 8 != 0 || K <= 0 || R <= 0) return -1;
  int v = -1;
  const int need = (K + 8 * 256 - 1) / (8 * 256);  // 8 consumer warps
  for (int c : kVpts)
    if (c >= need) { v = c; break; }
  if (v < 0) return -1;
  const int mm = mat == kMatHead ? 2 : mat == kMatHeadV ? 4 : batched ? m_batched(v) : 1;
  if ((mat == kMatHead || mat == kMatHeadV) && v > 4) return -1;
  const int t = tr_for(v, mm, mat);
  if (R % t != 0) return -1;
  if ((mat == kMatQKV || mat == kMatGU) && t < 2) return -1;
  const int nw = nw_for(v), rows_chunk = nw == 16 ? 64 : 128;
  const int cht = rows_chunk / t < 1 ? 1 : rows_chunk / t;
  const size_t tile = (size_t)t * K * 2;
  const size_t red = (size_t)cht * nw * mm * t * 4;
  // copies of >= 64 KB per stage, keeping >= 2 stages (3 when they fit)
  int sb = (int)((kMinCopy + tile - 1) / tile);
  if (sb < 1) sb = 1;
  while (sb > 1 && (kRingBudget - red) / (sb * tile) < 3 && (kRingBudget - red) / ((sb - 1) * tile) >= 3) --sb;
  const size_t stage = (size_t)sb * tile;
  int ns = (int)((kRingBudget - red) / stage);
  if (ns > 6) ns = 6;
  if (ns < 2) return -1;
  *vpt = v;
  *tr = t;
  *m = mm;
  *nstage = ns;
  *sub = sb;
  *smem = stage * ns + red + 2 * ns * sizeof(uint64_t);
  return 0;
}

cudaError_t gemv_set_attrs(int vpt, int m, int mat, int ksplit, size_t smem) {
  GemvArgs dummy{};
  return dispatch(dummy, vpt, m, smem, 0, 0, true, mat == kMatDown && ksplit ? kMatDownS : mat);
}

cudaError_t gemv_launch(const GemvArgs& a, int vpt, int m, size_t smem, int grid, cudaStream_t st) {
  return dispatch(a, vpt, m, smem, grid, st, false, a.mat == kMatDown && a.ksplit ? kMatDownS : a.mat);
}

}  // namespace ppsd
