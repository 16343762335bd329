// umma.cu — tcgen05 (5th-gen tensor core) weight-streaming GEMM for the
// batched prompt prefill on sm_100a.
//
// A prefill chunk multiplies every weight matrix W [R][K] (bf16, row-major)
// by up to kUmN = 64 token vectors. The bs=1 decode GEMV (gemv.cu) keeps each
// vector's input slice in registers, which caps it at 4 vectors per weight
// pass; here the tokens are the N dimension of a UMMA and the weights are
// streamed from HBM exactly once per chunk:
//
//   D[128 rows][64 tokens] (fp32, TMEM) += W_tile[128][K] . X[64][K]^T
//
// X is split into two bf16 halves (hi = bf16(x), lo = bf16(x - hi)) and both
// are multiplied into the same accumulator, so the activations keep ~16
// mantissa bits (the decode path multiplies fp32 activations; a single bf16
// rounding of x would cost 8 of them). Weights are exact in bf16.
//
// One CTA per SM, 192 threads:
//   warp 0 (one lane)   TMA producer: 2-D tensor copies with 128-byte swizzle
//                       into a 3-deep ring of 64 KB stages (two 16 KB weight
//                       boxes + four 8 KB activation boxes), mbarrier expect_tx.
//                       Weight boxes of the first stages are issued before
//                       griddepcontrol.wait (weights never depend on the
//                       previous kernel).
//   warp 1              TMEM owner (alloc/dealloc, 128 columns = two 64-column
//                       accumulators) and, on one lane, the MMA issuer:
//                       tcgen05.mma.cta_group::1.kind::f16 M=128 N=64 K=16,
//                       smem descriptors in the canonical K-major SW128
//                       layout, tcgen05.commit frees ring stages and
//                       publishes finished accumulators.
//   warps 2-5           epilogue: tcgen05.ld 32x32b.x16 x4 (one TMEM lane = one
//                       weight row per thread, 64 token columns), then the
//                       same fused epilogues as the decode GEMV (RoPE + KV
//                       append, SwiGLU, residual add).
//
// Work split: the (row tile, 128-wide K stage) units of the matrix are cut
// into one contiguous range per CTA (stream-K). A tile whose K range spans
// several CTAs is reduced by the last of them to arrive, summing the partials
// in CTA order — deterministic, and independent of the chunk's token count,
// so the pipelined multi-rank prefill (one token per step) reproduces the
// single-GPU chunked prefill bit for bit.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <vector>

#include "kernels.cuh"

namespace ppsd {

constexpr int kUmTileRows = 128;
constexpr int kUmN = 64;    // tokens per chunk (UMMA N); hi + lo halves = 2N operand rows
constexpr int kUmKS = 128;  // K elements per ring stage
constexpr int kUmStages = 3;
constexpr int kUmABox = kUmTileRows * 64 * 2;  // 16 KB
constexpr int kUmBBox = kUmN * 64 * 2;         // 2 KB
constexpr int kUmStageBytes = 2 * kUmABox + 4 * kUmBBox;
constexpr int kUmThreads = 192;
constexpr size_t kUmSmem = (size_t)kUmStages * kUmStageBytes + 1024 + 256;

// ---------------------------------------------------------------------------
// PTX wrappers

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand, 128-byte swizzle: 8-row x 128 B atoms, 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
  const uint32_t a = smem_u32(p);
  uint64_t d = (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;             // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // stride byte offset: next 8-row group
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}
// kind::f16 instruction descriptor: bf16 x bf16 -> fp32, both K-major, M=128, N=16
constexpr uint32_t kUmIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kUmN >> 3) << 17) |
                              ((uint32_t)(kUmTileRows >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kUmIdesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// one accumulator row (this thread's weight row) x kUmN token columns
__device__ __forceinline__ void tmem_ld_row(uint32_t taddr, float (&v)[kUmN]) {
#pragma unroll
  for (int c = 0; c < kUmN; c += 16) tmem_ld16_nowait(taddr + (uint32_t)c, v + c);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// The CTA whose unit range [U*b/G, U*(b+1)/G) holds unit u.
__device__ __forceinline__ int unit_owner(long long u, long long U, int G) {
  return (int)(((u + 1) * G - 1) / U);
}
__device__ __forceinline__ long long unit_start(int b, long long U, int G) { return U * b / G; }

// ---------------------------------------------------------------------------
// fused epilogue on one weight row (`rr`, this thread) x nv token columns

template <int EPI>
__device__ __forceinline__ void um_epilogue_pairs(const UmmaArgs& a, int rr, const float (&y)[kUmN], int lane) {
  const Work* w = a.work;
  const int slot0 = w->slot[0], pos0 = w->pos[0], nv = w->nv[0];
  // row pairs (2i, 2i+1) sit on adjacent lanes
  float yp[kUmN];
#pragma unroll
  for (int n = 0; n < kUmN; ++n) yp[n] = __shfl_xor_sync(0xffffffffu, y[n], 1);
  if (lane & 1) return;
  if (EPI == kMatGU) {
    for (int n = 0; n < nv; ++n)
      a.h[(size_t)(slot0 + n) * a.dm.ffn + (rr >> 1)] = y[n] / (1.0f + expf(-y[n])) * yp[n];
    return;
  }
  // kMatQKV: fused q|k|v rows, RoPE on (q,k) pairs, k/v into the paged cache
  const int H = a.dm.H, KVh = a.dm.KV, hd = a.dm.hd;
  const LayerW& L = a.layers[w->first[0] + a.layer_i];
  const int head = rr / hd, wi = rr - head * hd;
  for (int n = 0; n < nv; ++n) {
    const int pos = pos0 + n, slot = slot0 + n;
    float o0 = y[n], o1 = yp[n];
    void* cache = nullptr;
    int kvh = 0;
    if (head < H + KVh) {
      const int half = hd >> 1;
      const float c = a.rope_cos[(size_t)pos * half + (wi >> 1)];
      const float sn = a.rope_sin[(size_t)pos * half + (wi >> 1)];
      o0 = y[n] * c - yp[n] * sn;
      o1 = yp[n] * c + y[n] * sn;
      if (head < H) {
        float* q = a.q + (size_t)slot * H * hd + head * hd + wi;
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
      const size_t off = (((size_t)page * KVh + kvh) * kPage + (pos % kPage)) * hd + wi;
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

// ---------------------------------------------------------------------------

template <int EPI>
__device__ __forceinline__ void um_epilogue(const UmmaArgs& a, int rr, const float (&y)[kUmN], int lane) {
  if constexpr (EPI == kMatO || EPI == kMatDown) {
    const Work* w = a.work;
    const int slot0 = w->slot[0], nv = w->nv[0];
    for (int n = 0; n < nv; ++n) a.x[(size_t)(slot0 + n) * a.dm.d + rr] += y[n];
  } else {
    um_epilogue_pairs<EPI>(a, rr, y, lane);
  }
}

template <int EPI>
__global__ void __launch_bounds__(kUmThreads, 1) umma_gemm_kernel(const UmmaArgs a) {
  extern __shared__ unsigned char um_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(um_smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kUmStages * kUmStageBytes);
  uint64_t* empty = full + kUmStages;
  uint64_t* acc_full = empty + kUmStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;       // [2]
  uint32_t* s_taddr = reinterpret_cast<uint32_t*>(acc_empty + 2);
  __shared__ int s_last;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const Work* work = a.work;
  // the work descriptor is >= 2 kernels old (the prep kernel sits between)
  const bool active = work->slot[0] >= 0;
  const int KS = a.K / kUmKS;
  const long long T = a.R / kUmTileRows;
  const long long U = T * KS;
  const int G = gridDim.x, b = blockIdx.x;
  const long long u0 = unit_start(b, U, G), u1 = unit_start(b + 1, U, G);
  const int nunits = (int)(u1 - u0);
  if (!active || nunits == 0) {
    pdl_wait();
    pdl_trigger();
    return;
  }

  if (tid == 0) {
    for (int i = 0; i < kUmStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 128);
    }
    fence_mbar_init();
  }
  if (warp == 1) {  // TMEM: 2 * kUmN columns = two kUmN-column fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_taddr)),
                 "n"(2 * kUmN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = *s_taddr;
  const CUtensorMap* wmap =
      reinterpret_cast<const CUtensorMap*>(a.wmaps) + (size_t)(work->first[0] + a.layer_i) * 4 + EPI;
  const CUtensorMap* xmap = reinterpret_cast<const CUtensorMap*>(a.xmap);

  if (warp == 0) {  // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pw = policy_evict_first(), px = policy_evict_last();
      const int npre = nunits < kUmStages ? nunits : kUmStages;
      auto issue_a = [&](int n) {
        const long long u = u0 + n;
        const int tile = (int)(u / KS), ks = (int)(u % KS);
        unsigned char* st = smem + (size_t)(n % kUmStages) * kUmStageBytes;
        mbar_expect_tx(&full[n % kUmStages], kUmStageBytes);
        tma_load_2d(st, wmap, ks * kUmKS, tile * kUmTileRows, &full[n % kUmStages], pw);
        tma_load_2d(st + kUmABox, wmap, ks * kUmKS + 64, tile * kUmTileRows, &full[n % kUmStages], pw);
      };
      auto issue_b = [&](int n) {
        const long long u = u0 + n;
        const int ks = (int)(u % KS);
        unsigned char* st = smem + (size_t)(n % kUmStages) * kUmStageBytes + 2 * kUmABox;
        for (int j = 0; j < 2; ++j) {
          tma_load_2d(st + j * kUmBBox, xmap, ks * kUmKS + 64 * j, 0, &full[n % kUmStages], px);
          tma_load_2d(st + (2 + j) * kUmBBox, xmap, ks * kUmKS + 64 * j, kUmN, &full[n % kUmStages], px);
        }
      };
      for (int n = 0; n < npre; ++n) issue_a(n);  // weights before the dependency resolves
      pdl_wait();
      pdl_trigger();
      for (int n = 0; n < npre; ++n) issue_b(n);
      for (int n = npre; n < nunits; ++n) {
        mbar_wait(&empty[n % kUmStages], ((n / kUmStages) & 1) ^ 1);
        issue_a(n);
        issue_b(n);
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer ----------------
    if (lane == 0) {
      pdl_wait();
      pdl_trigger();
      int seg = 0;
      bool seg_first = true;
      for (int n = 0; n < nunits; ++n) {
        const long long u = u0 + n;
        const int ks = (int)(u % KS);
        const int acc = seg & 1;
        if (seg_first && seg >= 2) mbar_wait(&acc_empty[acc], ((seg >> 1) - 1) & 1);
        mbar_wait(&full[n % kUmStages], (n / kUmStages) & 1);
        tc_fence_after();
        const unsigned char* st = smem + (size_t)(n % kUmStages) * kUmStageBytes;
        const uint32_t d = taddr + (uint32_t)(acc * kUmN);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = sw128_desc(st + j * kUmABox + 32 * k);
            const uint64_t bh = sw128_desc(st + 2 * kUmABox + j * kUmBBox + 32 * k);
            const uint64_t bl = sw128_desc(st + 2 * kUmABox + (2 + j) * kUmBBox + 32 * k);
            umma_bf16(d, ad, bh, (seg_first && j == 0 && k == 0) ? 0u : 1u);
            umma_bf16(d, ad, bl, 1u);
          }
        }
        umma_commit(&empty[n % kUmStages]);  // ring stage free once these MMAs retire
        seg_first = false;
        if (ks == KS - 1 || n == nunits - 1) {
          umma_commit(&acc_full[acc]);
          ++seg;
          seg_first = true;
        }
      }
    }
  } else {  // ---------------- epilogue (warps 2-5) ----------------
    pdl_wait();
    pdl_trigger();
    const int row = 32 * (warp & 3) + lane;  // TMEM lane = weight row in the tile
    const int t_first = (int)(u0 / KS), t_last = (int)((u1 - 1) / KS);
    for (int t = t_first, seg = 0; t <= t_last; ++t, ++seg) {
      const int acc = seg & 1;
      mbar_wait(&acc_full[acc], (seg >> 1) & 1);
      tc_fence_after();
      float y[kUmN];
      tmem_ld_row(taddr + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(acc * kUmN), y);
      tc_fence_before();
      mbar_arrive(&acc_empty[acc]);
      const int rr = t * kUmTileRows + row;
      const int cf = unit_owner((long long)t * KS, U, G), cl = unit_owner((long long)t * KS + KS - 1, U, G);
      if (cf == cl) {
        um_epilogue<EPI>(a, rr, y, lane);
        continue;
      }
      // split tile: publish this CTA's partial, the last contributor reduces
      const int my_slot = (t == t_first) ? 0 : 1;
      float4* dst = reinterpret_cast<float4*>(a.ws + (((size_t)b * 2 + my_slot) * kUmTileRows + row) * kUmN);
#pragma unroll
      for (int i = 0; i < kUmN / 4; ++i) dst[i] = make_float4(y[4 * i], y[4 * i + 1], y[4 * i + 2], y[4 * i + 3]);
      __threadfence();
      named_bar_sync(1, 128);
      int ncontrib = 0;
      for (int c = cf; c <= cl; ++c) ncontrib += unit_start(c + 1, U, G) > unit_start(c, U, G);
      if (tid == 64) s_last = atomicAdd(&a.cnt[t], 1) == ncontrib - 1;
      named_bar_sync(1, 128);
      if (!s_last) continue;
      __threadfence();
      float s[kUmN];
#pragma unroll
      for (int i = 0; i < kUmN; ++i) s[i] = 0.f;
      for (int c = cf; c <= cl; ++c) {
        const long long cs = unit_start(c, U, G);
        if (unit_start(c + 1, U, G) == cs) continue;  // empty range
        const int slot = (cs / KS == t) ? 0 : 1;
        const float4* src =
            reinterpret_cast<const float4*>(a.ws + (((size_t)c * 2 + slot) * kUmTileRows + row) * kUmN);
#pragma unroll
        for (int i = 0; i < kUmN / 4; ++i) {
          const float4 v = __ldcg(src + i);
          s[4 * i] += v.x;
          s[4 * i + 1] += v.y;
          s[4 * i + 2] += v.z;
          s[4 * i + 3] += v.w;
        }
      }
      um_epilogue<EPI>(a, rr, s, lane);
      if (tid == 64) a.cnt[t] = 0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(2 * kUmN));
  }
}

// Input staging: the chunk's vectors (RMS-normalised for QKV / GU) split into
// bf16 hi/lo rows of the [2 * kUmN][K] activation operand. One CTA per token.
__global__ void __launch_bounds__(256) umma_prep_kernel(const UmmaArgs a) {
  pdl_wait();
  pdl_trigger();
  const Work* w = a.work;
  const int n = blockIdx.x;
  if (w->slot[0] < 0 || n >= w->nv[0]) return;
  const int slot = w->slot[0] + n, K = a.K;
  const float* src;
  const float* nw = nullptr;
  const LayerW& L = a.layers[w->first[0] + a.layer_i];
  if (a.mat == kMatQKV) { src = a.x + (size_t)slot * a.dm.d; nw = L.attn_norm; }
  else if (a.mat == kMatGU) { src = a.x + (size_t)slot * a.dm.d; nw = L.mlp_norm; }
  else if (a.mat == kMatO) src = a.o + (size_t)slot * a.dm.H * a.dm.hd;
  else src = a.h + (size_t)slot * a.dm.ffn;
  float rstd = 1.f;
  if (nw) {
    __shared__ float s_ss[8];
    float ss = 0.f;
    for (int k = threadIdx.x; k < K; k += blockDim.x) ss = fmaf(src[k], src[k], ss);
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) s_ss[threadIdx.x >> 5] = ss;
    __syncthreads();
    float tot = 0.f;
    for (int i = 0; i < 8; ++i) tot += s_ss[i];
    rstd = 1.0f / sqrtf(tot / (float)K + a.dm.eps);
  }
  __nv_bfloat16* hi = a.xs + (size_t)n * K;
  __nv_bfloat16* lo = a.xs + (size_t)(kUmN + n) * K;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const float v = nw ? (src[k] * rstd) * nw[k] : src[k];
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
    hi[k] = h;
    lo[k] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
}

// ---------------------------------------------------------------------------
// host side

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool umma_shape_ok(int R, int K) { return R > 0 && K > 0 && R % kUmTileRows == 0 && K % kUmKS == 0; }

int umma_encode_map(void* map, const void* base, int rows, int K, int box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc) return -1;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                   dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -1;
}

size_t umma_map_bytes() { return sizeof(CUtensorMap); }
size_t umma_smem_bytes() { return kUmSmem; }
int umma_tile_rows() { return kUmTileRows; }
int umma_n() { return kUmN; }

cudaError_t umma_set_attrs() {
  cudaError_t e = cudaSuccess;
  auto set = [&](auto fn) {
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUmSmem);
  };
  set(umma_gemm_kernel<kMatQKV>);
  set(umma_gemm_kernel<kMatO>);
  set(umma_gemm_kernel<kMatGU>);
  set(umma_gemm_kernel<kMatDown>);
  if (e == cudaSuccess) {
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, umma_prep_kernel);
  }
  return e;
}

cudaError_t umma_launch(const UmmaArgs& a, int grid, cudaStream_t st) {
  cudaError_t e = launch_pdl(umma_prep_kernel, dim3(kUmN), dim3(256), 0, st, a);
  if (e != cudaSuccess) return e;
  switch (a.mat) {
    case kMatQKV: return launch_pdl(umma_gemm_kernel<kMatQKV>, dim3(grid), dim3(kUmThreads), kUmSmem, st, a);
    case kMatO: return launch_pdl(umma_gemm_kernel<kMatO>, dim3(grid), dim3(kUmThreads), kUmSmem, st, a);
    case kMatGU: return launch_pdl(umma_gemm_kernel<kMatGU>, dim3(grid), dim3(kUmThreads), kUmSmem, st, a);
    case kMatDown: return launch_pdl(umma_gemm_kernel<kMatDown>, dim3(grid), dim3(kUmThreads), kUmSmem, st, a);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ppsd
