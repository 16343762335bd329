// tc_dev.cuh — tcgen05 / TMEM / cluster helpers shared by the tensor-core
// GEMV (tcgemv.cu) and the persistent layer pass (tcpass.cu).
#pragma once
#include <float.h>
#include <limits.h>

#include "kernels.cuh"

namespace ppsd {


constexpr int kTcMaxBlk = (3 * kMaxVec + 15) / 16;  // 16-column blocks for 16 vectors x 3 parts: 3
constexpr int kTcThreads = 320;
constexpr int kTcAccCols = 64;                   // one accumulator (N <= 48 columns used)
constexpr int kTcTmemCols = 2 * kTcAccCols;      // double-buffered: 128
constexpr int kTcMaxProb = 32;
constexpr int kTcVecPerBlk = 5;  // vectors whose three parts fit one 16-column B block

// kind::f16 instruction descriptor: bf16 x bf16 -> fp32, A and B K-major,
// M = 128 (bits 24-28: M >> 4); N (bits 17-22: N >> 3) per launch
constexpr uint32_t kTcIdescBase = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 4) << 24);

// ---- thread-block cluster helpers (split-K across the CS CTAs of a cluster)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of the same smem variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool tc_better(float v, int i, float bv, int bi) {
  return v > bv || (v == bv && i < bi);
}

// K-major SWIZZLE_128B smem descriptor: 8-row x 128 B atoms, `sbo` bytes
// between consecutive 8-row groups
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                       // leading byte offset (unused, swizzled K-major)
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;   // stride byte offset
  d |= (uint64_t)1 << 46;                       // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// one lane of the (converged) warp: the MMA issue idiom that keeps the
// operands in uniform registers (measured: 42 cycles per N=16 MMA issued
// from a converged warp vs 143 from a lone divergent thread)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// Pipeline timeline of CTA 0 (debugging: PPSD_TC_TRACE=1, ppsd_debug_tc_trace):
// [event][stage] %globaltimer ns. Events: 0 producer issued, 1 MMA saw full,
// 2 MMA issued all, 3 builder arrived, 4 epilogue saw acc_full (per tile),
// 5 epilogue done (per tile), 6 kernel start (slot 0)
constexpr int kTcTraceN = 128;
static __device__ unsigned long long g_tc_trace[8][kTcTraceN];
static __device__ int g_tc_trace_on;
static __device__ int g_tc_exp;  // experiments: 1 = no weight copies, 2 = no operand stores
// the experiment switch: a global load on the producer's critical path, so
// only trace builds read it
__device__ __forceinline__ int tc_exp() {
#ifdef PPSD_TC_TRACE
  return g_tc_exp;
#else
  return 0;
#endif
}
static __device__ unsigned long long g_tc_cta[160][4];  // per CTA: start, first copy, last MMA issued, exit
// compiled in only with -DPPSD_TC_TRACE (the probes perturb the pipeline)
__device__ __forceinline__ void tc_cta_mark(int k) {
#ifdef PPSD_TC_TRACE
  if (g_tc_trace_on && blockIdx.x < 160) g_tc_cta[blockIdx.x][k] = globaltimer();
#endif
}
__device__ __forceinline__ void tc_trace(int ev, int n) {
#ifdef PPSD_TC_TRACE
  if (g_tc_trace_on && blockIdx.x == 0 && n < kTcTraceN) g_tc_trace[ev][n] = globaltimer();
#endif
}

// The tiles of a CTA's group range [u0, u1): problem by problem, each
// problem's part cut into ceil(len / TG) near-equal tiles. Every role walks
// the same sequence.
struct TcTiles {
  int u, u1, G, TG;
  int p, seg_lo, seg_len, nt, i;  // current segment and tile index inside it
  __device__ void init(int u0_, int u1_, int G_, int TG_) {
    u = u0_;
    u1 = u1_;
    G = G_;
    TG = TG_;
    seg_len = 0;
    nt = 0;
    i = 0;
  }
  // the tile just returned by next() was the range's last
  __device__ bool last() const { return i == nt && u >= u1; }
  // next tile: problem p, first group g0 (within the problem), tg groups
  __device__ bool next(int& tp, int& g0, int& tg) {
    if (i == nt) {
      if (u >= u1) return false;
      p = u / G;
      const int pend = min(u1, (p + 1) * G);
      seg_lo = u - p * G;
      seg_len = pend - u;
      nt = (seg_len + TG - 1) / TG;
      i = 0;
      u = pend;
    }
    const int a = seg_len * i / nt, b = seg_len * (i + 1) / nt;
    ++i;
    tp = p;
    g0 = seg_lo + a;
    tg = b - a;
    return true;
  }
};


}  // namespace ppsd
