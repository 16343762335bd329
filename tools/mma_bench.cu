// mma_bench.cu — tcgen05.mma issue/throughput microbenchmark (one CTA per SM,
// smem operands, no data movement): cycles per MMA for the decode GEMV's
// shapes (M=128, N=16, K=16) against larger N, and the A stride (SBO).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench tools/mma_bench.cu && tools/mma_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t sbo) {
  uint64_t d = (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

__global__ void __launch_bounds__(128, 1) bench(int n_mma, int N, int M, uint32_t sbo_a, int nacc, int mode,
                                                long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t taddr;
  __shared__ __align__(8) uint64_t bar;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~(uintptr_t)1023);
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3f803f80u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (mode == 1 && threadIdx.x < 32) {  // whole warp runs the loop, one elected lane issues
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = smem_u32(base), b0 = smem_u32(base + 128 * 1024);
    const uint64_t ad0 = desc(a0, sbo_a), bd0 = desc(b0, 1024);
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const uint32_t kk = (i & 3) * 2;  // 32 B in descriptor units (16 B)
      if (elect_one()) mma(taddr + (uint32_t)((i % nacc) * N), ad0 + kk, bd0 + kk, idesc, i >= nacc);
      __syncwarp();
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    __syncwarp();
    asm volatile(
        "{\n\t.reg .pred P1;\nW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W1;\n}" ::"r"(
            smem_u32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
  }
  if (mode >= 2 && threadIdx.x < 32) {  // unrolled, constant offsets, one elected lane (2: per mma, 3: per 8)
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = smem_u32(base), b0 = smem_u32(base + 128 * 1024);
    const uint64_t ad0 = desc(a0, sbo_a), bd0 = desc(b0, 1024);
    const uint32_t tm = taddr;
    long long t0 = clock64();
    for (int i = 0; i < n_mma; i += 8) {
      if (mode == 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (elect_one()) mma(tm, ad0 + (k & 3) * 2, bd0 + (k & 3) * 2, idesc, (i | k) != 0);
      } else if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) mma(tm, ad0 + (k & 3) * 2, bd0 + (k & 3) * 2, idesc, (i | k) != 0);
      }
      __syncwarp();
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    __syncwarp();
    asm volatile(
        "{\n\t.reg .pred P1;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W2;\n}" ::"r"(
            smem_u32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
  }
  if (mode == 0 && threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t a0 = smem_u32(base), b0 = smem_u32(base + 128 * 1024);
    long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const uint32_t kk = (i & 3) * 32;
      mma(taddr + (uint32_t)((i % nacc) * N), desc(a0 + kk, sbo_a), desc(b0 + kk, 1024), idesc, i >= nacc);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}" ::"r"(
            smem_u32(&bar)));
    long long t1 = clock64();
    if (blockIdx.x == 0) *out = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct C { int N, M; uint32_t sbo; int nacc; } cs[] = {
      {16, 128, 1024, 1}, {16, 128, 8192, 1}, {48, 128, 1024, 1}, {64, 128, 1024, 1}, {16, 64, 1024, 1},
      {16, 64, 4096, 1}, {48, 64, 1024, 1}, {8, 64, 1024, 1}, {256, 128, 1024, 1}};
  for (int mode = 2; mode < 3; ++mode)
  for (const C& c : cs) {
    const int n = 2048;
    bench<<<148, 128, 200 * 1024>>>(n, c.N, c.M, c.sbo, c.nacc, mode, d);
    bench<<<148, 128, 200 * 1024>>>(n, c.N, c.M, c.sbo, c.nacc, mode, d);
    long long cyc = 0;
    cudaError_t e = cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("mode %d M=%3d N=%3d sbo=%5u chains=%d: %6.1f cycles/mma  (%s)\n", mode, c.M, c.N, c.sbo, c.nacc,
           (double)cyc / n, cudaGetErrorString(e));
  }
  return 0;
}
