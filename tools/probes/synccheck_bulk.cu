// Does compute-sanitizer synccheck mistake a bulk copy's shared destination
// at shared address 0 for an mbarrier? Variant bits: 1 destination 1 KB past
// the dynamic shared base, 2 the L2::cache_hint form, 4 an L2 bulk prefetch
// first.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/sb synccheck_bulk.cu
//   compute-sanitizer --tool synccheck /tmp/sb 0 ; ... /tmp/sb 1
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const float* src, float* dst, int v) {
  const int off = (v & 1) ? 1024 : 0;
  extern __shared__ __align__(1024) unsigned char buf[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(1024) : "memory");
    if (v & 4) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(1024) : "memory");
    if (v & 2) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                   " [%0], [%1], %2, [%3], %4;" ::"r"(su32(buf + off)), "l"(src), "r"(1024), "r"(su32(&bar)),
                   "l"(pol) : "memory");
    } else {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(buf + off)), "l"(src), "r"(1024), "r"(su32(&bar)) : "memory");
    }
  }
  asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}"
               ::"r"(su32(&bar)) : "memory");
  const float* f = reinterpret_cast<const float*>(buf + off);
  dst[threadIdx.x] = f[threadIdx.x];
}

int main(int argc, char** argv) {
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  float *s, *d;
  cudaMalloc(&s, 1024);
  cudaMalloc(&d, 1024);
  float h[256];
  for (int i = 0; i < 256; ++i) h[i] = (float)i;
  cudaMemcpy(s, h, 1024, cudaMemcpyHostToDevice);
  k<<<4, 256, 4096>>>(s, d, v);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 1024, cudaMemcpyDeviceToHost);
  printf("variant %d: %s, h[255]=%g\n", v, cudaGetErrorString(e), h[255]);
  return 0;
}
