// Does a flag-spinning kernel on one stream let a kernel on another stream
// (plain launch or inside a CUDA graph, small or SM-filling with large smem)
// of the same process run? Prints how long the spinner waited.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void spin(volatile unsigned* flag, unsigned long long* waited) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag == 0) {
    __nanosleep(100);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 3000000000ull) break;
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  *waited = t1 - t0;
}
__global__ void big(float* x) {  // SM-filling grid with large dynamic smem
  extern __shared__ float sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0) x[blockIdx.x] = sm[blockIdx.x % blockDim.x];
}
__global__ void setf(volatile unsigned* flag) { *flag = 1; }

int main() {
  unsigned* flag;
  unsigned long long* waited;
  float* x;
  cudaMalloc(&flag, 4);
  cudaMalloc(&waited, 8);
  cudaMalloc(&x, 4096 * 4);
  cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, 212 * 1024);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 4; ++mode) {
    cudaMemset(flag, 0, 4);
    cudaDeviceSynchronize();
    spin<<<1, 256, 0, a>>>(flag, waited);
    if (mode == 0) {
      setf<<<1, 1, 0, b>>>(flag);
    } else if (mode == 1) {
      big<<<sms, 256, 212 * 1024, b>>>(x);
      setf<<<1, 1, 0, b>>>(flag);
    } else {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStream_t cs;
      cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
      cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
      if (mode == 3) big<<<sms, 256, 212 * 1024, cs>>>(x);
      setf<<<1, 1, 0, cs>>>(flag);
      cudaStreamEndCapture(cs, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, b);
    }
    cudaDeviceSynchronize();
    unsigned long long w;
    cudaMemcpy(&w, waited, 8, cudaMemcpyDeviceToHost);
    printf("mode %d (%s): spinner waited %.3f ms  err=%s\n", mode,
           mode == 0 ? "plain small" : mode == 1 ? "plain SM-filling 212KB" : mode == 2 ? "graph small" : "graph SM-filling",
           w / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
