// attn.cu — standalone split-K decode attention kernel: one 128-thread
// worker (attn_core.cuh) per CTA. The persistent layer pass (tcpass.cu) runs
// the same worker code between its QKV and O phases.
#include "attn_core.cuh"

namespace ppsd {

template <int HD, typename KVT, int QPK>
__global__ void __launch_bounds__(kAttnThreads) attn_kernel(const AttnArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ AttnScratch<HD, QPK> S;
  if (threadIdx.x == 0) {
    mbar_init(&S.bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  attn_items<HD, KVT, QPK>(a, blockIdx.x, gridDim.x, threadIdx.x, reinterpret_cast<KVT*>(smem), S, phase,
                           [] { __syncthreads(); },
                           [] {  // q / this layer's KV rows come from the preceding QKV kernel
                             pdl_wait();
                             pdl_trigger();
                           });
}

namespace {
int g_attn_occ = 0;  // attn_set_attrs: resident CTAs per SM of the configured instantiation

template <int HD, typename KVT, int QPK>
cudaError_t launch_k(const AttnArgs& a, int grid, cudaStream_t st, bool attrs) {
  const size_t smem = 2 * (size_t)kPage * HD * sizeof(KVT);
  if (attrs) {
    cudaError_t e = cudaFuncSetAttribute(attn_kernel<HD, KVT, QPK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e == cudaSuccess)
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_attn_occ, attn_kernel<HD, KVT, QPK>, kAttnThreads, smem);
    return e;
  }
  return launch_pdl(attn_kernel<HD, KVT, QPK>, dim3(grid), dim3(kAttnThreads), smem, st, a);
}
template <int HD, typename KVT>
cudaError_t launch_qpk(const AttnArgs& a, int grid, cudaStream_t st, bool attrs) {
  switch (a.dm.H / a.dm.KV) {
    case 1: return launch_k<HD, KVT, 1>(a, grid, st, attrs);
    case 2: return launch_k<HD, KVT, 2>(a, grid, st, attrs);
    case 4: return launch_k<HD, KVT, 4>(a, grid, st, attrs);
    case 8: return launch_k<HD, KVT, 8>(a, grid, st, attrs);
  }
  return cudaErrorInvalidValue;
}
template <int HD>
cudaError_t launch_hd(const AttnArgs& a, int grid, cudaStream_t st, bool attrs) {
  return a.dm.kv_bf16 ? launch_qpk<HD, __nv_bfloat16>(a, grid, st, attrs)
                      : launch_qpk<HD, float>(a, grid, st, attrs);
}
cudaError_t dispatch(const AttnArgs& a, int grid, cudaStream_t st, bool attrs) {
  switch (a.dm.hd) {
    case 16: return launch_hd<16>(a, grid, st, attrs);
    case 32: return launch_hd<32>(a, grid, st, attrs);
    case 64: return launch_hd<64>(a, grid, st, attrs);
    case 128: return launch_hd<128>(a, grid, st, attrs);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

bool attn_supported(int hd, int qpk) {
  return (hd == 16 || hd == 32 || hd == 64 || hd == 128) && (qpk == 1 || qpk == 2 || qpk == 4 || qpk == 8);
}

cudaError_t attn_set_attrs(const AttnArgs& a) { return dispatch(a, 0, 0, true); }

// CTAs per SM that are resident at once (after attn_set_attrs): the grid is
// sized to one wave, a second wave of item-less CTAs costs ~2 us
int attn_ctas_per_sm() { return g_attn_occ; }

int attn_trace_enable(int on) { return cudaMemcpyToSymbol(g_attn_tr_on, &on, sizeof(int)) == cudaSuccess ? 0 : -1; }
int attn_trace_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_attn_tr, sizeof(g_attn_tr)) == cudaSuccess ? 0 : -1;
}

cudaError_t attn_launch(const AttnArgs& a, int grid, cudaStream_t st) { return dispatch(a, grid, st, false); }

}  // namespace ppsd
