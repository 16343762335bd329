// init.cu — counter-hash weight initialiser, bit-identical to
// oracle/transformer.py:init_tensor, written directly in the engine's
// physical layout (RoPE pair-interleaved q/k rows, interleaved gate/up rows).
#include "engine_dev.cuh"

namespace ppsd {

__device__ __forceinline__ __nv_bfloat16 hash_weight(uint64_t base, long long idx, float a) {
  const uint64_t h = hmix64(base + (uint64_t)(idx + 1) * kGoldenGamma);
  const float u = __fmul_rn((float)(h >> 40), 0x1p-24f);
  const float t = __fsub_rn(__fmul_rn(2.0f, u), 1.0f);
  return __float2bfloat16_rn(__fmul_rn(t, a));
}

// tiled = 1: the TC-tiled layout of the tensor-core GEMV (kernels.cuh:
// tc_offset), K padded with zeros to a multiple of 64
__global__ void init_weight_kernel(__nv_bfloat16* dst, int layout, int tiled, long long rows, long long cols,
                                   uint64_t b0, uint64_t b1, uint64_t b2, float a0, float a1, float a2,
                                   int H, int KV, int hd) {
  int js = 1, kp = (int)cols;
  if (tiled) tc_layout((int)rows, (int)cols, &js, &kp);
  const long long n = rows * kp;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long pr = i / kp, col = i - pr * kp;
    const long long di = tiled ? tc_offset((int)rows, (int)cols, pr, col) : i;
    if (col >= cols) {  // K padding (tiled only)
      dst[di] = __float2bfloat16_rn(0.f);
      continue;
    }
    uint64_t base = b0;
    float a = a0;
    long long lr = pr;  // logical row in the logical tensor
    if (layout == 1) {  // fused qkv, q/k rows pair-interleaved for RoPE
      const long long qrows = (long long)H * hd, krows = (long long)KV * hd;
      if (pr < qrows + krows) {
        const long long r = pr < qrows ? pr : pr - qrows;
        const long long head = r / hd;
        const int w = (int)(r - head * hd);
        const int dim = (w & 1) ? hd / 2 + (w >> 1) : (w >> 1);
        lr = head * hd + dim;
        if (pr >= qrows) { base = b1; a = a1; }
      } else {
        lr = pr - qrows - krows;
        base = b2;
        a = a2;
      }
    } else if (layout == 2) {  // fused gate/up, rows interleaved (gate_i, up_i)
      lr = pr >> 1;
      if (pr & 1) { base = b1; a = a1; }
    }
    dst[di] = hash_weight(base, lr * cols + col, a);
  }
}

}  // namespace ppsd
