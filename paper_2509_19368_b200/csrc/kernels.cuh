// kernels.cuh — device-side data structures and kernel entry points shared by
// the engine (engine.cu) and the kernel translation units.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"
#include "sched.h"

namespace ppsd {

constexpr int kPage = 64;          // KV page = attention chunk (tokens)
constexpr int kGemvConsumers = 256;  // 8 consumer warps
constexpr int kGemvThreads = 288;    // + 1 bulk-copy producer warp
constexpr int kMaxVec = 16;         // vectors per group (batched prefill / EESD verify)

// Per-tick local work: one group per local pipeline stage. Written by the
// scheduler kernel at the start of every tick, read by every layer kernel.
struct Work {
  int32_t G;                    // local stage count
  int32_t slot[kMaxStages];     // chain activation slot, -1 = stage idle this tick
  int32_t pos[kMaxStages];      // token index the chain processes (RoPE / KV index)
  int32_t first[kMaxStages];    // global index of the stage's first layer
  int32_t nl[kMaxStages];       // layers in the stage
  int32_t nv[kMaxStages];       // vectors (consecutive slots / positions) in the group: 1 per
                                // pipeline chain; >1 for batched prefill and EESD verify
  int32_t head_slot[2];         // [0] exit head input slot, [1] final head input slot
  int32_t head_out[2];          // argmax written by the head kernel
  int32_t vec_out[kMaxVec];     // kMatHeadV: argmax of each vector of group 0 (final head)
  int32_t src_slot;             // exit-head layer (head_copy_kernel): first row copied into slot[0]
};

struct LayerW {
  const __nv_bfloat16* qkv;
  const __nv_bfloat16* o;
  const __nv_bfloat16* gu;
  const __nv_bfloat16* down;
  const float* attn_norm;
  const float* mlp_norm;
  void* kc;  // [pages][KV][kPage][hd] in the KV dtype
  void* vc;
};

struct Dims {
  int32_t d, H, KV, hd, ffn, V, max_ctx, nslot;
  float eps;
  int32_t kv_bf16;
};

enum : int { kMatQKV = 0, kMatO = 1, kMatGU = 2, kMatDown = 3, kMatHead = 4, kMatHeadV = 5 };
constexpr int kNumMats = 6;
// gemv_kernel instantiation tag (not a matrix index): the down projection
// split over K across the two grid halves (GemvArgs.ksplit = 1)
constexpr int kMatDownS = 6;

struct GemvArgs {
  Work* work;
  int32_t layer_i;        // layer offset inside each stage
  int32_t desc_early;     // 1: the work descriptor was written >= 2 kernels ago
  int32_t mat;            // kMat*
  const LayerW* layers;   // [n_layers]
  const __nv_bfloat16* head_w;
  const float* head_norm0;  // exit norm
  const float* head_norm1;  // final norm
  int32_t R, K, nstage;
  int32_t sub;            // tiles (TR rows each) per bulk-copy stage
  Dims dm;
  float* x;   // [nslot][d]   residual stream (fp32)
  float* q;   // [nslot][H*hd]
  float* o;   // [nslot][H*hd]
  float* h;   // [nslot][ffn]
  float* logits;  // [2][V]
  const float* rope_cos;
  const float* rope_sin;
  const int32_t* page_table;
  float* head_part;  // [grid][kMaxVec][2] (value, index-as-float bits)
  int32_t* head_cnt; // [kMaxVec] arrival tickets
  // K split (wide down projections, ksplit = 1): the two halves of the grid
  // stream the two column halves [h*K, h*K + K) of rows k_ld long; the CTAs
  // streaming the second column half (low blockIdx, dispatched first)
  // publish their row sums (part_buf + a publication count), their partners
  // add them in fixed order before the residual add
  int32_t ksplit, k_ld;
  float* part_buf;     // [nslot][d]
  // [2][grid][kSplitChunks] monotone sequence numbers per (CTA pair, chunk
  // slot): [0] publications by the second-half CTA, [1] consumptions by its
  // partner. A wait is for "publications > consumptions", so a late or
  // stale publication can never be mistaken for a later one.
  int32_t* part_flag;
  int32_t* err;  // sticky device error word (kGemvErrSplitTimeout), checked by the host
};
constexpr int kSplitChunks = 64;  // epilogue chunk slots per CTA pair (sequence-numbered, may wrap)
constexpr int kGemvErrSplitTimeout = 1;

struct AttnArgs {
  const Work* work;
  int32_t layer_i;
  const LayerW* layers;
  Dims dm;
  const float* q;
  float* o;
  float* part;       // [nslot][H][max_pages][hd+2]
  int32_t* cnt;      // [nslot][KV]
  const int32_t* page_table;
  int32_t max_pages;
  // KV pool: [local layer][k | v][pages][KV][kPage][hd], layer stride 2 * kv_layer_bytes
  const void* kv_base;
  long long kv_layer_bytes;
  int32_t first_local;  // global index of the first local layer
  int32_t hl_global;    // exit-head layer: its global index (-1: none) ...
  int32_t hl_local;     // ... and its slot in the KV pool (after the local layers)
};

// tcgen05 prefill GEMM (umma.cu): one matrix of one layer for the chunk of
// up to 16 vectors in group 0 of `work`.
struct UmmaArgs {
  const Work* work;
  int32_t layer_i;
  int32_t mat;           // kMatQKV / kMatO / kMatGU / kMatDown
  int32_t R, K;
  const LayerW* layers;
  const void* wmaps;     // CUtensorMap [n_layers][4] over the weight matrices
  const void* xmap;      // CUtensorMap over xs
  __nv_bfloat16* xs;     // [32][K] activation operand: rows 0-15 hi, 16-31 lo
  Dims dm;
  float* x;
  float* q;
  float* o;
  float* h;
  const float* rope_cos;
  const float* rope_sin;
  const int32_t* page_table;
  float* ws;             // [grid][2][128][16] split-tile partials
  int32_t* cnt;          // [R / 128] arrival tickets
};

// Programmatic dependent launch (PDL): every kernel of a decode step is
// launched with programmatic stream serialization so it can be scheduled
// while its predecessor drains; kernels order their own accesses with
// griddepcontrol.wait / launch_dependents. Disable with PPSD_PDL=0.
extern bool g_pdl;

template <typename Kern, typename... Args>
cudaError_t launch_pdl(Kern fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, args...);
}

// launchers (gemv.cu / attn.cu)
// A GEMV plan: `m` = vectors per weight pass (1 for the decode tick; up to 4
// for batched prefill / EESD verify, where a group of nv vectors takes
// ceil(nv/m) passes).
int gemv_pick(int K, int R, int mat, int batched, int* vpt, int* tr, int* m, int* nstage, int* sub,
              size_t* smem);
cudaError_t gemv_launch(const GemvArgs& a, int vpt, int m, size_t smem, int grid, cudaStream_t st);
cudaError_t gemv_set_attrs(int vpt, int m, int mat, int ksplit, size_t smem);
cudaError_t attn_launch(const AttnArgs& a, int grid, cudaStream_t st);
cudaError_t attn_set_attrs(const AttnArgs& a);
bool umma_shape_ok(int R, int K);
int umma_encode_map(void* map, const void* base, int rows, int K, int box_rows);
size_t umma_map_bytes();
int umma_tile_rows();
int umma_n();
cudaError_t umma_set_attrs();
cudaError_t umma_launch(const UmmaArgs& a, int grid, cudaStream_t st);

}  // namespace ppsd
