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
  // rank fold (sched.h: sched_rfold_plan), written by the scheduler kernel:
  // `work` = the eager stages of the chain reaching stage lo, `work_deep` =
  // the deferred batch; the box of this tick carries row out_row (-1: none),
  // the exit token exit_tok (-2: this tick's exit head, -1: not the owner) and
  // the final token vec_out[final_idx] of work_deep (-1: none); rf_src: the
  // batch chains' activation slots, gathered into the batch rows
  int32_t out_row, out_slot, out_pos, exit_tok, final_idx;
  // folded tick with a deep batch: the exit head of this row runs as vector 0
  // of the final-head launch (GemvArgs.comb_exit), -1: none
  int32_t head_exit;
  int32_t rf_src[kMaxVec];
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

constexpr int kTcMaxWp = 128;  // layers (incl. the exit-head layer) whose weight pointers ride in the launch

// the next GEMV of the decoder layer, for the producer's L2 prefetch
struct TcNext {
  const void* wbase;     // layer 0's matrix; nullptr: no prefetch
  long long wstride;     // bytes between layers
  int32_t wn;            // layers [0, wn) at the stride
  int32_t dli;           // layer offset from this launch's (0: same layer, 1: next layer)
  int32_t R, js, nj, tg, cs;
  int32_t bytes;         // per CTA
};

struct GemvArgs {
  Work* work;
  int32_t layer_i;        // layer offset inside each stage
  int32_t desc_early;     // 1: the work descriptor was written >= 2 kernels ago
  int32_t mat;            // kMat*
  const LayerW* layers;   // [n_layers]
  const __nv_bfloat16* head_w;
  const float* head_norm0;  // exit norm
  const float* head_norm1;  // final norm
  int32_t R, K, nstage;   // matrix [R][K], weight-ring stages
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
  int32_t* err;  // sticky device error word (kGemvErr*), checked by the host
  // tensor-core GEMV (tcgemv.cu): TC-tiled weight layout and ring plan
  int32_t js, nj;       // 64-wide K slabs per J-block, J-blocks
  int32_t nb, tg;       // J-blocks per ring stage, max 8-row groups per tile
  int32_t nblk;         // 16-column B blocks reserved per stage (<= 3: 16 vectors x 3 parts)
  int32_t bar_off;      // smem offset of the mbarriers
  // this matrix's weights per global layer index (launch parameters: the
  // producer issues its first copy without a dependent load of LayerW)
  const void* wp[kTcMaxWp];
  // ... or, when every layer's matrix sits at a fixed stride from layer 0's
  // (one allocation per matrix kind), base + layer * stride for layers < wn
  const void* wbase;
  long long wstride;
  int32_t wn;
  // >= 0: the launch has at most one problem, layer hint_li (any value for
  // the heads): the producer starts streaming before reading the descriptor
  int32_t hint_li;
  // kMatHeadV: vector 0 is the exit head of work->head_exit when >= 0 (logits
  // rows: exit 0, batch 1..)
  int32_t comb_exit;
  // L2 prefetch of the NEXT GEMV's weights (this CTA's slice of its first
  // nx_bytes), issued after this launch's last copy: it lands while the
  // launch drains, the next launch starts and (QKV -> O) attention runs
  TcNext nx;
};

// tensor-core GEMV plan (tcgemv.cu: tc_pick)
struct TcPlan {
  int R = 0, K = 0, js = 1, nj = 0, nb = 1, tg = 1, nblk = 1, ns = 0, bar_off = 0, cs = 1, grid = 0;
  size_t smem = 0;
};
constexpr int kGemvErrPassTimeout = 2;  // a layer-pass grid barrier waited > 5 s
constexpr int kGemvErrHint = 4;         // a speculative-start hint did not match the work descriptor
constexpr int kAttnErrRows = 8;         // a cluster attention launch had fewer rows than active vectors

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
  int32_t multi;        // cluster kernel: rows enumerate every vector of a group (batched launches)
  int32_t* err;         // sticky device error word (kAttnErrRows), checked by the host
};

// one matrix of the persistent layer pass (tcpass.cu); the arithmetic plan
// (js, nj, cs) is the standalone GEMV's, tg / nb follow the pass's ring
struct TcPassMat {
  int32_t R, K, js, nj, tg, nb, cs, wn;
  const void* wbase;  // layers at a fixed stride (else LayerW)
  long long wstride;
};
struct TcPassArgs {
  GemvArgs g;          // shared fields: work, layers, dims, activations, RoPE, page table, err
  AttnArgs at;         // attention of the pass (layer_i set per slot)
  TcPassMat mat[4];    // kMatQKV, kMatO, kMatGU, kMatDown
  int32_t n_slots;     // layer slots (layer_i = 0 .. n_slots-1 of every active group)
  int32_t desc_early;  // 1: the work descriptor was written >= 2 kernels ago
  int32_t ns, slot_bytes, b_stage, nblk;  // weight ring slots, operand stage bytes, B blocks
  int32_t attn_off, attn_kv_bytes, scr_off, bar_off, attn_workers;
  unsigned long long prefetch_bytes;  // L2 prefetch distance of the weight producer (bytes ahead)
  unsigned long long* bar_cnt;  // grid-barrier arrivals (monotone)
  unsigned long long* bar_seq;  // arrivals at the end of the previous pass
  uint32_t* done_cnt;           // CTAs finished (the last publishes bar_seq)
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

// launchers (tcgemv.cu / tcpass.cu / attn.cu)
// TC-tiled weight layout (tcgemv.cu header comment): K padded to KP
// (multiple of 64) and cut into J-blocks of JS 64-wide slabs, rows into
// 8-row groups; element (r, k) sits in the 1 KB SWIZZLE_128B atom
// [k / (64 JS)][r / 8][(k / 64) % JS], row r % 8, 16-byte chunk
// ((k % 64) / 8) ^ (r % 8). JS = 4 where K allows (one CTA's J-block copy
// is tg * 4 KB); a property of the matrix shape only.
__host__ __device__ inline void tc_layout(int R, int K, int* js, int* kp) {
  (void)R;
  const int KP = (K + 63) / 64 * 64, NSL = KP / 64;
  *js = NSL % 4 == 0 ? 4 : NSL % 2 == 0 ? 2 : 1;
  *kp = KP;
}
// element offset of (r, k) in a TC-tiled [R][K] matrix
__host__ __device__ inline long long tc_offset(int R, int K, long long r, long long k) {
  int JS, KP;
  tc_layout(R, K, &JS, &KP);
  const long long G = R / 8;
  const long long slab = k / 64, j = slab / JS, s = slab % JS, g = r / 8, rr = r % 8, c = (k % 64) / 8, e = k % 8;
  return ((((j * G + g) * JS + s) * 8 + rr) * 64) + ((c ^ rr) * 8) + e;
}

// tensor-core GEMV (tcgemv.cu); weights in the TC-tiled layout
int tc_pick(int K, int R, int nblk, int grid, TcPlan* p, int mat = -1);
cudaError_t tc_set_attrs(int mat, int cs, size_t smem);
cudaError_t tc_launch(const GemvArgs& a, int cs, size_t smem, int grid, cudaStream_t st);
bool tc_pass_supported(int hd, int qpk);
size_t tc_pass_scratch_bytes(int hd, int qpk, int kv_bf16);
cudaError_t tc_pass_set_attrs(int cs, int hd, int qpk, int kv_bf16, size_t smem);
cudaError_t tc_pass_launch(const TcPassArgs& a, int cs, int hd, int qpk, int kv_bf16, size_t smem, int grid,
                           cudaStream_t st);
cudaError_t attn_launch(const AttnArgs& a, int grid, cudaStream_t st);
cudaError_t attn_set_attrs(const AttnArgs& a);
int attn_ctas_per_sm();
bool attn_cl_setup(const AttnArgs& a);
bool attn_cl4_ok();  // clusters of 4 (batched launches) after attn_cl_setup
cudaError_t attn_cl_launch(const AttnArgs& a, int rows, cudaStream_t st, int cs = 0);
int attn_trace_enable(int on);
int attn_trace_read(unsigned long long* out);

}  // namespace ppsd
