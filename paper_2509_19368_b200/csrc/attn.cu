// attn.cu — standalone split-K decode attention kernel: one 128-thread
// worker (attn_core.cuh) per CTA. The persistent layer pass (tcpass.cu) runs
// the same worker code between its QKV and O phases.
#include "attn_core.cuh"
#include "tc_dev.cuh"

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

// Cluster decode attention: one thread-block cluster of CS CTAs per
// (group, kv head) row for one-vector groups (decode ticks, AR; CS 8), or
// per (group, vector, kv head) row for a bounded batch (a.multi: folded deep
// batches; CS 4). kClWorkers 128-thread page workers per CTA (1; 2 measured
// slower); worker w of rank r takes the row's pages r + CS w, r + CS (w + NW),
// ... with the split-K kernel's page arithmetic (attn_page) and stores each
// page partial into the cluster leader's shared memory over DSMEM. One
// cluster barrier replaces the global partials and the arrival ticket; the
// leader merges in page order (attn_merge), so results are bit-identical to
// attn_kernel (prefill chunks and EESD verify keep it). Rows past
// kMergePages pages keep global partials (the same merge reads them).
#ifndef PPSD_CL_WORKERS
#define PPSD_CL_WORKERS 1
#endif
constexpr int kClWorkers = PPSD_CL_WORKERS;  // page workers per CTA (A/B builds: -DPPSD_CL_WORKERS=2)
template <int HD, typename KVT, int QPK, int CS>
__global__ void __launch_bounds__(kAttnThreads* kClWorkers) attn_cl_kernel(const AttnArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ AttnScratch<HD, QPK> SW[kClWorkers];
  __shared__ int s_row[6];  // g, kv head, pos, local layer, slot, group's first pos (g < 0: idle row)
  using Gm = AttnGeom<HD, KVT, QPK>;
  constexpr int BLK = Gm::BLK, PS = HD + 2, NW = kClWorkers;
  const int tid = threadIdx.x, wk = tid >> 7, wt = tid & 127;
  AttnScratch<HD, QPK>& S = SW[wk];
  AttnScratch<HD, QPK>& S0 = SW[0];
  KVT* ks = reinterpret_cast<KVT*>(smem) + (size_t)wk * 2 * BLK;
  KVT* vs = ks + BLK;
  float* slots = reinterpret_cast<float*>(smem + (size_t)NW * 2 * BLK * sizeof(KVT));  // leader: [kMergePages][QPK][PS]
  const int rank = (int)cluster_rank(), row = (int)blockIdx.x / CS;
  const int H = a.dm.H, KVh = a.dm.KV;
  const Work* w = a.work;
  constexpr int kPg = kStagePages / (CS * NW);  // staged page-table entries per worker
  // the work descriptor and this CTA's page-table entries: independent
  // loads, one round trip (the descriptor was written >= 2 kernels ago)
  if (tid < kStageG) {
    S0.st_slot[tid] = w->slot[tid];
    S0.st_pos[tid] = w->pos[tid];
    S0.st_first[tid] = w->first[tid];
    S0.st_nl[tid] = w->nl[tid];
    S0.st_nv[tid] = w->nv[tid];
  } else if (tid >= 64 && tid < 64 + NW * kPg) {
    const int ww = (tid - 64) / kPg, k = (tid - 64) % kPg;
    const int c = rank + CS * ww + NW * CS * k;
    if (c < a.max_pages) SW[ww].st_page[k] = a.page_table[c];
  }
  if (tid == 32) S0.st_G = w->G;
  if (wt == 0) {
    mbar_init(&S.bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    // row -> (group, vector, kv head): active groups in order, KV rows per
    // vector (one vector per group unless a.multi: batched launches, vector
    // v of group g at slot[g] + v, position pos[g] + v)
    int r = row, g = -1, v = 0;
    const int G = min(S0.st_G, kStageG);
    for (int gg = 0; gg < G; ++gg) {
      if (S0.st_slot[gg] < 0 || a.layer_i >= S0.st_nl[gg]) continue;
      const int nvg = a.multi ? S0.st_nv[gg] : 1;
      if (r < nvg * KVh) {
        g = gg;
        v = r / KVh;
        r -= v * KVh;
        break;
      }
      r -= nvg * KVh;
    }
    if (blockIdx.x == 0 && a.err) {  // every active (vector, kv head) row must have a cluster
      int need = 0;
      for (int gg = 0; gg < G; ++gg)
        if (S0.st_slot[gg] >= 0 && a.layer_i < S0.st_nl[gg]) need += (a.multi ? S0.st_nv[gg] : 1) * KVh;
      if (need * CS > (int)gridDim.x || S0.st_G > kStageG) atomicOr(a.err, kAttnErrRows);
    }
    s_row[0] = g;
    s_row[1] = r;
    if (g >= 0) {
      s_row[2] = S0.st_pos[g] + v;
      const int gl = S0.st_first[g] + a.layer_i;
      s_row[3] = gl == a.hl_global ? a.hl_local : gl - a.first_local;
      s_row[4] = S0.st_slot[g] + v;
      s_row[5] = S0.st_pos[g];
    }
  }
  __syncthreads();
  const int g = s_row[0], kvh = s_row[1];
  const int pos = g >= 0 ? s_row[2] : 0, slot = g >= 0 ? s_row[4] : 0;
  const int nch = g >= 0 ? (pos + kPage) / kPage : 0;
  const bool dsm = nch <= kMergePages;
  const char* kvl = static_cast<const char*>(a.kv_base) + a.kv_layer_bytes * (2 * (size_t)(g >= 0 ? s_row[3] : 0));
  const int c0 = rank + CS * wk;  // this worker's first page
  auto issue_rows = [&](int c, int r0, int r1, bool arrive) {
    const int k = (c - c0) / (NW * CS);
    const int page = k < kPg ? S.st_page[k] : a.page_table[c];
    const size_t blk = ((size_t)page * KVh + kvh) * BLK + (size_t)r0 * HD;
    const uint32_t bytes = (uint32_t)((r1 - r0) * HD * sizeof(KVT));
    if (arrive) mbar_expect_tx(&S.bar, 2 * bytes);
    else mbar_expect_tx_only(&S.bar, 2 * bytes);
    if (bytes) {
      bulk_g2s(ks + (size_t)r0 * HD, reinterpret_cast<const KVT*>(kvl) + blk, bytes, &S.bar);
      bulk_g2s(vs + (size_t)r0 * HD, reinterpret_cast<const KVT*>(kvl + a.kv_layer_bytes) + blk, bytes, &S.bar);
    }
  };
  auto page_rows = [&](int c) { return min(kPage, pos + 1 - c * kPage); };
  auto sync = [wk] { named_bar_sync(1 + wk, kAttnThreads); };
  // rows of the first page below the group's first position written by this
  // layer (earlier vectors of the group write theirs too): before the wait
  const int pos0 = g >= 0 ? s_row[5] : 0;
  const int early = c0 < nch ? max(0, min(page_rows(c0), pos0 - c0 * kPage)) : 0;
  if (early > 0 && wt == 0) issue_rows(c0, 0, early, false);
  pdl_wait();
  pdl_trigger();
  float* pglob = a.part + (((size_t)slot * H + (size_t)kvh * QPK) * a.max_pages) * PS;
  const uint32_t slots_lead = map_rank(smem_u32(slots), 0);
  uint32_t phase = 0;
  for (int c = c0; c < nch; c += NW * CS) {
    const int n = page_rows(c);
    if (wt == 0) issue_rows(c, c == c0 ? early : 0, n, true);
    if (c == c0)
      for (int i = wt; i < QPK * HD; i += kAttnThreads)
        S.qs[i / HD][i % HD] = a.q[(size_t)slot * H * HD + (size_t)kvh * QPK * HD + i];
    sync();
    mbar_wait(&S.bar, phase);
    phase ^= 1;
    if (dsm) {
      attn_page<HD, KVT, QPK>(
          ks, vs, S, n, wt, sync, [](int) {},
          [&](int i, int d, float v) { st_cluster_f32(slots_lead + (uint32_t)(((c * QPK + i) * PS + d) * 4), v); },
          [&](int i, float m, float l) {
            st_cluster_f32(slots_lead + (uint32_t)(((c * QPK + i) * PS + HD) * 4), m);
            st_cluster_f32(slots_lead + (uint32_t)(((c * QPK + i) * PS + HD + 1) * 4), l);
          });
    } else {
      attn_page<HD, KVT, QPK>(
          ks, vs, S, n, wt, sync, [](int) {},
          [&](int i, int d, float v) { pglob[((size_t)i * a.max_pages + c) * PS + d] = v; },
          [&](int i, float m, float l) {
            pglob[((size_t)i * a.max_pages + c) * PS + HD] = m;
            pglob[((size_t)i * a.max_pages + c) * PS + HD + 1] = l;
          });
    }
    sync();  // the next page's copy reuses ks / vs
  }
  // every worker's partials (DSMEM or global) before the leader merges
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank == 0 && wk == 0 && nch > 0) {
    float* out = a.o + (size_t)slot * H * HD + (size_t)kvh * QPK * HD;
    if (dsm)
      attn_merge<HD, QPK>(S0, nch, out, wt, sync, [&](int i, int cc, int k) { return slots[(cc * QPK + i) * PS + k]; });
    else
      attn_merge<HD, QPK>(S0, nch, out, wt, sync,
                          [&](int i, int cc, int k) { return __ldcg(pglob + ((size_t)i * a.max_pages + cc) * PS + k); });
  }
}

namespace {
int g_attn_occ = 0;
int g_attn_cl_cs = 0;  // cluster size of the cluster kernel (0: unavailable)
bool g_attn_cl4 = false;  // clusters of 4 available (batched launches)

template <int HD, typename KVT, int QPK, int CS>
size_t cl_smem() {
  return kClWorkers * 2 * (size_t)kPage * HD * sizeof(KVT) + (size_t)kMergePages * QPK * (HD + 2) * sizeof(float);
}

template <int HD, typename KVT, int QPK, int CS>
cudaError_t launch_cl(const AttnArgs& a, int rows, cudaStream_t st, bool attrs) {
  auto fn = attn_cl_kernel<HD, KVT, QPK, CS>;
  const size_t smem = cl_smem<HD, KVT, QPK, CS>();
  if (attrs) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && CS > 8) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS * 8);
    cfg.blockDim = dim3(kAttnThreads * kClWorkers);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    e = cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg);
    if (e == cudaSuccess && ncl > 0) g_attn_cl_cs = CS;
    return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(rows * CS);
  cfg.blockDim = dim3(kAttnThreads * kClWorkers);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = CS;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, fn, a);
}

// the cluster kernel for (hd, dtype, qpk): hd 128 and qpk <= 2 (the leader's
// page slots must fit shared memory); cluster size 16, else 8. Launches may
// ask for clusters of 4 (cs = 4: batched launches, more rows per wave).
template <typename KVT, int QPK>
cudaError_t cl_qpk(const AttnArgs& a, int rows, cudaStream_t st, bool attrs, int cs) {
  if (attrs) {
    g_attn_cl_cs = 0;
    // clusters of 4 for the batched launches (attributes only)
    launch_cl<128, KVT, QPK, 4>(a, rows, st, true);
    cudaGetLastError();
    g_attn_cl4 = g_attn_cl_cs == 4;
    g_attn_cl_cs = 0;
    // clusters of 8 (portable; 16 measured ~3 us slower per launch), PPSD_ATTN_CL=16 to compare
    const char* v = getenv("PPSD_ATTN_CL");
    cudaError_t e = cudaSuccess;
    if (v && atoi(v) == 16) e = launch_cl<128, KVT, QPK, 16>(a, rows, st, true);
    cudaGetLastError();
    if (g_attn_cl_cs == 0) e = launch_cl<128, KVT, QPK, 8>(a, rows, st, true);
    cudaGetLastError();
    return g_attn_cl_cs ? cudaSuccess : (e == cudaSuccess ? cudaErrorNotSupported : e);
  }
  if (cs == 4) return g_attn_cl4 ? launch_cl<128, KVT, QPK, 4>(a, rows, st, false) : cudaErrorNotSupported;
  return g_attn_cl_cs == 16 ? launch_cl<128, KVT, QPK, 16>(a, rows, st, false)
                            : launch_cl<128, KVT, QPK, 8>(a, rows, st, false);
}
cudaError_t cl_dispatch(const AttnArgs& a, int rows, cudaStream_t st, bool attrs, int cs = 0) {
  if (a.dm.hd != 128) return cudaErrorNotSupported;
  const int qpk = a.dm.H / a.dm.KV;
  if (qpk == 1)
    return a.dm.kv_bf16 ? cl_qpk<__nv_bfloat16, 1>(a, rows, st, attrs, cs) : cl_qpk<float, 1>(a, rows, st, attrs, cs);
  if (qpk == 2)
    return a.dm.kv_bf16 ? cl_qpk<__nv_bfloat16, 2>(a, rows, st, attrs, cs) : cl_qpk<float, 2>(a, rows, st, attrs, cs);
  return cudaErrorNotSupported;
}  // attn_set_attrs: resident CTAs per SM of the configured instantiation

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

// cluster kernel: attrs once per engine (returns false when unavailable for
// the shape), launch with `rows` >= the active one-vector (group, kv head) rows
bool attn_cl_setup(const AttnArgs& a) { return cl_dispatch(a, 0, 0, true) == cudaSuccess; }
bool attn_cl4_ok() { return g_attn_cl4; }
cudaError_t attn_cl_launch(const AttnArgs& a, int rows, cudaStream_t st, int cs) {
  return cl_dispatch(a, rows, st, false, cs);
}

}  // namespace ppsd
