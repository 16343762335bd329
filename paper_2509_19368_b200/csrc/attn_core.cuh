// attn_core.cuh — split-K decode attention over the paged KV cache, as a
// device routine run by a 128-thread worker (attn.cu runs one per CTA). Kept
// separate so other kernels can embed workers; measured on B200: fusing two
// workers into the O-projection GEMV (attention while its producer streams
// W_o, then a grid barrier) was 2% slower than the separate kernel, because
// the O ring dropped to two stages; one CTA per SM co-resident with the
// GEMVs was slower still (items run back to back per CTA).
//
// Work item = (stage group, vector, kv head, KV page). A KV page is kPage=64
// positions of one kv head stored contiguously ([page][kvh][64][hd]); an item
// pulls its K block and V block into shared memory with two 1-D bulk copies
// (UBLKCP, one mbarrier) — one DRAM round trip per item instead of a chain of
// dependent loads — then scores every q head that shares the kv head (GQA)
// against the block, takes a chunk-local softmax and accumulates V from smem.
// Page boundaries are absolute positions, so the partial results, and the
// ordered merge done by the worker that finishes a (chain, kv head) last,
// depend only on the context length — never on how many pipeline stages or
// vectors share the launch: PPSD and AR attention are bit-identical.
#pragma once
#include <float.h>

#include "kernels.cuh"

namespace ppsd {

template <typename T>
__device__ __forceinline__ void unpack16(const uint4& v, float* out);
template <>
__device__ __forceinline__ void unpack16<float>(const uint4& v, float* out) {
  out[0] = __uint_as_float(v.x); out[1] = __uint_as_float(v.y);
  out[2] = __uint_as_float(v.z); out[3] = __uint_as_float(v.w);
}
template <>
__device__ __forceinline__ void unpack16<__nv_bfloat16>(const uint4& v, float* out) {
  out[0] = bf16lo(v.x); out[1] = bf16hi(v.x); out[2] = bf16lo(v.y); out[3] = bf16hi(v.y);
  out[4] = bf16lo(v.z); out[5] = bf16hi(v.z); out[6] = bf16lo(v.w); out[7] = bf16hi(v.w);
}
__device__ __forceinline__ float tof(float v) { return v; }
__device__ __forceinline__ float tof(__nv_bfloat16 v) { return __bfloat162float(v); }

constexpr int kAttnThreads = 128;  // one attention worker
constexpr int kMergePages = 32;    // contexts up to 2048 positions merge from smem

// Timeline of each worker's first item (debugging: compiled in only with
// -DPPSD_ATTN_TRACE, enabled by ppsd_debug_tc_trace(5), read with -4):
// [worker][event] %globaltimer ns. Events: 0 start, 1 descriptor staged,
// 2 inputs visible, 3 q staged, 4 K/V landed, 5 scores, 6 softmax, 7 partial
// stored, 8 ticket taken, 9 merged (last worker), 10 item done
constexpr int kAttnTraceW = 1024;
static __device__ unsigned long long g_attn_tr[kAttnTraceW][12];
static __device__ int g_attn_tr_on;
__device__ __forceinline__ void attn_mark(int worker, int first, int tid, int ev) {
#ifdef PPSD_ATTN_TRACE
  if (g_attn_tr_on && first && tid == 0 && worker < kAttnTraceW) g_attn_tr[worker][ev] = globaltimer();
#else
  (void)worker; (void)first; (void)tid; (void)ev;
#endif
}

constexpr int kStageG = 32;      // groups staged in shared memory (more: read from global)
constexpr int kStagePages = 64;  // page-table entries staged

// per-worker shared scratch (besides the K/V page blocks)
template <int HD, int QPK>
struct AttnScratch {
  float qs[QPK][HD];
  float sc[QPK][kPage];
  float s_m[QPK], s_l[QPK];
  float s_lw[QPK][4];  // per-warp softmax sums (QPK < 4)
  float s_pm[QPK][kMergePages], s_pl[QPK][kMergePages];
  int s_last;
  uint64_t bar;
  // the work descriptor and page table, staged once per worker in one round
  // trip (the item walk would otherwise chain dependent global loads)
  int st_G;
  int st_slot[kStageG], st_pos[kStageG], st_first[kStageG], st_nl[kStageG], st_nv[kStageG];
  int st_page[kStagePages];
};

template <int HD, typename KVT>
constexpr size_t attn_kv_bytes() {
  return 2 * (size_t)kPage * HD * sizeof(KVT);
}

// work split of one page (attn_page): see the comments inside
template <int HD, typename KVT, int QPK>
struct AttnGeom {
  static constexpr int EPV = 16 / (int)sizeof(KVT);  // elements per 16-byte vector
  static constexpr int CPR = HD / EPV;                // 16-byte chunks per K / V row
  static_assert(CPR >= 1 && CPR <= 32 && (32 % CPR) == 0, "head_dim / dtype combination");
  // scores: LPT lanes per token, CPL chunks per lane; as few lanes as keep
  // the lane's q slice within 32 registers (fewer butterfly shuffles)
  static constexpr int LPT0 = (HD * QPK + 31) / 32;
  static constexpr int LPT1 = LPT0 <= 1 ? 1 : LPT0 <= 2 ? 2 : LPT0 <= 4 ? 4 : LPT0 <= 8 ? 8 : LPT0 <= 16 ? 16 : 32;
  static constexpr int LPT = LPT1 < CPR ? LPT1 : CPR;
  static constexpr int CPL = CPR / LPT;
  static constexpr int TPW = 32 / LPT;                // tokens per warp pass
  static constexpr int BLK = kPage * HD;              // elements per K (or V) page block
  static constexpr int NIT = (kPage + 4 * TPW - 1) / (4 * TPW);  // score passes per warp
  static constexpr int UC0 = 32 / (QPK * CPL) < 1 ? 1 : 32 / (QPK * CPL);  // unrolled tokens per chunk
  static constexpr int UC = NIT < UC0 ? NIT : UC0;
  static_assert(NIT % UC == 0, "score chunking");
  // PV: a thread accumulates one 16-byte V chunk (EPV dims) of one head over
  // every TS-th token; the TS token splits are added in order through the K
  // block (free once the scores are taken)
  static constexpr int NGRP = QPK * CPR;                             // (head, chunk) groups
  static constexpr int GT = NGRP < kAttnThreads ? NGRP : kAttnThreads;  // threads per split
  static constexpr int TS0 = kAttnThreads / GT;
  static constexpr int TSC0 = 16 * (int)sizeof(KVT) / QPK;            // splits that fit the K block
  static constexpr int TSC = TSC0 < 1 ? 1 : TSC0;
  static constexpr int TS = TS0 < TSC ? TS0 : TSC;
};

// One page of one (vector, kv head) row: scores of the QPK heads against
// the page's n K rows in ks (q rows staged in S.qs), chunk-local softmax,
// PV over vs. The page partial goes out through st_acc(head, dim, value)
// and st_stat(head, max, sum) (global split-K partials, or a cluster
// leader's shared memory): one arithmetic whoever merges it. Barriers over
// the 128 threads of the worker (`sync`); ks is scratch afterwards.
template <int HD, typename KVT, int QPK, class Sync, class Mark, class StAcc, class StStat>
__device__ __forceinline__ void attn_page(KVT* ks, const KVT* vs, AttnScratch<HD, QPK>& S, int n, int tid, Sync sync,
                                          Mark mark, StAcc st_acc, StStat st_stat) {
  using Gm = AttnGeom<HD, KVT, QPK>;
  constexpr int EPV = Gm::EPV, CPR = Gm::CPR, LPT = Gm::LPT, CPL = Gm::CPL, TPW = Gm::TPW, NIT = Gm::NIT,
                UC = Gm::UC, NGRP = Gm::NGRP, GT = Gm::GT, TS = Gm::TS;
  const int warp = tid >> 5, lane = tid & 31;
  const float scale = 1.0f / sqrtf((float)HD);
  // scores: LPT lanes per token, one 16-byte K vector per lane; the
  // lane's q slice sits in registers and a warp's tokens are unrolled in
  // chunks of UC (independent chains: the K loads of a chunk are in flight
  // together instead of one shared-memory round trip per token)
  {
    const int li = lane % LPT, tw = lane / LPT;
    // lane (li, tw) reads its chunks in the rotated order (s + f) % CPL,
    // f from the lane's place j in its 8-lane shared-memory wavefront: the
    // 8 lanes hit 8 distinct 16-byte bank groups; its q slice is loaded
    // once in the same order
    const int jq = lane & 7, f = CPL >= 8 ? jq : jq / (8 / (CPL < 8 ? CPL : 8));
    float qr[QPK][CPL][EPV];
#pragma unroll
    for (int i = 0; i < QPK; ++i)
#pragma unroll
      for (int sc = 0; sc < CPL; ++sc) {
        const int ch = li * CPL + (sc + f) % CPL;
#pragma unroll
        for (int e = 0; e < EPV; ++e) qr[i][sc][e] = S.qs[i][ch * EPV + e];
      }
#pragma unroll
    for (int c0 = 0; c0 < NIT; c0 += UC) {
      uint4 kv[UC][CPL];
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int tt = (warp + 4 * (c0 + u)) * TPW + tw;
#pragma unroll
        for (int sc = 0; sc < CPL; ++sc) {
          const int ch = li * CPL + (sc + f) % CPL;
          kv[u][sc] = tt < n ? lds128(ks + (size_t)tt * HD + ch * EPV) : make_uint4(0, 0, 0, 0);
        }
      }
      float part[UC][QPK];
#pragma unroll
      for (int u = 0; u < UC; ++u) {
#pragma unroll
        for (int i = 0; i < QPK; ++i) part[u][i] = 0.f;
#pragma unroll
        for (int sc = 0; sc < CPL; ++sc) {
          float kf[EPV];
          unpack16<KVT>(kv[u][sc], kf);
#pragma unroll
          for (int i = 0; i < QPK; ++i)
#pragma unroll
            for (int e = 0; e < EPV; ++e) part[u][i] = fmaf(kf[e], qr[i][sc][e], part[u][i]);
        }
      }
#pragma unroll
      for (int off = LPT / 2; off > 0; off >>= 1)
#pragma unroll
        for (int u = 0; u < UC; ++u)
#pragma unroll
          for (int i = 0; i < QPK; ++i) part[u][i] += __shfl_xor_sync(0xffffffffu, part[u][i], off);
#pragma unroll
      for (int u = 0; u < UC; ++u) {
        const int tt = (warp + 4 * (c0 + u)) * TPW + tw;
        if (li == 0 && tt < n)
#pragma unroll
          for (int i = 0; i < QPK; ++i) S.sc[i][tt] = part[u][i] * scale;
      }
    }
  }
  sync();
  mark(5);

  // chunk-local softmax statistics
  if constexpr (QPK >= 4) {  // one warp per head
    for (int i = warp; i < QPK; i += 4) {
      float mx = -FLT_MAX;
      for (int tt = lane; tt < n; tt += 32) mx = fmaxf(mx, S.sc[i][tt]);
      mx = warp_max(mx);
      float l = 0.f;
      for (int tt = lane; tt < n; tt += 32) {
        const float p = expf(S.sc[i][tt] - mx);
        S.sc[i][tt] = p;
        l += p;
      }
      l = warp_sum(l);
      if (lane == 0) { S.s_m[i] = mx; S.s_l[i] = l; }
    }
  } else {  // every warp takes the max, then exponentiates its 16 tokens
    static_assert(kPage == 64, "16 tokens per warp");
#pragma unroll
    for (int i = 0; i < QPK; ++i) {
      float mx = -FLT_MAX;
      for (int tt = lane; tt < n; tt += 32) mx = fmaxf(mx, S.sc[i][tt]);
      mx = warp_max(mx);
      const int tt = warp * 16 + (lane & 15);
      float p = 0.f;
      if (lane < 16 && tt < n) {
        p = expf(S.sc[i][tt] - mx);
        S.sc[i][tt] = p;
      }
#pragma unroll
      for (int off = 8; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
      if (lane == 0) {
        S.s_lw[i][warp] = p;
        if (warp == 0) S.s_m[i] = mx;
      }
    }
  }
  sync();
  if constexpr (QPK < 4) {
    if (tid < QPK) S.s_l[tid] = (S.s_lw[tid][0] + S.s_lw[tid][1]) + (S.s_lw[tid][2] + S.s_lw[tid][3]);
  }
  mark(6);

  // PV: thread -> (token split ts, group gi); group -> (head i, V chunk ch)
  if (tid < TS * GT) {
    const int ts = tid / GT;
    float* pvs = reinterpret_cast<float*>(ks);  // [TS][QPK * HD]
    for (int gi = tid % GT; gi < NGRP; gi += GT) {
      const int i = gi / CPR, ch = gi - i * CPR;
      float acc[EPV];
#pragma unroll
      for (int e = 0; e < EPV; ++e) acc[e] = 0.f;
      const KVT* vrow = vs + ch * EPV;
#pragma unroll 4
      for (int tt = ts; tt < n; tt += TS) {
        float vf[EPV];
        unpack16<KVT>(lds128(vrow + (size_t)tt * HD), vf);
        const float pp = S.sc[i][tt];
#pragma unroll
        for (int e = 0; e < EPV; ++e) acc[e] = fmaf(pp, vf[e], acc[e]);
      }
      if constexpr (TS == 1) {
#pragma unroll
        for (int e = 0; e < EPV; ++e) st_acc(i, ch * EPV + e, acc[e]);
      } else {
#pragma unroll
        for (int e = 0; e < EPV; ++e) pvs[ts * QPK * HD + gi * EPV + e] = acc[e];
      }
    }
  }
  if constexpr (TS > 1) {
    // the splits go through the K block with generic stores; the next
    // item's bulk copy rewrites it through the async proxy: every writer
    // orders its stores before that (CUTLASS's TMA-store fence pattern)
    fence_proxy_async_smem();
    sync();
    const float* pvs = reinterpret_cast<const float*>(ks);
    for (int idx = tid; idx < QPK * HD; idx += kAttnThreads) {
      float acc = pvs[idx];
#pragma unroll
      for (int t2 = 1; t2 < TS; ++t2) acc += pvs[t2 * QPK * HD + idx];
      const int i = idx / HD, d = idx - i * HD;
      st_acc(i, d, acc);
    }
  }
  if (tid < QPK) st_stat(tid, S.s_m[tid], S.s_l[tid]);
}

// Ordered merge of a row's nch page partials into out[QPK][HD]: rd(head,
// page, k) reads a partial (k < HD: the PV row, HD: the page max, HD + 1: the
// page sum), from global memory or a cluster leader's shared memory; the
// same arithmetic either way (page weights exp(m_c - M), in page order).
template <int HD, int QPK, class Sync, class Rd>
__device__ __forceinline__ void attn_merge(AttnScratch<HD, QPK>& S, int nch, float* out, int tid, Sync sync, Rd rd) {
  const int warp = tid >> 5, lane = tid & 31;
  if (nch <= kMergePages) {
    // one (head, dim) per thread: its page partials are loaded before the
    // page statistics are reduced (one L2 round trip for the merge)
    constexpr bool kPre = QPK * HD <= kAttnThreads;
    float pv[kPre ? kMergePages : 1];
    if constexpr (kPre) {
      if (tid < QPK * HD) {
#pragma unroll
        for (int cc = 0; cc < kMergePages; ++cc)
          if (cc < nch) pv[cc] = rd(tid / HD, cc, tid % HD);
      }
    }
    for (int idx = tid; idx < QPK * nch; idx += kAttnThreads) {
      const int i = idx / nch, cc = idx - i * nch;
      S.s_pm[i][cc] = rd(i, cc, HD);
      S.s_pl[i][cc] = rd(i, cc, HD + 1);
    }
    sync();
    for (int i = warp; i < QPK; i += 4) {
      float M = -FLT_MAX;
      for (int cc = lane; cc < nch; cc += 32) M = fmaxf(M, S.s_pm[i][cc]);
      M = warp_max(M);
      float Ls = 0.f;
      for (int cc = lane; cc < nch; cc += 32) {
        const float e = expf(S.s_pm[i][cc] - M);
        S.s_pm[i][cc] = e;  // page weight
        Ls = fmaf(S.s_pl[i][cc], e, Ls);
      }
      Ls = warp_sum(Ls);
      if (lane == 0) S.s_l[i] = Ls;
    }
    sync();
    if constexpr (kPre) {
      if (tid < QPK * HD) {
        const int i = tid / HD, d = tid % HD;
        float O = 0.f;
#pragma unroll
        for (int cc = 0; cc < kMergePages; ++cc)
          if (cc < nch) O = fmaf(pv[cc], S.s_pm[i][cc], O);
        out[i * HD + d] = O / S.s_l[i];
      }
    } else {
      for (int idx = tid; idx < QPK * HD; idx += kAttnThreads) {
        const int i = idx / HD, d = idx - i * HD;
        float O = 0.f;
#pragma unroll 4
        for (int cc = 0; cc < nch; ++cc) O = fmaf(rd(i, cc, d), S.s_pm[i][cc], O);
        out[i * HD + d] = O / S.s_l[i];
      }
    }
  } else {
    for (int idx = tid; idx < QPK * HD; idx += kAttnThreads) {
      const int i = idx / HD, d = idx - i * HD;
      float M = -FLT_MAX;
      for (int cc = 0; cc < nch; ++cc) M = fmaxf(M, rd(i, cc, HD));
      float Ls = 0.f, O = 0.f;
      for (int cc = 0; cc < nch; ++cc) {
        const float e = expf(rd(i, cc, HD) - M);
        Ls = fmaf(rd(i, cc, HD + 1), e, Ls);
        O = fmaf(rd(i, cc, d), e, O);
      }
      out[i * HD + d] = O / Ls;
    }
  }
}

// One worker (128 consecutive threads, `tid` in [0, 128)) processes items
// worker, worker + nworkers, ... `sync()` is a barrier over exactly these
// 128 threads. The scratch mbarrier must have been initialised (count 1)
// and fenced by the caller; `phase` carries its parity across calls.
// `wait_inputs()` makes the producing kernel's q / K / V rows visible
// (griddepcontrol.wait): the work descriptor (written by the scheduler >= 2
// kernels earlier) is staged and the first item's K/V copy is issued before
// it when that page holds no position this layer's QKV kernel writes.
template <int HD, typename KVT, int QPK, class Sync, class Wait>
__device__ void attn_items(const AttnArgs& a, int worker, int nworkers, int tid, KVT* ks,
                           AttnScratch<HD, QPK>& S, uint32_t& phase, Sync sync, Wait wait_inputs) {
  using Gm = AttnGeom<HD, KVT, QPK>;
  constexpr int EPV = Gm::EPV, BLK = Gm::BLK;
  KVT* vs = ks + BLK;
  const Work* w = a.work;
  const int warp = tid >> 5, lane = tid & 31;
  const int H = a.dm.H, KVh = a.dm.KV;
  const float scale = 1.0f / sqrtf((float)HD);

  attn_mark(worker, 1, tid, 0);
  // stage the descriptor + page table: independent loads, one round trip
  if (tid < kStageG) {
    S.st_slot[tid] = w->slot[tid];
    S.st_pos[tid] = w->pos[tid];
    S.st_first[tid] = w->first[tid];
    S.st_nl[tid] = w->nl[tid];
    S.st_nv[tid] = w->nv[tid];
  }
  if (tid == 0) S.st_G = w->G;
  for (int i = tid; i < min(a.max_pages, kStagePages); i += kAttnThreads) S.st_page[i] = a.page_table[i];
  sync();
  attn_mark(worker, 1, tid, 1);
  const int G = S.st_G;
  const bool staged = G <= kStageG;
  auto wslot = [&](int g) { return staged ? S.st_slot[g] : w->slot[g]; };
  auto wpos = [&](int g) { return staged ? S.st_pos[g] : w->pos[g]; };
  auto wfirst = [&](int g) { return staged ? S.st_first[g] : w->first[g]; };
  auto wnl = [&](int g) { return staged ? S.st_nl[g] : w->nl[g]; };
  auto wnv = [&](int g) { return staged ? S.st_nv[g] : w->nv[g]; };

  // items: (group, vector, kv head, page); vector v of group g sits at
  // slot[g]+v and position pos[g]+v (batched prefill / EESD / folded verify)
  struct Item {
    int g, vv, kvh, c, nch;
  };
  auto decode = [&](int item, Item& it) -> bool {
    int rem = item;
    for (int gg = 0; gg < G; ++gg) {
      if (wslot(gg) < 0 || a.layer_i >= wnl(gg)) continue;
      const int nvg = wnv(gg), pg = wpos(gg);
      for (int v = 0; v < nvg; ++v) {
        const int nch = (pg + v + kPage) / kPage;  // ceil((pos+1)/kPage)
        if (rem < nch * KVh) {
          it.g = gg;
          it.vv = v;
          it.nch = nch;
          it.kvh = rem / nch;
          it.c = rem - it.kvh * nch;
          return true;
        }
        rem -= nch * KVh;
      }
    }
    return false;
  };
  // rows [r0, r1) of the item's K and V page blocks (thread 0); `arrive`:
  // the copy that completes the item's mbarrier phase (arrive + its bytes),
  // else bytes only (the phase waits for the later arriving copy)
  auto issue_rows = [&](const Item& it, int r0, int r1, bool arrive) {
    // this layer's K / V caches: [k, v] per local layer, contiguous (engine.cu)
    const int gl = wfirst(it.g) + a.layer_i;
    const int lloc = gl == a.hl_global ? a.hl_local : gl - a.first_local;
    const char* kvl = static_cast<const char*>(a.kv_base) + a.kv_layer_bytes * (2 * (size_t)lloc);
    const int page = it.c < kStagePages ? S.st_page[it.c] : a.page_table[it.c];
    const size_t blk = ((size_t)page * KVh + it.kvh) * BLK + (size_t)r0 * HD;
    const uint32_t bytes = (uint32_t)((r1 - r0) * HD * sizeof(KVT));
    if (arrive) mbar_expect_tx(&S.bar, 2 * bytes);
    else mbar_expect_tx_only(&S.bar, 2 * bytes);
    if (bytes) {
      bulk_g2s(ks + (size_t)r0 * HD, reinterpret_cast<const KVT*>(kvl) + blk, bytes, &S.bar);
      bulk_g2s(vs + (size_t)r0 * HD, reinterpret_cast<const KVT*>(kvl + a.kv_layer_bytes) + blk, bytes, &S.bar);
    }
  };
  auto page_rows = [&](const Item& it) { return min(kPage, wpos(it.g) + it.vv + 1 - it.c * kPage); };
  Item it;
  bool have = decode(worker, it);
  // The rows of the first item's page below the group's first written
  // position are final: fetch them while the producing kernel drains; the
  // rows this layer's QKV kernel writes follow griddepcontrol.wait.
  const int early = have ? max(0, min(page_rows(it), wpos(it.g) - it.c * kPage)) : 0;
  if (early > 0 && tid == 0) issue_rows(it, 0, early, false);
  wait_inputs();
  attn_mark(worker, 1, tid, 2);

  for (int item = worker, first = 1; have; item += nworkers, have = decode(item, it), first = 0) {
    const int g = it.g, vv = it.vv, kvh = it.kvh, c = it.c, nch = it.nch;
    const int slot = wslot(g) + vv;
    const int n = page_rows(it);
    if (tid == 0) issue_rows(it, first ? early : 0, n, true);
    const float* qsrc = a.q + (size_t)slot * H * HD + (size_t)kvh * QPK * HD;
    for (int i = tid; i < QPK * HD; i += kAttnThreads) S.qs[i / HD][i % HD] = qsrc[i];
    sync();
    attn_mark(worker, first, tid, 3);
    mbar_wait(&S.bar, phase);
    phase ^= 1;
    attn_mark(worker, first, tid, 4);
    float* pbase = a.part + (((size_t)slot * H + (size_t)kvh * QPK) * a.max_pages) * (HD + 2);

    attn_page<HD, KVT, QPK>(
        ks, vs, S, n, tid, sync, [&](int m) { attn_mark(worker, first, tid, m); },
        [&](int i, int d, float v) { pbase[((size_t)i * a.max_pages + c) * (HD + 2) + d] = v; },
        [&](int i, float m, float l) {
          pbase[((size_t)i * a.max_pages + c) * (HD + 2) + HD] = m;
          pbase[((size_t)i * a.max_pages + c) * (HD + 2) + HD + 1] = l;
        });
    sync();
    attn_mark(worker, first, tid, 7);
    // arrival ticket: one acq_rel atomic (release: the CTA's partial stores,
    // ordered before it by the barrier; acquire: the other pages' partials
    // for the merge, made visible to the CTA by the barrier below)
    if (tid == 0) S.s_last = atom_add_acqrel_gpu(&a.cnt[slot * KVh + kvh], 1) == (uint32_t)(nch - 1);
    sync();
    attn_mark(worker, first, tid, 8);
    if (S.s_last) {  // ordered merge of the page partials (page statistics staged in smem)
      attn_merge<HD, QPK>(S, nch, a.o + (size_t)slot * H * HD + (size_t)kvh * QPK * HD, tid, sync,
                          [&](int i, int cc, int k) {
                            return __ldcg(pbase + ((size_t)i * a.max_pages + cc) * (HD + 2) + k);
                          });
      if (tid == 0) a.cnt[slot * KVh + kvh] = 0;
      attn_mark(worker, first, tid, 9);
    }
    sync();
    attn_mark(worker, first, tid, 10);
  }
}

}  // namespace ppsd
