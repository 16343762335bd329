// tcgemv.cu — tcgen05 (5th-gen tensor core) weight-streaming GEMV for the
// decode step, one arithmetic for every vector count (1 .. 16).
//
// Every decode matmul is y_v = W x_v, W bf16 [R][K] streamed from HBM once
// per launch, x_v fp32 (RMS-normalised on the fly for QKV / gate-up / head).
// The weights are the MMA's A operand (M = 128 rows = 16 groups of 8 rows),
// the vectors its B operand (N = 16 columns):
//
//   D[128 rows][16 cols] (fp32, TMEM) += W_tile[128][16] . Xs[16 cols][16]^T
//
// Exact fp32 activations: each x is split into three bf16 parts
// (hi = bf16(x), mid = bf16(x - hi), lo = bf16(x - hi - mid); hi + mid + lo
// = x exactly) which take three B columns; the products with the bf16
// weights are exact and the epilogue adds the three column sums in fixed
// order, y = (d_hi + d_mid) + d_lo. Five vectors share one 16-column block,
// so 1-5 vectors cost ONE MMA per 16-wide K step, 16 vectors four.
//
// Batch invariance (PPSD == AR token for token): a row's result depends
// only on its own weights and vector — every row is reduced over the whole
// K by ONE CTA, in the same J-block / K-step order, by the same MMA shape,
// whatever the number of vectors, groups or CTAs in the launch. The MMA
// columns do not interact.
//
// Weight layout in HBM ("TC-tiled", written by ppsd_init_weight): K is
// padded to KP (multiple of 64) and cut into J-blocks of JS 64-wide slabs;
// rows into groups of 8. Element (r, k) lives in the 1 KB swizzle atom
// [J = k / (64 JS)][group g = r / 8][slab s] at row r % 8, 16-byte chunk
// ((k % 64) / 8) ^ (r % 8) — exactly the canonical K-major SWIZZLE_128B
// layout the MMA reads. A CTA's row groups [g0, g0 + tg) of one J-block are
// therefore ONE contiguous tg * JS KB block: the producer streams them with
// plain bulk copies (UBLKCP), no tensor maps.
//
// One CTA per SM, 320 threads:
//   warp 0 (one lane)   bulk-copy producer into an NS-deep ring of stages
//                       (nb J-blocks of the tile's groups per stage); starts
//                       before griddepcontrol.wait (weights never depend on
//                       the previous kernel).
//   warp 1              TMEM owner (128 columns: two 64-column accumulators)
//                       and, on one lane, the MMA issuer: per 16-wide K step
//                       one tcgen05.mma.cta_group::1.kind::f16 M=128 N=16 per
//                       vector block; tcgen05.commit frees ring stages and
//                       publishes finished accumulators.
//   warps 2-5           operand builders: per stage, the vectors' K slice
//                       (normalised) split into hi/mid/lo bf16, stored in the
//                       swizzled B layout, fence.proxy.async, arrive.
//   warps 6-9           epilogue: tcgen05.ld 32x32b (one TMEM lane = one weight
//                       row per thread, 16 columns per block), then the fused
//                       epilogues: RoPE + paged-KV append (QKV), SwiGLU (gate/
//                       up), residual add (O, down), logits + first-index
//                       argmax across CTAs (heads).
//
// Work split: the 8-row groups of all problems of the launch (the same layer
// slot of every stage with a chain this tick; one problem per group of
// vectors) are cut into one contiguous range per CTA; a CTA's range is
// processed as tiles of <= TG groups (TG <= 16), each tile over the whole K.
#include <float.h>
#include <limits.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "tc_dev.cuh"

namespace ppsd {

// this launch's matrix for global layer li (the LM head: head_w)
template <int EPI>
__device__ __forceinline__ const unsigned char* tc_weights_t(const GemvArgs& a, int li) {
  if constexpr (EPI == kMatHead || EPI == kMatHeadV) {
    return reinterpret_cast<const unsigned char*>(a.head_w);
  } else {
    if (a.wstride && li < a.wn)  // layers at a fixed stride: no dependent load
      return reinterpret_cast<const unsigned char*>(a.wbase) + (size_t)li * a.wstride;
    if (a.wp[0] && li < kTcMaxWp)  // launch parameter
      return reinterpret_cast<const unsigned char*>(a.wp[li]);
    const LayerW& L = a.layers[li];
    return reinterpret_cast<const unsigned char*>(EPI == kMatQKV ? L.qkv : EPI == kMatO ? L.o
                                                  : EPI == kMatGU ? L.gu : L.down);
  }
}
#define tc_weights(a, li) tc_weights_t<EPI>(a, li)

template <int EPI, int CS>
__global__ void __launch_bounds__(kTcThreads, 1) tcgemv_kernel(const GemvArgs a) {
  constexpr bool kHead2 = EPI == kMatHead;   // PPSD tick: exit (v=0) + final (v=1) head
  constexpr bool kHeadV = EPI == kMatHeadV;  // final head on the vectors of group 0
  constexpr bool kHead = kHead2 || kHeadV;
  constexpr bool kNorm = EPI == kMatQKV || EPI == kMatGU || kHead;
  extern __shared__ unsigned char tc_smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ int s_pg[kTcMaxProb], s_nv[kTcMaxProb], s_li[kTcMaxProb];  // group, vectors, layer
  __shared__ int s_np;
  __shared__ uint32_t s_taddr;
  __shared__ float s_ss[4][kMaxVec];
  __shared__ float s_rstd[kMaxVec];
  __shared__ float s_bv[4][kMaxVec];
  __shared__ int s_bi[4][kMaxVec];
  __shared__ int s_last;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = a.K, G = a.R >> 3, NS = a.nstage;
  const int JS = a.js, NJ = a.nj, NB = a.nb, TG = a.tg, NBLK = a.nblk;
  const uint32_t JSB = (uint32_t)JS << 10;                  // bytes of one group's J-block
  const uint32_t w_stage = (uint32_t)NB * TG * JSB;         // weight bytes per ring stage
  const uint32_t b_stage = (uint32_t)NB * NBLK * JS * 2048;  // operand bytes per ring stage
  const uint32_t ring_w = smem_u32(smem);
  const uint32_t ring_b = ring_w + (uint32_t)NS * w_stage;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  uint64_t* empty = full + NS;
  uint64_t* acc_full = empty + NS;  // [2]
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* recv_full = acc_empty + 2;   // CS > 1, leader: partials of the other ranks landed
  uint64_t* recv_empty = recv_full + 1;  // CS > 1, other ranks: the leader consumed the last partials
  // CS > 1: the leader's receive buffer [CS-1][kMaxVec][128 rows] fp32 (after the barriers)
  float* recv = reinterpret_cast<float*>(smem + a.bar_off + 256);
  const Work* work = a.work;

  if (tid == 0) {
    tc_trace(6, 0);
    tc_cta_mark(0);
  }
  // Speculative start (a.hint_li >= 0: the caller guarantees the launch has
  // at most one problem, layer hint_li / the LM head): the producer issues
  // the first ring stages before reading the work descriptor (and, for the
  // first kernel of a tick, before the scheduler kernel has finished).
  __shared__ int s_spec;  // stages issued speculatively
  __shared__ int s_ex;    // kHeadV: 1 if vector 0 is a combined exit head
  int spec_n = 0;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 2);      // producer (expect_tx) + the builder warp of the stage
      mbar_init(&empty[i], 1);     // MMA commit
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);  // epilogue warps
    }
    if (CS > 1) {
      mbar_init(recv_full, 4 * (CS - 1));  // every epilogue warp of the other ranks
      mbar_init(recv_empty, 4);            // the leader's epilogue warps
    }
    fence_mbar_init();
    const unsigned char* wsp = nullptr;
    if (a.hint_li >= 0) {
      if (kHead) wsp = reinterpret_cast<const unsigned char*>(a.head_w);
      else if (a.wstride && a.hint_li < a.wn)
        wsp = reinterpret_cast<const unsigned char*>(a.wbase) + (size_t)a.hint_li * a.wstride;
    }
    if (wsp) {  // the first tile of this CTA's share of one problem
      const int sc = CS > 1 ? (int)cluster_rank() : 0;
      const int snc = (int)gridDim.x / CS, sb = (int)blockIdx.x / CS;
      const int su0 = (int)((unsigned)(G * sb) / (unsigned)snc), su1 = (int)((unsigned)(G * (sb + 1)) / (unsigned)snc);
      const int sjlo = NJ * sc / CS, sjhi = NJ * (sc + 1) / CS;
      TcTiles tl;
      tl.init(su0, su1, G, TG);
      int tp, g0, tg;
      if (su0 < su1 && tl.next(tp, g0, tg)) {
        const uint64_t pol = policy_evict_first();
        const uint32_t tb = (uint32_t)tg * JSB;
        for (int j = sjlo; j < sjhi && spec_n < NS; j += NB, ++spec_n) {
          const int nbj = min(NB, sjhi - j);
          mbar_expect_tx(&full[spec_n], (uint32_t)nbj * tb);
          for (int jj = 0; jj < nbj; ++jj)
            bulk_g2s(smem + (size_t)spec_n * w_stage + (size_t)jj * tb, wsp + ((size_t)(j + jj) * G + g0) * JSB, tb,
                     &full[spec_n], pol);
        }
      }
    }
  }
  if (!a.desc_early) pdl_wait();
  if (tid == 0) {
    int np = 0;
    if (kHead2) {
      if (work->head_slot[0] >= 0 || work->head_slot[1] >= 0) { s_pg[0] = -1; s_nv[0] = 2; np = 1; }
    } else if (kHeadV) {
      // a.comb_exit: vector 0 is the exit head of row work->head_exit (if >= 0),
      // the batch follows (the folded tick's exit + final heads in one pass)
      const int ex = a.comb_exit && work->head_exit >= 0 ? 1 : 0;
      s_ex = ex;
      if (work->G >= 1 && work->slot[0] >= 0 && work->nv[0] > 0) { s_pg[0] = 0; s_nv[0] = work->nv[0] + ex; np = 1; }
    } else {
      for (int g = 0; g < work->G && np < kTcMaxProb; ++g)
        if (work->slot[g] >= 0 && a.layer_i < work->nl[g] && work->nv[g] > 0) {
          s_pg[np] = g;
          s_li[np] = work->first[g] + a.layer_i;
          s_nv[np++] = work->nv[g];
        }
    }
    if (spec_n > 0 && np == 1 && !kHead && s_li[0] != a.hint_li) {
      // a wrong hint is a caller bug: flag it (the decode reports PPSD_ESTATE)
      // and run nothing; the speculative copies are drained below
      atomicOr(a.err, kGemvErrHint);
      np = 0;
    }
    if (np > 1 && spec_n > 0) {
      atomicOr(a.err, kGemvErrHint);
      np = 0;
    }
    s_spec = np == 1 ? spec_n : 0;
    s_np = np;
    if (np == 0 && spec_n > 0) {  // nothing to do: let the copies land before exit
      for (int i = 0; i < spec_n; ++i) {
        mbar_arrive(&full[i]);
        mbar_wait(&full[i], 0);
      }
    }
    tc_trace(7, 0);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_taddr)),
                 "n"(kTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // warp 0 (the producer) publishes the problem list and the barriers and
  // goes straight on to stream weights; the other warps wait for them (and
  // for the TMEM allocation)
  tc_fence_before_sync();
  if (warp == 0) {
    __syncwarp();
    asm volatile("bar.arrive 3, %0;" ::"n"(kTcThreads) : "memory");
  } else {
    named_bar_sync(3, kTcThreads);
  }
  if (tid == 0) tc_trace(7, 2);
  // every rank's barriers are initialised before any remote arrival: arrive
  // here, wait only where remote traffic starts (the epilogue) or at the end
  if (CS > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  if (tid == 0) tc_trace(7, 3);
  tc_fence_after_sync();
  const int np = s_np;
  const uint32_t taddr = s_taddr;
  const int U = np * G;
  // split-K: the CS CTAs of a cluster share the cluster's tiles; rank r
  // reduces J-blocks [NJ r / CS, NJ (r+1) / CS) and the leader (rank 0) adds
  // the ranks' row sums in rank order
  const int crank = CS > 1 ? (int)cluster_rank() : 0;
  const int ncl = (int)gridDim.x / CS, b = (int)blockIdx.x / CS;  // clusters, this cluster
  // (32-bit: U * ncl < 2^31 for every plan; a 64-bit division is a slow subroutine)
  const int u0 = (int)((unsigned)(U * b) / (unsigned)ncl), u1 = (int)((unsigned)(U * (b + 1)) / (unsigned)ncl);
  const int ncta = U < ncl ? U : ncl;  // clusters with work (heads: argmax tickets)
  const int jlo = NJ * crank / CS, jhi = NJ * (crank + 1) / CS;

  if (u0 < u1) {
    if (warp == 0) {  // ---------------- bulk-copy producer ----------------
      if (lane == 0) {
        tc_trace(7, 5);
        const uint64_t pol = policy_evict_first();
        tc_trace(7, 6);
        TcTiles tl;
        tl.init(u0, u1, G, TG);
        int tp, g0, tg, n = 0;
        bool triggered = false;
        while (tl.next(tp, g0, tg)) {
          if (n == 0) tc_trace(7, 7);
          const unsigned char* w = tc_weights(a, kHead ? 0 : s_li[tp]);
          const uint32_t tb = (uint32_t)tg * JSB;
          tc_trace(7, 4);
          for (int j = jlo; j < jhi; j += NB, ++n) {
            const int nbj = min(NB, jhi - j);
            const int st = n % NS;
            if (n >= s_spec) {  // (stages below s_spec were issued before the descriptor was read)
              if (n >= NS) mbar_wait(&empty[st], ((n / NS) & 1) ^ 1);
              if (tc_exp() & 1) {
                mbar_arrive(&full[st]);
              } else {
                mbar_expect_tx(&full[st], (uint32_t)nbj * tb);
                if (n == 0) tc_trace(7, 8);
                for (int jj = 0; jj < nbj; ++jj) {
                  bulk_g2s(smem + (size_t)st * w_stage + (size_t)jj * tb,
                           w + ((size_t)(j + jj) * G + g0) * JSB, tb, &full[st], pol);
                  if (n == 0 && jj == 0) tc_trace(7, 9);
                }
              }
            }
            // the ring is full: only now wait for the predecessor (and let the
            // successor launch; every thread of the CTA triggers after its wait)
            if (n == NS - 1) {
              pdl_wait();
              pdl_trigger();
              triggered = true;
            }
            tc_trace(0, n);
            if (n == 0) tc_cta_mark(1);
          }
        }
        if (!triggered) {
          pdl_wait();
          pdl_trigger();
        }
        // the next GEMV's weights into L2: this CTA's slice of the next
        // matrix (same tile split as that launch), first nx.bytes of it
        if (a.nx.wbase && np == 1 && !kHead) {
          const TcNext& X = a.nx;
          const int li = s_li[0] + X.dli;
          if (li < X.wn) {
            const unsigned char* xw = reinterpret_cast<const unsigned char*>(X.wbase) + (size_t)li * X.wstride;
            const int xG = X.R >> 3, xncl = (int)gridDim.x / X.cs;
            if ((int)blockIdx.x < xncl * X.cs) {
              const int xb = (int)blockIdx.x / X.cs, xr = (int)blockIdx.x % X.cs;
              const int xu0 = (int)((unsigned)(xG * xb) / (unsigned)xncl), xu1 = (int)((unsigned)(xG * (xb + 1)) / (unsigned)xncl);
              const int xjlo = X.nj * xr / X.cs, xjhi = X.nj * (xr + 1) / X.cs;
              const uint32_t xJSB = (uint32_t)X.js << 10;
              TcTiles xt;
              xt.init(xu0, xu1, xG, X.tg);
              int xp, xg0, xtg, left = X.bytes;
              while (left > 0 && xt.next(xp, xg0, xtg)) {
                const uint32_t xtb = (uint32_t)xtg * xJSB;
                for (int j = xjlo; j < xjhi && left > 0; ++j, left -= (int)xtb)
                  prefetch_l2(xw + ((size_t)j * xG + xg0) * xJSB, xtb);
              }
            }
          }
        }
      } else {
        pdl_wait();
        pdl_trigger();
      }
    } else if (warp == 1) {  // ---------------- MMA issuer (whole warp, one elected lane) ----------------
      pdl_wait();
      pdl_trigger();
      TcTiles tl;
      tl.init(u0, u1, G, TG);
      int tp, g0, tg, n = 0, ti = 0;
      while (tl.next(tp, g0, tg)) {
        const int buf = ti & 1;
        const int nblk = (3 * s_nv[tp] + 15) >> 4;  // N = 16 * nblk columns: rows 3v + part
        const uint32_t idesc = kTcIdescBase | ((uint32_t)(2 * nblk) << 17);
        if (ti >= 2) mbar_wait(&acc_empty[buf], ((ti >> 1) - 1) & 1);
        tc_fence_after_sync();
        const uint32_t d = taddr + (uint32_t)(buf * kTcAccCols);
        const uint32_t tb = (uint32_t)tg * JSB;
        for (int j = jlo; j < jhi; j += NB, ++n) {
          const int nbj = min(NB, jhi - j);
          const int st = n % NS;
          mbar_wait(&full[st], (n / NS) & 1);
          tc_fence_after_sync();
          if (lane == 0) tc_trace(1, n);
          const uint64_t a0 = tc_desc(ring_w + (uint32_t)st * w_stage, JSB);
          const uint64_t b0 = tc_desc(ring_b + (uint32_t)st * b_stage, 1024);
          // JS slabs x 4 K steps per J-block, fully unrolled: constant
          // descriptor offsets keep the issue loop in uniform registers
          auto jblock = [&](auto js_c, int jj) {
            constexpr int kJS = decltype(js_c)::value;
            const uint64_t aj = a0 + ((jj * tb) >> 4);
            const uint64_t bj = b0 + (((uint32_t)(jj * kJS * NBLK)) << 7);  // (jj*JS*NBLK*2KB) >> 4
            const uint32_t acc0 = (j != jlo || jj != 0);
            if (elect_one()) {  // one lane issues the J-block's JS x 4 MMAs
#pragma unroll
              for (int sl = 0; sl < kJS; ++sl)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  tc_mma(d, aj + (sl << 6) + 2 * kk, bj + ((uint32_t)(sl * NBLK) << 7) + 2 * kk, idesc,
                         (sl | kk) ? 1u : acc0);
            }
            __syncwarp();
          };
          for (int jj = 0; jj < nbj; ++jj) {
            if (JS == 4) jblock(std::integral_constant<int, 4>{}, jj);
            else if (JS == 2) jblock(std::integral_constant<int, 2>{}, jj);
            else jblock(std::integral_constant<int, 1>{}, jj);
          }
          __syncwarp();
          if (lane == 0) tc_trace(2, n);
          if (elect_one()) tc_commit(&empty[st]);  // ring stage free once these MMAs retire
          __syncwarp();
        }
        if (elect_one()) tc_commit(&acc_full[buf]);
        __syncwarp();
        if (lane == 0) tc_cta_mark(2);
        ++ti;
      }
    } else if (warp < 6) {  // ---------------- operand builders ----------------
      // builder warp bw builds the B operand of ring stages n = bw (mod nbw):
      // the vectors' K slice (x, times the RMSNorm weight for QKV / gate-up /
      // heads; the 1/rms scale is applied in the epilogue) split exactly into
      // hi / mid / lo bf16 at rows 3v, 3v+1, 3v+2 of the swizzled operand
      const int bw = warp - 2, bt = tid - 64;
      const int nbw = NS < 4 ? NS : 4;
      pdl_wait();
      pdl_trigger();
      TcTiles tl;
      tl.init(u0, u1, G, TG);
      int tp, g0, tg, n = 0, cur_p = -1;
      __shared__ const float* s_srcv[4][kMaxVec];
      __shared__ const float* s_nwv[4][kMaxVec];
      const float** srcv = s_srcv[bw];
      const float** nwv = s_nwv[bw];
      int nvp = 0;
      while (tl.next(tp, g0, tg)) {
        if (tp != cur_p) {  // this problem's vectors
          cur_p = tp;
          nvp = s_nv[tp];
          const int g = s_pg[tp];
          __syncwarp();
          if (lane < kMaxVec) {
            const int v = lane;
            const float* sp = nullptr;
            const float* np_ = nullptr;
            if (v < nvp) {
              if (kHead2) {
                const int sl = work->head_slot[v];
                if (sl >= 0) sp = a.x + (size_t)sl * a.dm.d;
                np_ = v == 0 ? a.head_norm0 : a.head_norm1;
              } else if (kHeadV) {
                const int ex = s_ex;
                sp = a.x + (size_t)(ex && v == 0 ? work->head_exit : work->slot[0] + v - ex) * a.dm.d;
                np_ = ex && v == 0 ? a.head_norm0 : a.head_norm1;
              } else {
                const int sl = work->slot[g] + v;
                const LayerW& L = a.layers[work->first[g] + a.layer_i];
                if (EPI == kMatQKV) { sp = a.x + (size_t)sl * a.dm.d; np_ = L.attn_norm; }
                if (EPI == kMatGU) { sp = a.x + (size_t)sl * a.dm.d; np_ = L.mlp_norm; }
                if (EPI == kMatO) sp = a.o + (size_t)sl * a.dm.H * a.dm.hd;
                if (EPI == kMatDown) sp = a.h + (size_t)sl * a.dm.ffn;
              }
            }
            srcv[v] = sp;
            nwv[v] = np_;
          }
          __syncwarp();
        }
        // > 8 vectors (prefill chunks, EESD verify): the four warps build
        // every stage together (one round of loads per stage); else stage n
        // belongs to builder warp n % nbw (stages in flight hide the load
        // latency); nbw <= NS keeps every warp within one ring lap (an
        // mbarrier parity wait cannot tell phases two laps apart)
        const bool coop = nvp > 8;
        const int tstride = coop ? 128 : 32, tlane = coop ? bt : lane;
        for (int j = jlo; j < jhi; j += NB, ++n) {
          if (!coop && n % nbw != bw) continue;
          const int nbj = min(NB, jhi - j);
          const int st = n % NS;
          if (n >= NS) mbar_wait(&empty[st], ((n / NS) & 1) ^ 1);
          const uint32_t ba = ring_b + (uint32_t)st * b_stage;
          const int per_v = nbj * JS * 8;  // 16-byte K chunks of one vector in this stage
          const int items = nvp * per_v;
          for (int i0 = 0; i0 < ((tc_exp() & 2) ? 0 : items); i0 += 4 * tstride) {
            float xv[4][8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // all loads of up to 4 items first
              const int it = i0 + u * tstride + tlane;
              const int v = it / per_v, rem = it - v * per_v;
              const int k0 = (j * JS * 64) + rem * 8;  // rem = (jj * JS + s) * 8 + c
              const float* sp = it < items ? srcv[v] : nullptr;
              if (sp && k0 < K) {
                const float4 lo = __ldcg(reinterpret_cast<const float4*>(sp + k0));
                const float4 hi = __ldcg(reinterpret_cast<const float4*>(sp + k0 + 4));
                xv[u][0] = lo.x; xv[u][1] = lo.y; xv[u][2] = lo.z; xv[u][3] = lo.w;
                xv[u][4] = hi.x; xv[u][5] = hi.y; xv[u][6] = hi.z; xv[u][7] = hi.w;
                if (kNorm) {
                  const float4 w0 = __ldg(reinterpret_cast<const float4*>(nwv[v] + k0));
                  const float4 w1 = __ldg(reinterpret_cast<const float4*>(nwv[v] + k0 + 4));
                  xv[u][0] *= w0.x; xv[u][1] *= w0.y; xv[u][2] *= w0.z; xv[u][3] *= w0.w;
                  xv[u][4] *= w1.x; xv[u][5] *= w1.y; xv[u][6] *= w1.z; xv[u][7] *= w1.w;
                }
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) xv[u][e] = 0.f;
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int it = i0 + u * tstride + tlane;
              if (it >= items) break;
              const int v = it / per_v, rem = it - v * per_v;
              const int js_ = rem >> 3, c = rem & 7;  // (jj * JS + s), chunk
              float hi[8], mid[8], lo[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {  // exact three-way bf16 split
                hi[e] = __bfloat162float(__float2bfloat16_rn(xv[u][e]));
                const float r = xv[u][e] - hi[e];
                mid[e] = __bfloat162float(__float2bfloat16_rn(r));
                lo[e] = r - mid[e];
              }
              const uint32_t base = ba + ((uint32_t)(js_ * NBLK) << 11);
              const float* parts[3] = {hi, mid, lo};
#pragma unroll
              for (int pt = 0; pt < 3; ++pt) {
                const int row = 3 * v + pt;
                const float* q = parts[pt];
                const uint4 val = make_uint4(pack_bf16(q[0], q[1]), pack_bf16(q[2], q[3]), pack_bf16(q[4], q[5]),
                                             pack_bf16(q[6], q[7]));
                sts128(base + (uint32_t)((row >> 3) << 10) + (uint32_t)((row & 7) << 7) +
                           (uint32_t)(((c ^ (row & 7))) << 4),
                       val);
              }
            }
          }
          fence_proxy_async_smem();
          if (coop) {
            named_bar_sync(2, 128);
            if (bt == 0) mbar_arrive(&full[st]);
          } else {
            __syncwarp();
            if (lane == 0) {
              tc_trace(3, n);
              mbar_arrive(&full[st]);
            }
          }
        }
      }
    } else {  // ---------------- epilogue (warps 6-9) ----------------
      if (CS > 1) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      pdl_wait();
      pdl_trigger();
      const int quad = warp & 3;  // TMEM lanes 32*quad .. +31
      float bestv[2] = {-FLT_MAX, -FLT_MAX};
      int besti[2] = {INT_MAX, INT_MAX};
      float hbv[kMaxVec];
      int hbi[kMaxVec];
      if (kHeadV) {
#pragma unroll
        for (int v = 0; v < kMaxVec; ++v) { hbv[v] = -FLT_MAX; hbi[v] = INT_MAX; }
      }
      TcTiles tl;
      tl.init(u0, u1, G, TG);
      int tp, g0, tg, ti = 0, cur_p = -1;
      const int et = tid - 192;  // 0..127
      while (tl.next(tp, g0, tg)) {
        const int buf = ti & 1;
        const int nvp = s_nv[tp];
        const int nblk = (3 * nvp + 15) >> 4;
        if (kNorm && crank == 0 && tp != cur_p) {
          // 1/rms of this problem's vectors while the MMAs run: thread et sums
          // the 8-wide chunks et, et+128, ... (fixed order, independent of
          // the vector count and of the plan), then a warp tree, then warps
          // 0..3 in order
          cur_p = tp;
          const int nvec8 = K >> 3;
          for (int v = 0; v < nvp; ++v) {
            const float* sp = nullptr;
            if (kHead2) {
              const int sl = work->head_slot[v];
              if (sl >= 0) sp = a.x + (size_t)sl * a.dm.d;
            } else if (kHeadV) {
              const int ex = s_ex;
              sp = a.x + (size_t)(ex && v == 0 ? work->head_exit : work->slot[0] + v - ex) * a.dm.d;
            } else {
              sp = a.x + (size_t)(work->slot[s_pg[tp]] + v) * a.dm.d;
            }
            float ss = 0.f;
            if (sp)
              for (int c = et; c < nvec8; c += 128) {
                const float4 lo = __ldcg(reinterpret_cast<const float4*>(sp + c * 8));
                const float4 hi = __ldcg(reinterpret_cast<const float4*>(sp + c * 8 + 4));
                ss = fmaf(lo.x, lo.x, ss); ss = fmaf(lo.y, lo.y, ss); ss = fmaf(lo.z, lo.z, ss); ss = fmaf(lo.w, lo.w, ss);
                ss = fmaf(hi.x, hi.x, ss); ss = fmaf(hi.y, hi.y, ss); ss = fmaf(hi.z, hi.z, ss); ss = fmaf(hi.w, hi.w, ss);
              }
            ss = warp_sum(ss);
            if (lane == 0) s_ss[warp - 6][v] = ss;
          }
          named_bar_sync(1, 128);
          if (et < nvp) {
            const float tot = ((s_ss[0][et] + s_ss[1][et]) + s_ss[2][et]) + s_ss[3][et];
            s_rstd[et] = 1.0f / sqrtf(tot / (float)K + a.dm.eps);
          }
          named_bar_sync(1, 128);
        }
        // residual projections: fetch the hidden-state rows this thread will
        // update while the MMAs run (the add is then a plain store)
        float xres[kMaxVec];
        const int rl0 = 32 * quad + lane;
        if constexpr (EPI == kMatO || EPI == kMatDown) {
          if (crank == 0 && rl0 < tg * 8) {
            const float* xr = a.x + (size_t)work->slot[s_pg[tp]] * a.dm.d + g0 * 8 + rl0;
#pragma unroll
            for (int v = 0; v < kMaxVec; ++v)
              if (v < nvp) xres[v] = __ldcg(xr + (size_t)v * a.dm.d);
          }
        }
        // QKV: each vector's RoPE factors and KV page for this thread's row,
        // fetched while the MMAs run (the epilogue is then compute + stores,
        // not a chain of dependent loads per vector)
        float rcs[kMaxVec], rsn[kMaxVec];
        int rpg[kMaxVec];
        if constexpr (EPI == kMatQKV) {
          const int hd = a.dm.hd, H = a.dm.H, KVh = a.dm.KV;
          const int rr0 = g0 * 8 + rl0, head = rr0 / hd, wi = rr0 - head * hd;
          const bool live = rl0 < tg * 8 && !(lane & 1);
          const int pos0 = work->pos[s_pg[tp]];
#pragma unroll
          for (int v = 0; v < kMaxVec; ++v) {
            rcs[v] = 0.f;
            rsn[v] = 0.f;
            rpg[v] = 0;
            if (v < nvp && live) {
              const int pos = pos0 + v;
              if (head < H + KVh) {
                rcs[v] = a.rope_cos[(size_t)pos * (hd >> 1) + (wi >> 1)];
                rsn[v] = a.rope_sin[(size_t)pos * (hd >> 1) + (wi >> 1)];
              }
              if (head >= H) rpg[v] = a.page_table[pos / kPage];
            }
          }
        }
        mbar_wait(&acc_full[buf], (ti >> 1) & 1);
        tc_fence_after_sync();
        if (et == 0) tc_trace(4, ti);
        float c[16 * kTcMaxBlk];
        const bool quad_live = 32 * quad < tg * 8;
        if (quad_live) {
          const uint32_t ta = taddr + ((uint32_t)(32 * quad) << 16) + (uint32_t)(buf * kTcAccCols);
#pragma unroll
          for (int blk = 0; blk < kTcMaxBlk; ++blk)
            if (blk < nblk) tc_ld16(ta + (uint32_t)(blk * 16), c + blk * 16);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        tc_fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        const int rl = 32 * quad + lane;           // row within the tile
        if constexpr (CS > 1) {
          if (crank != 0) {  // ship this rank's row sums to the leader's receive buffer
            if (ti >= 1) mbar_wait_cluster(recv_empty, (ti - 1) & 1);
            if (quad_live) {
              const uint32_t dst = map_rank(smem_u32(recv), 0) + (uint32_t)(((crank - 1) * kMaxVec * 128 + rl) * 4);
#pragma unroll
              for (int v = 0; v < kMaxVec; ++v) {
                if (v >= nvp) break;
                st_cluster_f32(dst + (uint32_t)(v * 128 * 4), (c[3 * v] + c[3 * v + 1]) + c[3 * v + 2]);
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(map_rank(smem_u32(recv_full), 0));
            ++ti;
            continue;
          }
          mbar_wait_cluster(recv_full, ti & 1);
        }
        float part[kMaxVec];  // the other ranks' row sums (CS > 1), read before releasing the buffer
#pragma unroll
        for (int v = 0; v < kMaxVec; ++v) {
          part[v] = 0.f;
          if (CS > 1 && v < nvp && quad_live) {
            float t = 0.f;
#pragma unroll
            for (int r = 1; r < CS; ++r) {
              const float pr = recv[((r - 1) * kMaxVec + v) * 128 + rl];
              t = r == 1 ? pr : t + pr;
            }
            part[v] = t;
          }
        }
        if constexpr (CS > 1) {  // buffer free: every other rank may ship its next tile
          __syncwarp();
          if (lane == 0 && !tl.last())
            for (int r = 1; r < CS; ++r) mbar_arrive_cluster(map_rank(smem_u32(recv_empty), (uint32_t)r));
        }
        ++ti;
        if (!quad_live) continue;
        const bool valid = rl < tg * 8;
        const int rr = g0 * 8 + rl;                 // row within the matrix
        // fixed order: y_0 + ((y_1 + y_2) + y_3), then the 1/rms scale
        auto yv = [&](int v) {
          float y = (c[3 * v] + c[3 * v + 1]) + c[3 * v + 2];
          if (CS > 1) y = y + part[v];
          return kNorm ? y * s_rstd[v] : y;
        };
        if constexpr (EPI == kMatQKV || EPI == kMatGU) {
          const int g = s_pg[tp];
          const int slot0 = work->slot[g], pos0 = work->pos[g];
          void* kv_cache = nullptr;  // this row's K or V cache (QKV rows past the q heads)
          if (EPI == kMatQKV && valid && !(lane & 1) && rr / a.dm.hd >= a.dm.H) {
            const LayerW& L = a.layers[work->first[g] + a.layer_i];
            kv_cache = rr / a.dm.hd < a.dm.H + a.dm.KV ? L.kc : L.vc;
          }
#pragma unroll
          for (int v = 0; v < kMaxVec; ++v) {
            if (v >= nvp) break;
            const float y = yv(v);
            const float yp = __shfl_xor_sync(0xffffffffu, y, 1);
            if (!valid || (lane & 1)) continue;
            const int slot = slot0 + v, pos = pos0 + v;
            if (EPI == kMatGU) {
              a.h[(size_t)slot * a.dm.ffn + (rr >> 1)] = y / (1.0f + expf(-y)) * yp;
            } else {
              const int H = a.dm.H, KVh = a.dm.KV, hd = a.dm.hd;
              const int head = rr / hd, wi = rr - head * hd;
              float o0 = y, o1 = yp;
              void* cache = nullptr;
              int kvh = 0;
              if (head < H + KVh) {
                const float cs = rcs[v];
                const float sn = rsn[v];
                o0 = y * cs - yp * sn;
                o1 = yp * cs + y * sn;
                if (head < H) {
                  float* q = a.q + (size_t)slot * H * hd + head * hd + wi;
                  q[0] = o0;
                  q[1] = o1;
                } else {
                  cache = kv_cache;
                  kvh = head - H;
                }
              } else {
                cache = kv_cache;
                kvh = head - H - KVh;
              }
              if (cache) {
                const int page = rpg[v];
                const size_t off = (((size_t)page * KVh + kvh) * kPage + (pos % kPage)) * hd + wi;
                if (a.dm.kv_bf16) {
                  *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(cache) + off) =
                      __floats2bfloat162_rn(o0, o1);
                } else {
                  float* cp = reinterpret_cast<float*>(cache) + off;
                  cp[0] = o0;
                  cp[1] = o1;
                }
              }
            }
          }
        } else if constexpr (EPI == kMatO || EPI == kMatDown) {
          if (valid) {
            const int g = s_pg[tp];
#pragma unroll
            for (int v = 0; v < kMaxVec; ++v) {
              if (v >= nvp) break;
              a.x[(size_t)(work->slot[g] + v) * a.dm.d + rr] = xres[v] + yv(v);
            }
          }
        } else if constexpr (kHead2) {
          if (valid) {
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              if (work->head_slot[v] < 0) continue;
              const float y = yv(v);
              a.logits[(size_t)v * a.dm.V + rr] = y;
              if (y > bestv[v]) { bestv[v] = y; besti[v] = rr; }  // rows ascend per thread
            }
          }
        } else {  // kHeadV (comb_exit: logits row 0 = the exit vector, rows 1.. the batch)
          if (valid) {
            const int lrow0 = a.comb_exit ? 1 - s_ex : 0;
#pragma unroll
            for (int v = 0; v < kMaxVec; ++v) {
              if (v >= nvp) break;
              const float y = yv(v);
              a.logits[(size_t)(v + lrow0) * a.dm.V + rr] = y;
              if (y > hbv[v]) { hbv[v] = y; hbi[v] = rr; }
            }
          }
        }
      }
      if (kHead && crank == 0) {  // deterministic first-index argmax across the clusters' leaders
        const int nvh = kHead2 ? 2 : s_nv[0];
#pragma unroll
        for (int v = 0; v < kMaxVec; ++v) {
          if (v >= nvh) break;
          float bv = kHead2 ? (v == 0 ? bestv[0] : bestv[1]) : hbv[v];
          int bi = kHead2 ? (v == 0 ? besti[0] : besti[1]) : hbi[v];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (tc_better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
          }
          if (lane == 0) { s_bv[quad][v] = bv; s_bi[quad][v] = bi; }
        }
        named_bar_sync(1, 128);
        int* ticket = a.head_cnt;
        if (et == 0) {
          for (int v = 0; v < nvh; ++v) {
            float bv = s_bv[0][v];
            int bi = s_bi[0][v];
            for (int w = 1; w < 4; ++w)
              if (tc_better(s_bv[w][v], s_bi[w][v], bv, bi)) { bv = s_bv[w][v]; bi = s_bi[w][v]; }
            // partial slot: the cluster's rank among the clusters with work
            // (u0 when every working cluster holds one group, else b)
            const int slot = U <= ncl ? u0 : b;
            a.head_part[((size_t)slot * kMaxVec + v) * 2 + 0] = bv;
            a.head_part[((size_t)slot * kMaxVec + v) * 2 + 1] = __int_as_float(bi);
          }
          __threadfence();
          s_last = atomicAdd(ticket, 1) == ncta - 1;
        }
        named_bar_sync(1, 128);
        if (s_last) {  // the last CTA merges the per-CTA partials
          __threadfence();
          for (int v = 0; v < nvh; ++v) {
            float bv = -FLT_MAX;
            int bi = INT_MAX;
            for (int cb = et; cb < ncta; cb += 128) {
              const float pv = __ldcg(&a.head_part[((size_t)cb * kMaxVec + v) * 2 + 0]);
              const int pi = __float_as_int(__ldcg(&a.head_part[((size_t)cb * kMaxVec + v) * 2 + 1]));
              if (tc_better(pv, pi, bv, bi)) { bv = pv; bi = pi; }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
              const float ov = __shfl_xor_sync(0xffffffffu, bv, off);
              const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
              if (tc_better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
            }
            if (lane == 0) { s_bv[quad][v] = bv; s_bi[quad][v] = bi; }
          }
          named_bar_sync(1, 128);
          if (et == 0) {
            Work* wk = const_cast<Work*>(work);
            for (int v = 0; v < nvh; ++v) {
              float bv = s_bv[0][v];
              int bi = s_bi[0][v];
              for (int w = 1; w < 4; ++w)
                if (tc_better(s_bv[w][v], s_bi[w][v], bv, bi)) { bv = s_bv[w][v]; bi = s_bi[w][v]; }
              if (kHead2) wk->head_out[v] = work->head_slot[v] >= 0 ? bi : -1;
              else if (s_ex && v == 0) wk->head_out[0] = bi;
              else wk->vec_out[v - s_ex] = bi;
            }
            *ticket = 0;
          }
        }
      }
    }
  } else {
    pdl_wait();
    pdl_trigger();
  }
  // no cluster barrier at exit: remote traffic only targets the leader's
  // receive buffer (which the leader waits for) and the other ranks'
  // recv_empty barriers (each waited before that rank ships its next tile;
  // none after the last)
  tc_fence_before_sync();
  __syncthreads();
  if (tid == 0) tc_cta_mark(3);
  if (warp == 1) {
    tc_fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kTcTmemCols));
  }
}

// ---------------------------------------------------------------------------
// host side

int tc_max_clusters(int cs);

namespace {
constexpr size_t kTcSmemCap = 221 * 1024;  // + static smem <= 227 KB
// dynamic smem budget of a plan (PPSD_TC_SMEM=<KB> experiments: <= ~110 KB lets
// two GEMV CTAs share an SM, so a PDL-launched successor starts streaming
// while its predecessor drains)
static size_t tc_smem_budget() {
  static size_t b = 0;
  if (!b) {
    b = kTcSmemCap;
    if (const char* v = getenv("PPSD_TC_SMEM")) b = std::min(kTcSmemCap, (size_t)std::max(atoi(v), 48) * 1024);
  }
  return b;
}
constexpr size_t kTcStageTarget = 48 * 1024;  // weight bytes per ring stage to aim for
}  // namespace

// Plan a [R][K] matrix for `num_sms` SMs with up to nblk 16-column B blocks.
// Split-K cluster size CS in {1, 2, 4}: the smallest whose per-CTA MMA work
// (1 MMA per 16-wide K step and 128-row tile, ~60 cycles each measured in
// situ) stays well under the CTA's HBM time; the rest streams like CS = 1.
int tc_pick(int K, int R, int nblk, int num_sms, TcPlan* p, int p_mat_hint) {
  if (K <= 0 || R <= 0 || R % 8 != 0 || K % 8 != 0 || nblk < 1 || nblk > kTcMaxBlk) return -1;
  int JS, KP;
  tc_layout(R, K, &JS, &KP);
  const int G = R / 8, NJ = KP / 64 / JS;
  // Split-K cluster size: measured on the 7B shapes (tools/probe_gemv.py,
  // tools/quick_decode.py with PPSD_TC_CS), a CTA with fewer than 8 row
  // groups (64 rows) is bound by its MMA issue rate (one M=128 MMA per 16-wide
  // K step whatever the rows) and by the fixed per-launch cost; 4-CTA
  // clusters give each CTA 4x the rows over a quarter of K (O 12.3 -> 10.7 us,
  // down 21.5 -> 18.6 us); the wide matrices stay unsplit (gate/up with CS 2
  // or 4: 30.1 -> 31.3 / 37.0 us).
  int best_cs = 1;
  if ((G + num_sms - 1) / num_sms < 8 && NJ >= 4 && tc_max_clusters(4) >= 8) best_cs = 4;
  int CS = best_cs;
  if (const char* v = getenv("PPSD_TC_CS")) {  // experiments: force the split-K cluster size
    // "<cs>" for the matrices that split at all, "<qkv>,<o>,<gu>,<down>" per matrix (row counts R
    // identify them: the 7B probe shapes)
    int f[4] = {0, 0, 0, 0};
    const int nf = sscanf(v, "%d,%d,%d,%d", &f[0], &f[1], &f[2], &f[3]);
    if (nf == 1) {
      if ((f[0] == 1 || f[0] == 2 || f[0] == 4) && f[0] <= NJ && CS > 1) CS = f[0];
    } else if (nf == 4) {
      const int idx = p_mat_hint;
      if (idx >= 0 && idx < 4 && (f[idx] == 1 || f[idx] == 2 || f[idx] == 4) && f[idx] <= NJ) CS = f[idx];
    }
  }
  int ncl = num_sms / CS;
  if (CS > 1) {
    const int maxc = tc_max_clusters(CS);
    if (maxc > 0 && maxc < ncl) ncl = maxc;
    // whole M=128 tiles: when the row groups split into >= 80 % as many
    // 16-group tiles as there are clusters, one full tile per cluster beats
    // uneven partial tiles (7B O / down: 32 clusters of 16 groups instead of
    // 37 of 13-14; decode 458.9 -> 461.5 tok/s, AR 374.8 -> 377.2)
    if (G % 16 == 0 && G / 16 <= ncl && 5 * (G / 16) >= 4 * ncl) ncl = G / 16;
  }
  const int c = (G + ncl - 1) / ncl;
  const int TG = (c + (c + 15) / 16 - 1) / ((c + 15) / 16);
  const size_t wj = (size_t)TG * JS * 1024, bj = (size_t)nblk * JS * 2048;
  int nb = (int)(kTcStageTarget / (wj + bj));
  if (nb < 1) nb = 1;
  const int njr = (NJ + CS - 1) / CS;  // J-blocks of one rank
  if (nb > njr) nb = njr;
  const size_t ws = nb * wj, bs = nb * bj;
  // the A descriptor of a tile with tg < 16 groups reads (16 - tg) groups
  // past the tile (rows of the MMA that are ignored): keep them inside smem
  const size_t over = (size_t)(16 - TG) * JS * 1024;
  const size_t recv = CS > 1 ? (size_t)(CS - 1) * kMaxVec * 128 * 4 : 0;
  const size_t fixed = 1024 + 256 + recv;  // alignment slack + barriers + receive buffer
  int ns = 0;
  for (const size_t budget : {tc_smem_budget(), kTcSmemCap}) {  // the cap when the budget cannot hold 2 stages
    for (int cand = 8; cand >= 2; --cand) {
      const size_t ring = cand * (ws + bs);
      const size_t pad = over > (size_t)cand * bs ? over - (size_t)cand * bs : 0;
      if (ring + pad + fixed <= budget) { ns = cand; break; }
    }
    if (ns) break;
  }
  if (ns < 2) return -1;
  const size_t ring = ns * (ws + bs);
  const size_t pad = over > (size_t)ns * bs ? over - (size_t)ns * bs : 0;
  p->R = R;
  p->K = K;
  p->js = JS;
  p->nj = NJ;
  p->nb = nb;
  p->tg = TG;
  p->nblk = nblk;
  p->ns = ns;
  p->cs = CS;
  p->grid = ncl * CS;
  p->bar_off = (int)(ring + pad);
  p->smem = ring + pad + fixed;
  return 0;
}

namespace {
template <int EPI, int CS>
cudaError_t tc_one(const GemvArgs& a, size_t smem, int grid, cudaStream_t st, bool attrs_only) {
  auto fn = tcgemv_kernel<EPI, CS>;
  if (attrs_only) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && CS > 1) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTcThreads);
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
  cfg.numAttrs = CS > 1 ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, fn, a);
}
template <int CS>
cudaError_t tc_dispatch_cs(const GemvArgs& a, int mat, size_t smem, int grid, cudaStream_t st, bool attrs_only) {
  switch (mat) {
    case kMatQKV: return tc_one<kMatQKV, CS>(a, smem, grid, st, attrs_only);
    case kMatO: return tc_one<kMatO, CS>(a, smem, grid, st, attrs_only);
    case kMatGU: return tc_one<kMatGU, CS>(a, smem, grid, st, attrs_only);
    case kMatDown: return tc_one<kMatDown, CS>(a, smem, grid, st, attrs_only);
    case kMatHead: return tc_one<kMatHead, CS>(a, smem, grid, st, attrs_only);
    case kMatHeadV: return tc_one<kMatHeadV, CS>(a, smem, grid, st, attrs_only);
  }
  return cudaErrorInvalidValue;
}
cudaError_t tc_dispatch(const GemvArgs& a, int mat, int cs, size_t smem, int grid, cudaStream_t st,
                        bool attrs_only) {
  switch (cs) {
    case 1: return tc_dispatch_cs<1>(a, mat, smem, grid, st, attrs_only);
    case 2: return tc_dispatch_cs<2>(a, mat, smem, grid, st, attrs_only);
    case 4: return tc_dispatch_cs<4>(a, mat, smem, grid, st, attrs_only);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

// clusters of `cs` CTAs (this kernel's smem) that can be co-resident on the device
int tc_max_clusters(int cs) {
  static int cache[5] = {-1, -1, -1, -1, -1};
  if (cs < 1 || cs > 4) return 0;
  if (cache[cs] >= 0) return cache[cs];
  GemvArgs dummy{};
  if (tc_dispatch(dummy, kMatO, cs, kTcSmemCap, 0, 0, true) != cudaSuccess) return cache[cs] = 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * 256);
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = kTcSmemCap;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  const cudaError_t e = cs == 1 ? cudaSuccess
                        : cs == 2 ? cudaOccupancyMaxActiveClusters(&n, tcgemv_kernel<kMatO, 2>, &cfg)
                                  : cudaOccupancyMaxActiveClusters(&n, tcgemv_kernel<kMatO, 4>, &cfg);
  if (e != cudaSuccess) { cudaGetLastError(); n = 0; }
  return cache[cs] = n;
}

// every plan of a matrix shares one kernel instantiation per CS: allow the largest
cudaError_t tc_set_attrs(int mat, int cs, size_t /*smem*/) {
  GemvArgs dummy{};
  return tc_dispatch(dummy, mat, cs, kTcSmemCap, 0, 0, true);
}

int tc_trace_enable(int on) {
  int exp = getenv("PPSD_TC_EXP") ? atoi(getenv("PPSD_TC_EXP")) : 0;
  cudaMemcpyToSymbol(g_tc_exp, &exp, sizeof(int));
  return cudaMemcpyToSymbol(g_tc_trace_on, &on, sizeof(int)) == cudaSuccess ? 0 : -1;
}
int tc_trace_read(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, g_tc_trace, sizeof(g_tc_trace)) != cudaSuccess) return -1;
  return cudaMemcpyFromSymbol(out + 8 * kTcTraceN, g_tc_cta, sizeof(g_tc_cta)) == cudaSuccess ? 0 : -1;
}

cudaError_t tc_launch(const GemvArgs& a, int cs, size_t smem, int grid, cudaStream_t st) {
  return tc_dispatch(a, a.mat, cs, smem, grid, st, false);
}

}  // namespace ppsd
