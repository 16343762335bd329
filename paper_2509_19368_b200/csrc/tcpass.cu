// tcpass.cu — the decoder layers of one tick (or AR step, prefill chunk,
// EESD verify) as ONE persistent launch: for every layer slot the QKV GEMV,
// attention, O GEMV, gate/up GEMV and down GEMV run as phases of the same
// grid, separated by grid-wide barriers, instead of five kernels.
//
// Why: on the 7B shape a tensor-core GEMV launch spends ~2.5 us before its
// first weight byte arrives (work descriptor, barriers, TMEM) and ~1-3 us in
// its tail (epilogue, the slowest CTA), with HBM idle in between. Here the
// weight producer never waits for activations: it streams the next phase's
// (and the next layer's) weights through the ring while the grid finishes
// the current phase, runs attention or sits in a barrier, so HBM stays busy
// across phase boundaries and the per-launch costs are paid once per pass.
//
// Roles (320 threads, one CTA per SM, clusters of CS CTAs):
//   warp 0, one lane     weight producer: the CTA's tiles of every phase, in
//                        phase order, through one NS-slot ring (bulk copies)
//   warp 1               TMEM + MMA issuer (tcgen05.mma kind::f16 M=128)
//   warps 2-5            operand builders; attention worker 0 in the
//                        attention phase
//   warps 6-9            epilogues (+ cluster split-K exchange, 1/rms);
//                        attention worker 1 when shared memory allows
// The GEMV arithmetic (tile K order, per-matrix cluster split, three-way bf16
// split, fold order) is exactly the standalone kernel's (tcgemv.cu), and the
// attention is the split-K worker of attn_core.cuh (results independent of
// the worker count), so a pass is bit-identical to the per-kernel sequence.
//
// Grid barriers: one monotone 64-bit arrival counter per engine. Barrier k of
// a launch completes when counter >= base + (k+1) * grid, base = the value
// the previous launch left in `bar_seq`; a CTA arrives at k only after it saw
// k-1 complete, so the count cannot run ahead. Each barrier is arrived at
// once per CTA: phase outputs written -> __threadfence -> red.add.
#include "attn_core.cuh"
#include "tc_dev.cuh"

namespace ppsd {

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void gbar_arrive(unsigned long long* cnt) {
  __threadfence();
  asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(cnt) : "memory");
}
// one thread spins; the caller releases its thread group with a named barrier
__device__ __forceinline__ void gbar_wait(const unsigned long long* cnt, unsigned long long target,
                                          int32_t* err) {
  const uint64_t t0 = globaltimer();
  while (ld_acquire_u64(cnt) < target) {
    __nanosleep(20);
    if (globaltimer() - t0 > 5000000000ull) {  // 5 s: sticky error, never a hang
      atomicOr(err, kGemvErrPassTimeout);
      break;
    }
  }
}

// The problem list of layer slot i: groups with a chain that have a layer i.
struct PassProblems {
  int np;
  int pg[kTcMaxProb], li[kTcMaxProb], nv[kTcMaxProb];
};
__device__ __forceinline__ void pass_problems(const Work& w, int i, PassProblems& P) {
  int np = 0;
  for (int g = 0; g < w.G && np < kTcMaxProb; ++g)
    if (w.slot[g] >= 0 && i < w.nl[g] && w.nv[g] > 0) {
      P.pg[np] = g;
      P.li[np] = w.first[g] + i;
      P.nv[np++] = w.nv[g];
    }
  P.np = np;
}

// This CTA's share of matrix m: group range [u0, u1) and J-block range.
struct PassShare {
  int u0, u1, jlo, jhi, crank, b, ncl;
};
__device__ __forceinline__ void pass_share(const TcPassMat& M, int np, PassShare& s) {
  const int G = M.R >> 3, U = np * G;
  s.crank = M.cs > 1 ? (int)(blockIdx.x % M.cs) : 0;
  s.ncl = (int)gridDim.x / M.cs;
  s.b = (int)blockIdx.x / M.cs;
  s.u0 = (int)((long long)U * s.b / s.ncl);
  s.u1 = (int)((long long)U * (s.b + 1) / s.ncl);
  s.jlo = M.nj * s.crank / M.cs;
  s.jhi = M.nj * (s.crank + 1) / M.cs;
}


// The producer's walk over the weight stages of a pass: (layer slot i,
// matrix m, tile, J-blocks [j, j + nbj)) in the order every role uses.
struct PassCursor {
  int i, m, j, nbj, tg, g0, G, nb, jhi;
  uint32_t tb, JSB;
  const unsigned char* wb;
  bool ok;
  PassShare sh;
  TcTiles tl;
  int np;
  int li[kTcMaxProb];
  __device__ const unsigned char* src(int jj) const { return wb + ((size_t)(j + jj) * G + g0) * JSB; }
  // tiles of (i, m) from the start; false when (i, m) has no tile for this CTA
  __device__ bool open_mat(const TcPassArgs& a) {
    const TcPassMat& M = a.mat[m];
    pass_share(M, np, sh);
    G = M.R >> 3;
    nb = M.nb;
    JSB = (uint32_t)M.js << 10;
    tl.init(sh.u0, sh.u1, G, M.tg);
    return open_tile(a);
  }
  __device__ bool open_tile(const TcPassArgs& a) {
    int tp;
    if (!tl.next(tp, g0, tg)) return false;
    const TcPassMat& M = a.mat[m];
    const int l = li[tp];
    if (M.wstride && l < M.wn) {
      wb = reinterpret_cast<const unsigned char*>(M.wbase) + (size_t)l * M.wstride;
    } else {
      const LayerW& L = a.g.layers[l];
      wb = reinterpret_cast<const unsigned char*>(m == 0 ? L.qkv : m == 1 ? L.o : m == 2 ? L.gu : L.down);
    }
    tb = (uint32_t)tg * JSB;
    j = sh.jlo;
    jhi = sh.jhi;
    nbj = min(nb, jhi - j);
    return j < jhi;
  }
  __device__ void open_slot(const Work& W) {
    PassProblems P;
    pass_problems(W, i, P);
    np = P.np;
    for (int p = 0; p < np; ++p) li[p] = P.li[p];
  }
  // first stage at or after (i, m)
  __device__ void settle(const TcPassArgs& a, const Work& W) {
    while (i < a.n_slots) {
      if (open_mat(a)) { ok = true; return; }
      if (++m == 4) {
        m = 0;
        if (++i < a.n_slots) open_slot(W);
      }
    }
    ok = false;
  }
  __device__ void begin(const TcPassArgs& a, const Work& W) {
    i = 0;
    m = 0;
    ok = false;
    if (a.n_slots > 0) {
      open_slot(W);
      settle(a, W);
    }
  }
  __device__ void advance(const TcPassArgs& a, const Work& W) {
    j += nb;
    if (j < jhi) {
      nbj = min(nb, jhi - j);
      return;
    }
    if (open_tile(a)) return;
    if (++m == 4) {
      m = 0;
      if (++i < a.n_slots) open_slot(W);
    }
    settle(a, W);
  }
};

template <int CS, int HD, typename KVT, int QPK>
__global__ void __launch_bounds__(kTcThreads, 1) tcpass_kernel(const TcPassArgs a) {
  extern __shared__ unsigned char tp_smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tp_smem_raw) + 1023) & ~(uintptr_t)1023);
  __shared__ Work s_work;
  __shared__ uint32_t s_taddr;
  __shared__ float s_ss[4][kMaxVec];
  __shared__ float s_rstd[kMaxVec];
  __shared__ const float* s_srcv[4][kMaxVec];
  __shared__ const float* s_nwv[4][kMaxVec];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NS = a.ns;
  const uint32_t slot_bytes = (uint32_t)a.slot_bytes, b_stage = (uint32_t)a.b_stage;
  const uint32_t ring_w = smem_u32(smem);
  const uint32_t ring_b = ring_w + (uint32_t)NS * slot_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + a.bar_off);
  uint64_t* empty = full + NS;
  uint64_t* acc_full = empty + NS;  // [2]
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* recv_full = acc_empty + 2;
  uint64_t* recv_empty = recv_full + 1;
  float* recv = reinterpret_cast<float*>(smem + a.bar_off + 256);
  using Scratch = AttnScratch<HD, QPK>;
  Scratch* scr = reinterpret_cast<Scratch*>(smem + a.scr_off);  // [n_workers]
  const int nwk = a.attn_workers;  // attention workers per CTA (1: warps 2-5, 2: + warps 6-9)
  const int ntot = a.n_slots * 5;  // grid barriers of this launch

  // ---- prologue: the work descriptor (written by the scheduler, the
  // immediately preceding kernel unless desc_early), barriers, TMEM ----
  if (tid == 0) tc_trace(6, 0);
  if (!a.desc_early) pdl_wait();
  for (int i = tid; i < (int)(sizeof(Work) / 4); i += kTcThreads)
    reinterpret_cast<int32_t*>(&s_work)[i] = reinterpret_cast<const int32_t*>(a.g.work)[i];
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 2);  // producer (expect_tx) + the builder warp of the stage
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
    }
    if (CS > 1) {
      mbar_init(recv_full, 4 * (CS - 1));
      mbar_init(recv_empty, 4);
    }
    for (int w = 0; w < nwk; ++w) mbar_init(&scr[w].bar, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_taddr)),
                 "n"(kTcTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before_sync();
  __syncthreads();
  if (CS > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  tc_fence_after_sync();
  const uint32_t taddr = s_taddr;
  const Work& W = s_work;

  if (warp == 0) {  // ================= weight producer =================
    if (lane == 0) {
      // Two cursors walk the same stage sequence: `cp` fills the smem ring;
      // `pf` runs up to kPassPrefetch bytes ahead with L2 prefetches, so HBM
      // keeps streaming while the ring is full (attention, grid barriers).
      const uint64_t pol = policy_evict_first();
      int n = 0;
      bool waited = a.desc_early == 0;
      PassCursor cp, pf;
      cp.begin(a, W);
      pf.begin(a, W);
      unsigned long long cp_bytes = 0, pf_bytes = 0;
      const unsigned long long ahead = a.prefetch_bytes;
      while (cp.ok) {
        while (pf.ok && pf_bytes < cp_bytes + ahead) {
          for (int jj = 0; jj < pf.nbj; ++jj) prefetch_l2(pf.src(jj), pf.tb);
          pf_bytes += (unsigned long long)pf.nbj * pf.tb;
          pf.advance(a, W);
        }
        const int st = n % NS;
        if (n >= NS) mbar_wait(&empty[st], ((n / NS) & 1) ^ 1);
        mbar_expect_tx(&full[st], (uint32_t)cp.nbj * cp.tb);
        for (int jj = 0; jj < cp.nbj; ++jj)
          bulk_g2s(smem + (size_t)st * slot_bytes + (size_t)jj * cp.tb, cp.src(jj), cp.tb, &full[st], pol);
        tc_trace(0, n);
        cp_bytes += (unsigned long long)cp.nbj * cp.tb;
        cp.advance(a, W);
        if (!waited && n == NS - 1) {  // ring full: now wait for the predecessor
          pdl_wait();
          waited = true;
        }
        ++n;
      }
      if (!waited) pdl_wait();
    } else {
      pdl_wait();
    }
  } else if (warp == 1) {  // ================= MMA issuer =================
    pdl_wait();
    int n = 0, ti = 0;
    PassProblems P;
    for (int i = 0; i < a.n_slots; ++i) {
      pass_problems(W, i, P);
      for (int m = 0; m < 4; ++m) {
        const TcPassMat& M = a.mat[m];
        PassShare sh;
        pass_share(M, P.np, sh);
        const uint32_t JSB = (uint32_t)M.js << 10;
        const int NBLK = a.nblk;
        TcTiles tl;
        tl.init(sh.u0, sh.u1, M.R >> 3, M.tg);
        int tp, g0, tg;
        while (tl.next(tp, g0, tg)) {
          const int buf = ti & 1;
          const int nblk = (3 * P.nv[tp] + 15) >> 4;
          const uint32_t idesc = kTcIdescBase | ((uint32_t)(2 * nblk) << 17);
          if (ti >= 2) mbar_wait(&acc_empty[buf], ((ti >> 1) - 1) & 1);
          tc_fence_after_sync();
          const uint32_t d = taddr + (uint32_t)(buf * kTcAccCols);
          const uint32_t tb = (uint32_t)tg * JSB;
          for (int j = sh.jlo; j < sh.jhi; j += M.nb, ++n) {
            const int nbj = min(M.nb, sh.jhi - j);
            const int st = n % NS;
            mbar_wait(&full[st], (n / NS) & 1);
            tc_fence_after_sync();
            if (lane == 0) tc_trace(1, n);
            const uint64_t a0 = tc_desc(ring_w + (uint32_t)st * slot_bytes, JSB);
            const uint64_t b0 = tc_desc(ring_b + (uint32_t)st * b_stage, 1024);
            auto jblock = [&](auto js_c, int jj) {
              constexpr int kJS = decltype(js_c)::value;
              const uint64_t aj = a0 + ((jj * tb) >> 4);
              const uint64_t bj = b0 + (((uint32_t)(jj * kJS * NBLK)) << 7);
              const uint32_t acc0 = (j != sh.jlo || jj != 0);
              if (elect_one()) {
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
              if (M.js == 4) jblock(std::integral_constant<int, 4>{}, jj);
              else if (M.js == 2) jblock(std::integral_constant<int, 2>{}, jj);
              else jblock(std::integral_constant<int, 1>{}, jj);
            }
            __syncwarp();
            if (elect_one()) tc_commit(&empty[st]);
            __syncwarp();
          }
          if (elect_one()) tc_commit(&acc_full[buf]);
          __syncwarp();
          ++ti;
        }
      }
    }
  } else if (warp < 6) {  // ================= operand builders (+ attention worker 0) =================
    const int bw = warp - 2, bt = tid - 64;
    const int nbw = NS < 4 ? NS : 4;
    pdl_wait();
    // barrier base of this launch: the previous pass completed before the
    // kernel this one waited for
    const unsigned long long base = *a.bar_seq;
    const unsigned long long grid = gridDim.x;
    auto wait_bar = [&](int k) {  // barrier k complete (k < 0: none)
      if (k >= 0) {
        if (bt == 0) {
          gbar_wait(a.bar_cnt, base + (unsigned long long)(k + 1) * grid, a.g.err);
          tc_trace(2, k);
        }
        named_bar_sync(2, 128);
      }
    };
    int n = 0;
    uint32_t aph = 0;  // attention worker 0's mbarrier parity, carried across layers
    PassProblems P;
    const float** srcv = s_srcv[bw];
    const float** nwv = s_nwv[bw];
    for (int i = 0; i < a.n_slots; ++i) {
      pass_problems(W, i, P);
      for (int m = 0; m < 4; ++m) {
        const TcPassMat& M = a.mat[m];
        if (m == 1) {  // attention between QKV and O
          wait_bar(5 * i + 0);
          AttnArgs at = a.at;
          at.layer_i = i;
          attn_items<HD, KVT, QPK>(at, (int)blockIdx.x * nwk, (int)gridDim.x * nwk, bt,
                                   reinterpret_cast<KVT*>(smem + a.attn_off), scr[0], aph,
                                   [] { named_bar_sync(2, 128); }, [] {});
          named_bar_sync(4, 256);  // both attention workers of the CTA are done
          if (bt == 0) {
            tc_trace(5, i);
            gbar_arrive(a.bar_cnt);  // barrier 5i+1: attention outputs
          }
          wait_bar(5 * i + 1);  // the inputs of O: every CTA's attention done
        } else {
          wait_bar(m == 0 ? 5 * i - 1 : 5 * i + m);  // QKV: the previous layer's down; GU: O; down: GU
        }
        PassShare sh;
        pass_share(M, P.np, sh);
        TcTiles tl;
        tl.init(sh.u0, sh.u1, M.R >> 3, M.tg);
        int tp, g0, tg, cur_p = -1, nvp = 0;
        const int K = M.K;
        const bool norm = m == 0 || m == 2;
        while (tl.next(tp, g0, tg)) {
          if (tp != cur_p) {
            cur_p = tp;
            nvp = P.nv[tp];
            const int g = P.pg[tp];
            __syncwarp();
            if (lane < kMaxVec) {
              const int v = lane;
              const float* sp = nullptr;
              const float* np_ = nullptr;
              if (v < nvp) {
                const int sl = W.slot[g] + v;
                const LayerW& L = a.g.layers[P.li[tp]];
                if (m == 0) { sp = a.g.x + (size_t)sl * a.g.dm.d; np_ = L.attn_norm; }
                if (m == 1) sp = a.g.o + (size_t)sl * a.g.dm.H * a.g.dm.hd;
                if (m == 2) { sp = a.g.x + (size_t)sl * a.g.dm.d; np_ = L.mlp_norm; }
                if (m == 3) sp = a.g.h + (size_t)sl * a.g.dm.ffn;
              }
              srcv[v] = sp;
              nwv[v] = np_;
            }
            __syncwarp();
          }
          const int NBLK = a.nblk, JS = M.js;
          for (int j = sh.jlo; j < sh.jhi; j += M.nb, ++n) {
            if (n % nbw != bw) continue;
            const int nbj = min(M.nb, sh.jhi - j);
            const int st = n % NS;
            if (n >= NS) mbar_wait(&empty[st], ((n / NS) & 1) ^ 1);
            const uint32_t ba = ring_b + (uint32_t)st * b_stage;
            const int per_v = nbj * JS * 8;
            const int items = nvp * per_v;
            for (int i0 = 0; i0 < items; i0 += 4 * 32) {
              float xv[4][8];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int it = i0 + u * 32 + lane;
                const int v = it / per_v, rem = it - v * per_v;
                const int k0 = (j * JS * 64) + rem * 8;
                const float* sp = it < items ? srcv[v] : nullptr;
                if (sp && k0 < K) {
                  const float4 lo = __ldcg(reinterpret_cast<const float4*>(sp + k0));
                  const float4 hi = __ldcg(reinterpret_cast<const float4*>(sp + k0 + 4));
                  xv[u][0] = lo.x; xv[u][1] = lo.y; xv[u][2] = lo.z; xv[u][3] = lo.w;
                  xv[u][4] = hi.x; xv[u][5] = hi.y; xv[u][6] = hi.z; xv[u][7] = hi.w;
                  if (norm) {
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
                const int it = i0 + u * 32 + lane;
                if (it >= items) break;
                const int v = it / per_v, rem = it - v * per_v;
                const int js_ = rem >> 3, c = rem & 7;
                float hi[8], mid[8], lo[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  hi[e] = __bfloat162float(__float2bfloat16_rn(xv[u][e]));
                  const float r = xv[u][e] - hi[e];
                  mid[e] = __bfloat162float(__float2bfloat16_rn(r));
                  lo[e] = r - mid[e];
                }
                const uint32_t bb = ba + ((uint32_t)(js_ * NBLK) << 11);
                const float* parts[3] = {hi, mid, lo};
#pragma unroll
                for (int pt = 0; pt < 3; ++pt) {
                  const int row = 3 * v + pt;
                  const float* q = parts[pt];
                  const uint4 val = make_uint4(pack_bf16(q[0], q[1]), pack_bf16(q[2], q[3]), pack_bf16(q[4], q[5]),
                                               pack_bf16(q[6], q[7]));
                  sts128(bb + (uint32_t)((row >> 3) << 10) + (uint32_t)((row & 7) << 7) +
                             (uint32_t)(((c ^ (row & 7))) << 4),
                         val);
                }
              }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[st]);
          }
        }
      }
    }
  } else {  // ================= epilogues (+ attention worker 1) =================
    if (CS > 1) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    pdl_wait();
    const int quad = warp & 3, et = tid - 192;
    const unsigned long long base = *a.bar_seq;  // the value the builders read
    const unsigned long long grid = gridDim.x;
    auto wait_bar = [&](int k) {
      if (k >= 0) {
        if (et == 0) {
          gbar_wait(a.bar_cnt, base + (unsigned long long)(k + 1) * grid, a.g.err);
          tc_trace(3, k);
        }
        named_bar_sync(1, 128);
      }
    };
    int narr = 0;
    auto arrive_bar = [&]() {  // this CTA's outputs of the phase are written
      named_bar_sync(1, 128);
      if (et == 0) {
        tc_trace(4, narr);
        gbar_arrive(a.bar_cnt);
      }
      ++narr;
    };
    int ti = 0, xt = 0;
    uint32_t aph = 0;  // attention worker 1's mbarrier parity
    PassProblems P;
    for (int i = 0; i < a.n_slots; ++i) {
      pass_problems(W, i, P);
      for (int m = 0; m < 4; ++m) {
        const TcPassMat& M = a.mat[m];
        if (m == 1) {  // attention: worker 1 (when two fit), then the barrier order
          wait_bar(5 * i + 0);
          if (nwk > 1) {
            AttnArgs at = a.at;
            at.layer_i = i;
            attn_items<HD, KVT, QPK>(at, (int)blockIdx.x * nwk + 1, (int)gridDim.x * nwk, et,
                                     reinterpret_cast<KVT*>(smem + a.attn_off + a.attn_kv_bytes), scr[1], aph,
                                     [] { named_bar_sync(1, 128); }, [] {});
          }
          named_bar_sync(4, 256);  // the CTA's attention done (worker 0 arrives for it)
          wait_bar(5 * i + 1);
        }
        // the phase's inputs (also orders this CTA's arrival after barrier k-1)
        const int kin = m == 0 ? 5 * i - 1 : 5 * i + m;
        if (m != 1) wait_bar(kin);
        const bool norm = m == 0 || m == 2;
        PassShare sh;
        pass_share(M, P.np, sh);
        const int crank = sh.crank;
        const int K = M.K;
        TcTiles tl;
        tl.init(sh.u0, sh.u1, M.R >> 3, M.tg);
        int tp, g0, tg, cur_p = -1;
        while (tl.next(tp, g0, tg)) {
          const int buf = ti & 1;
          const int nvp = P.nv[tp];
          const int nblk = (3 * nvp + 15) >> 4;
          const int g = P.pg[tp];
          if (norm && crank == 0 && tp != cur_p) {  // 1/rms of this problem's vectors
            cur_p = tp;
            const int nvec8 = K >> 3;
            for (int v = 0; v < nvp; ++v) {
              const float* sp = a.g.x + (size_t)(W.slot[g] + v) * a.g.dm.d;
              float ss = 0.f;
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
              s_rstd[et] = 1.0f / sqrtf(tot / (float)K + a.g.dm.eps);
            }
            named_bar_sync(1, 128);
          }
          const int rl = 32 * quad + lane;
          float xres[kMaxVec];
          if ((m == 1 || m == 3) && crank == 0 && rl < tg * 8) {
            const float* xr = a.g.x + (size_t)W.slot[g] * a.g.dm.d + g0 * 8 + rl;
#pragma unroll
            for (int v = 0; v < kMaxVec; ++v)
              if (v < nvp) xres[v] = __ldcg(xr + (size_t)v * a.g.dm.d);
          }
          mbar_wait(&acc_full[buf], (ti >> 1) & 1);
          tc_fence_after_sync();
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
          ++ti;
          float part[kMaxVec];
#pragma unroll
          for (int v = 0; v < kMaxVec; ++v) part[v] = 0.f;
          if constexpr (CS > 1) {
            if (M.cs > 1) {
              if (crank != 0) {  // ship this rank's row sums to the leader
                if (xt >= 1) mbar_wait_cluster(recv_empty, (xt - 1) & 1);
                if (quad_live) {
                  const uint32_t dst = map_rank(smem_u32(recv), 0) + (uint32_t)(rl * 4);
#pragma unroll
                  for (int v = 0; v < kMaxVec; ++v) {
                    if (v >= nvp) break;
                    st_cluster_f32(dst + (uint32_t)(v * 128 * 4), (c[3 * v] + c[3 * v + 1]) + c[3 * v + 2]);
                  }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(map_rank(smem_u32(recv_full), 0));
                ++xt;
                continue;
              }
              mbar_wait_cluster(recv_full, xt & 1);
#pragma unroll
              for (int v = 0; v < kMaxVec; ++v)
                if (v < nvp && quad_live) part[v] = recv[v * 128 + rl];
              __syncwarp();
              if (lane == 0)  // every tile's buffer release (the partner waits for each)
                mbar_arrive_cluster(map_rank(smem_u32(recv_empty), 1));
              ++xt;
            }
          }
          if (!quad_live) continue;
          const bool valid = rl < tg * 8;
          const int rr = g0 * 8 + rl;
          auto yv = [&](int v) {
            float y = (c[3 * v] + c[3 * v + 1]) + c[3 * v + 2];
            if (CS > 1 && M.cs > 1) y = y + part[v];
            return norm ? y * s_rstd[v] : y;
          };
          if (m == 0 || m == 2) {  // row pairs: RoPE + paged KV append / SwiGLU
#pragma unroll
            for (int v = 0; v < kMaxVec; ++v) {
              if (v >= nvp) break;
              const float y = yv(v);
              const float yp = __shfl_xor_sync(0xffffffffu, y, 1);
              if (!valid || (lane & 1)) continue;
              const int slot = W.slot[g] + v, pos = W.pos[g] + v;
              if (m == 2) {
                a.g.h[(size_t)slot * a.g.dm.ffn + (rr >> 1)] = y / (1.0f + expf(-y)) * yp;
              } else {
                const int H = a.g.dm.H, KVh = a.g.dm.KV, hd = a.g.dm.hd;
                const LayerW& L = a.g.layers[P.li[tp]];
                const int head = rr / hd, wi = rr - head * hd;
                float o0 = y, o1 = yp;
                void* cache = nullptr;
                int kvh = 0;
                if (head < H + KVh) {
                  const int half = hd >> 1;
                  const float cs_ = a.g.rope_cos[(size_t)pos * half + (wi >> 1)];
                  const float sn = a.g.rope_sin[(size_t)pos * half + (wi >> 1)];
                  o0 = y * cs_ - yp * sn;
                  o1 = yp * cs_ + y * sn;
                  if (head < H) {
                    float* q = a.g.q + (size_t)slot * H * hd + head * hd + wi;
                    q[0] = o0;
                    q[1] = o1;
                  } else {
                    cache = L.kc;
                    kvh = head - H;
                  }
                } else {
                  cache = L.vc;
                  kvh = head - H - KVh;
                }
                if (cache) {
                  const int page = a.g.page_table[pos / kPage];
                  const size_t off = (((size_t)page * KVh + kvh) * kPage + (pos % kPage)) * hd + wi;
                  if (a.g.dm.kv_bf16) {
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
          } else if (valid) {  // residual add
#pragma unroll
            for (int v = 0; v < kMaxVec; ++v) {
              if (v >= nvp) break;
              a.g.x[(size_t)(W.slot[g] + v) * a.g.dm.d + rr] = xres[v] + yv(v);
            }
          }
        }
        arrive_bar();  // barrier 5i + (0 | 2 | 3 | 4)
      }
    }
    // the launch's last barrier: every CTA's down projection is in x; the
    // last CTA to finish publishes the next launch's barrier base
    named_bar_sync(1, 128);
    if (et == 0) {
      __threadfence();
      if (atomicAdd(a.done_cnt, 1u) == gridDim.x - 1) {
        *a.done_cnt = 0;
        *a.bar_seq = base + (unsigned long long)ntot * grid;
        __threadfence();
      }
    }
  }
  if (CS > 1) {  // the leader's last buffer release reaches the partner before either exits
    if (warp < 6) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    cluster_sync_all();
  }
  tc_fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kTcTmemCols));
  }
}

// ---------------------------------------------------------------------------
// host side

namespace {
template <int CS, int HD, typename KVT, int QPK>
cudaError_t tp_one(const TcPassArgs& a, size_t smem, int grid, cudaStream_t st, bool attrs_only) {
  auto fn = tcpass_kernel<CS, HD, KVT, QPK>;
  if (attrs_only) return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
template <int CS, int HD, typename KVT>
cudaError_t tp_qpk(const TcPassArgs& a, int qpk, size_t smem, int grid, cudaStream_t st, bool attrs) {
  switch (qpk) {
    case 1: return tp_one<CS, HD, KVT, 1>(a, smem, grid, st, attrs);
    case 8: return tp_one<CS, HD, KVT, 8>(a, smem, grid, st, attrs);
  }
  return cudaErrorInvalidValue;
}
template <int CS>
cudaError_t tp_cs(const TcPassArgs& a, int qpk, int kv_bf16, size_t smem, int grid, cudaStream_t st, bool attrs) {
  return kv_bf16 ? tp_qpk<CS, 128, __nv_bfloat16>(a, qpk, smem, grid, st, attrs)
                 : tp_qpk<CS, 128, float>(a, qpk, smem, grid, st, attrs);
}
cudaError_t tp_dispatch(const TcPassArgs& a, int cs, int hd, int qpk, int kv_bf16, size_t smem, int grid,
                        cudaStream_t st, bool attrs) {
  if (hd != 128) return cudaErrorInvalidValue;
  switch (cs) {
    case 1: return tp_cs<1>(a, qpk, kv_bf16, smem, grid, st, attrs);
    case 2: return tp_cs<2>(a, qpk, kv_bf16, smem, grid, st, attrs);
  }
  return cudaErrorInvalidValue;
}
}  // namespace

bool tc_pass_supported(int hd, int qpk) { return hd == 128 && (qpk == 1 || qpk == 8); }

size_t tc_pass_scratch_bytes(int hd, int qpk, int kv_bf16) {
  (void)kv_bf16;
  if (hd != 128) return 0;
  return qpk == 8 ? sizeof(AttnScratch<128, 8>) : sizeof(AttnScratch<128, 1>);
}

cudaError_t tc_pass_set_attrs(int cs, int hd, int qpk, int kv_bf16, size_t smem) {
  TcPassArgs dummy{};
  return tp_dispatch(dummy, cs, hd, qpk, kv_bf16, smem, 0, 0, true);
}

int tc_pass_trace_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_tc_trace, sizeof(g_tc_trace)) == cudaSuccess ? 0 : -1;
}
int tc_pass_trace_enable(int on) {
  return cudaMemcpyToSymbol(g_tc_trace_on, &on, sizeof(int)) == cudaSuccess ? 0 : -1;
}

cudaError_t tc_pass_launch(const TcPassArgs& a, int cs, int hd, int qpk, int kv_bf16, size_t smem, int grid,
                           cudaStream_t st) {
  return tp_dispatch(a, cs, hd, qpk, kv_bf16, smem, grid, st, false);
}

}  // namespace ppsd
