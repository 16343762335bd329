// p2p.cuh — NVLink peer-store transport for the multi-rank pipeline.
//
// Every rank owns an exchange buffer (cudaMalloc, shared with the other ranks
// through CUDA IPC handles): [2 parity][world][box_words] fp32 boxes, then
// world uint64 flags. Exchange number e (a per-engine device counter that
// advances identically on every rank, because every rank performs the same
// exchanges) is published by storing this rank's box into slot [e & 1][rank]
// of EVERY rank's buffer, then releasing flag[rank] = e at system scope on
// each of them; consumers acquire-wait until flag[r] >= e for all r. Each
// consumer reads parity e & 1 while producers may already write e + 1 into
// the other parity; they cannot reach e + 2 before every rank has published
// e + 1, which happens only after it finished reading e.
#pragma once
#include "engine_dev.cuh"

namespace ppsd {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t* xbuf_flags(float* xbuf, int world, int box_words) {
  return reinterpret_cast<uint64_t*>(xbuf + (size_t)2 * world * box_words);
}

// store this rank's box (already built in c.outbox) into the ranks' buffers
// (activation to the next rank only) and release the flags; returns the
// exchange number. Block-wide.
__device__ inline uint64_t p2p_publish(const TickCtx& c) {
  __shared__ uint64_t s_e;
  if (threadIdx.x == 0) {
    volatile uint64_t* xc = c.xcount;
    s_e = *xc + 1;
    *xc = s_e;
  }
  __syncthreads();
  const uint64_t e = s_e;
  const size_t slot = ((e & 1) * c.world + c.rank) * (size_t)c.box_words;
  // point to point: the activation [kBoxHeader, kBoxHeader + d) goes only to
  // the rank that runs the next stage (rank + 1, contiguous split); the
  // header (draft / final tokens) and, sampling, the owners' logits go to
  // every rank (the replicated scheduler reads them)
  const int act_end = kBoxHeader + c.d;
  for (int r = 0; r < c.world; ++r) {
    float* dst = c.peer_xbuf[r] + slot;
    const bool act = r == c.rank + 1;
    for (int i = threadIdx.x; i < c.box_used; i += blockDim.x)
      if (act || i < kBoxHeader || i >= act_end) dst[i] = c.outbox[i];
  }
  __threadfence_system();  // every storing thread orders its box stores before the flag
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int r = 0; r < c.world; ++r) st_release_sys(xbuf_flags(c.peer_xbuf[r], c.world, c.box_words) + c.rank, e);
  }
  __syncthreads();
  return e;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// wait until every rank published the engine's latest exchange; returns the
// inbox view ([world][box_words]) for it. Block-wide. A peer that never
// publishes (dead rank, wedged device) trips a sticky 20 s timeout in
// *c.xerr instead of hanging the GPU; later waits return at once and the host
// reports the error.
__device__ inline const float* p2p_wait_latest(const TickCtx& c) {
  __shared__ uint64_t s_e;
  if (threadIdx.x == 0) {
    const uint64_t e = *(volatile const uint64_t*)c.xcount;
    const uint64_t* flags = xbuf_flags(c.my_xbuf, c.world, c.box_words);
    volatile int32_t* err = c.xerr;
    const uint64_t t0 = globaltimer_ns();
    for (int r = 0; r < c.world && !*err; ++r)
      while (ld_acquire_sys(flags + r) < e) {
        __nanosleep(100);
        if (globaltimer_ns() - t0 > 20000000000ull) {
          *err = 1;
          break;
        }
      }
    s_e = e;
#ifdef PPSD_P2P_DEBUG
    {
      uint64_t* dbg = const_cast<uint64_t*>(flags) + c.world;
      const uint64_t k = dbg[0]++;
      if (k < 500) {
        uint64_t* row = dbg + 1 + k * 8;
        const float* ib = c.my_xbuf + (e & 1) * (size_t)c.world * c.box_words;
        row[0] = e;
        row[1] = ld_acquire_sys(flags + 0);
        row[2] = ld_acquire_sys(flags + (c.world - 1));
        row[3] = (uint32_t)reinterpret_cast<const int32_t*>(ib)[0];
        row[4] = (uint32_t)reinterpret_cast<const int32_t*>(ib + (size_t)(c.world - 1) * c.box_words)[1];
        row[5] = globaltimer_ns() - t0;
        row[6] = (uint64_t)(uint32_t)*err;
        row[7] = c.rank;
      }
    }
#endif
  }
  __syncthreads();
  return c.my_xbuf + (s_e & 1) * (size_t)c.world * c.box_words;
}

}  // namespace ppsd
