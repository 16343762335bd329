// sched.cu — the device-resident tick machine and the per-tick bookkeeping
// kernels. One CTA: the scheduler state (~14 KB) is staged into shared memory
// by all threads, thread 0 runs sched_finish(t) + sched_plan(t+1) from
// sched.h, the local work descriptor is written for the layer kernels, and
// the chain launched at stage 1 gets its input (embedding row / ToyLM prefix
// digest). No host round trip per tick: the host only enqueues tick graphs.
#include "engine_dev.cuh"

namespace ppsd {

__device__ void copy_words(void* dst, const void* src, int bytes) {
  const int n = bytes / 4;
  const int* s = reinterpret_cast<const int*>(src);
  int* d = reinterpret_cast<int*>(dst);
  for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = s[i];
}

__device__ void embed_row(const TickCtx& c, int slot, int tok) {
  const __nv_bfloat16* row = c.embed + (size_t)tok * c.d;
  float* x = c.x + (size_t)slot * c.d;
  for (int i = threadIdx.x; i < c.d; i += blockDim.x) x[i] = __bfloat162float(row[i]);
}

__global__ void __launch_bounds__(256) sched_tick_kernel(const TickCtx* ctxp, int begin) {
  __shared__ __align__(16) Sched s;
  __shared__ int s_launch_slot, s_launch_pos;
  pdl_wait();  // head results of this tick
  pdl_trigger();
  const TickCtx c = *ctxp;
  copy_words(&s, c.sched, sizeof(Sched));
  __syncthreads();
  if (threadIdx.x == 0) {
    if (!begin) sched_finish(&s, c.work->head_out[0], c.work->head_out[1], c.tokens, c.pdig,
                             c.trace, c.trace_cap);
    sched_plan(&s);
    Work* w = c.work;
    w->G = c.hi - c.lo + 1;
    for (int g = 0; g < w->G; ++g) {
      const int st = c.lo + g;
      const int slot = s.work[st];
      w->slot[g] = slot;
      w->pos[g] = slot >= 0 ? s.c.n_prompt + s.ch_pos[slot] - 2 : 0;
      w->first[g] = s.c.stage_first[st];
      w->nl[g] = s.c.stage_layers[st];
    }
    w->head_slot[0] = (s.c.k >= c.lo && s.c.k <= c.hi) ? s.exit_slot : -1;
    w->head_slot[1] = (s.c.S >= c.lo && s.c.S <= c.hi) ? s.final_slot : -1;
    s_launch_slot = (s.launched && c.lo == 1) ? s.work[1] : -1;
    s_launch_pos = s_launch_slot >= 0 ? s.ch_pos[s_launch_slot] : 0;
  }
  __syncthreads();
  const int slot = s_launch_slot;
  if (slot >= 0) {
    const int idx = s.c.n_prompt + s_launch_pos - 2;  // last token of the chain's prefix
    if (c.model == PPSD_MODEL_TRANSFORMER) {
      embed_row(c, slot, c.tokens[idx]);
    } else if (c.model == PPSD_MODEL_TOYLM && threadIdx.x == 0) {
      c.chain_dig[slot] = c.pdig[idx + 1];  // prefix digest (pipesim.py:768)
    }
  }
  copy_words(c.sched, &s, sizeof(Sched));
}

// ---- autoregressive / prefill control (decode_autoregressive, pipesim.py:390-409)
__global__ void __launch_bounds__(256) ar_begin_kernel(const TickCtx* ctxp, ArCtl* ctl, int with_head) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  const int j = ctl->j;
  if (threadIdx.x == 0) {
    Work* w = c.work_ar;
    w->G = 1;
    w->slot[0] = 0;
    w->pos[0] = j;
    w->first[0] = ctl->first_layer;
    w->nl[0] = ctl->n_layers;
    w->head_slot[0] = -1;
    w->head_slot[1] = with_head ? 0 : -1;
  }
  embed_row(c, 0, c.tokens[j]);
}

__global__ void ar_end_kernel(const TickCtx* ctxp, ArCtl* ctl, int with_head) {
  pdl_wait();
  pdl_trigger();
  const TickCtx c = *ctxp;
  if (threadIdx.x == 0) {
    const int j = ctl->j;
    if (with_head) c.tokens[j + 1] = c.work_ar->head_out[1];
    ctl->j = j + 1;
  }
}

}  // namespace ppsd
