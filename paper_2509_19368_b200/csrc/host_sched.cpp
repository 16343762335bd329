// host_sched.cpp — host build of the tick machine in sched.h (g++, no CUDA).
//
// The device scheduler kernel (sched.cu) and this library compile the SAME
// sched.h. The CPU test-suite drives this build with oracle model compute to
// check (a) the plan/finish split against the reference goldens and (b) the
// replicated-scheduler protocol of the multi-rank path over gloo, which this
// container can run without a GPU. It is never loaded by the product path.
#include <stdlib.h>
#include <string.h>

#include "sched.h"

using namespace ppsd;

namespace {
struct HostSched {
  Sched s;
  int32_t* tokens;
  uint64_t* pdig;
  TraceRow* trace;
  int64_t cap;
};
}  // namespace

extern "C" {

void* ppsdh_create(int n_layers, int exit_depth, int exit_stage, int comm_latency, int model,
                   int force_reject, int stop, const int32_t* prompt, int n_prompt, int max_ctx,
                   double alpha, uint64_t verify_seed, int toy, uint64_t toy_seed, int64_t trace_cap) {
  HostSched* h = (HostSched*)calloc(1, sizeof(HostSched));
  if (!h) return nullptr;
  if (sched_configure(&h->s.c, n_layers, exit_depth, exit_stage, comm_latency) != 0) {
    free(h);
    return nullptr;
  }
  h->s.c.model = model;
  h->s.c.force_reject = force_reject;
  h->s.c.stop = stop;
  h->s.c.n_prompt = n_prompt;
  h->s.c.alpha = alpha;
  h->s.c.verify_seed = verify_seed;
  h->tokens = (int32_t*)calloc(max_ctx + 1, sizeof(int32_t));
  h->pdig = toy ? (uint64_t*)calloc(max_ctx + 2, sizeof(uint64_t)) : nullptr;
  for (int i = 0; i < n_prompt; ++i) h->tokens[i] = prompt[i];
  if (h->pdig) {
    h->pdig[0] = hmix64(toy_seed ^ kSeqSalt);
    for (int i = 0; i < n_prompt; ++i) h->pdig[i + 1] = toy_extend(h->pdig[i], prompt[i]);
  }
  h->cap = trace_cap;
  h->trace = trace_cap > 0 ? (TraceRow*)calloc(trace_cap, sizeof(TraceRow)) : nullptr;
  sched_reset(&h->s);
  return h;
}

void ppsdh_destroy(void* p) {
  HostSched* h = (HostSched*)p;
  if (!h) return;
  free(h->tokens);
  free(h->pdig);
  free(h->trace);
  free(h);
}

// info: [t, launched, exit_slot, final_slot, done, S, k, nslot]; work: [S+2]
int ppsdh_plan(void* p, int32_t* work, int32_t* info) {
  HostSched* h = (HostSched*)p;
  int r = sched_plan(&h->s);
  for (int i = 0; i <= h->s.c.S + 1; ++i) work[i] = h->s.work[i];
  info[0] = h->s.t;
  info[1] = h->s.launched;
  info[2] = h->s.exit_slot;
  info[3] = h->s.final_slot;
  info[4] = h->s.done;
  info[5] = h->s.c.S;
  info[6] = h->s.c.k;
  info[7] = h->s.c.nslot;
  return r;
}

void ppsdh_finish(void* p, int exit_tok, int final_tok) {
  HostSched* h = (HostSched*)p;
  sched_finish(&h->s, exit_tok, final_tok, h->tokens, h->pdig, h->trace, h->cap);
}

// sampling: the verdict (final_ok) and committed token come from the model side
void ppsdh_finish_sampled(void* p, int exit_tok, int final_tok, int final_ok) {
  HostSched* h = (HostSched*)p;
  sched_finish(&h->s, exit_tok, final_tok, h->tokens, h->pdig, h->trace, h->cap, final_ok);
}

// folded schedule (sched.h: sched_fold_plan)
void ppsdh_set_fold(void* p, int on) { ((HostSched*)p)->s.c.fold = on; }
int ppsdh_fold_width(void* p) { return sched_fold_width(&((HostSched*)p)->s.c); }

// out: [fold_row, fold_nb, fold_base, deep_done, shallow_layers, deep_done before]
void ppsdh_fold_plan(void* p, int32_t* out) {
  HostSched* h = (HostSched*)p;
  out[5] = h->s.deep_done;
  sched_fold_plan(&h->s);
  out[0] = h->s.fold_row;
  out[1] = h->s.fold_nb;
  out[2] = h->s.fold_base;
  out[3] = h->s.deep_done;
  out[4] = h->s.c.shallow_layers;
}

// rank fold (sched.h: sched_rfold_plan) of stages lo..hi; returns the batch width bound
int ppsdh_set_rfold(void* p, int lo, int hi) {
  HostSched* h = (HostSched*)p;
  h->s.c.rfold = 1;
  h->s.c.rf_lo = lo;
  h->s.c.rf_hi = hi;
  return sched_rfold_width(&h->s.c, lo, hi);
}
int ppsdh_rfold_first(void* p, int lo) { return sched_rfold_first(&((HostSched*)p)->s.c, lo); }
int ppsdh_rfold_useful(void* p, int lo, int hi) { return sched_rfold_useful(&((HostSched*)p)->s.c, lo, hi); }

// out: [fold_nb, fold_base, deep_done, rf_arrived, deep_done before]
void ppsdh_rfold_plan(void* p, int32_t* out) {
  HostSched* h = (HostSched*)p;
  out[4] = h->s.deep_done;
  sched_rfold_plan(&h->s);
  out[0] = h->s.fold_nb;
  out[1] = h->s.fold_base;
  out[2] = h->s.deep_done;
  out[3] = h->s.rf_arrived;
}

int ppsdh_chain_pos(void* p, int slot) { return ((HostSched*)p)->s.ch_pos[slot]; }
int ppsdh_chain_tok(void* p, int slot) { return ((HostSched*)p)->s.ch_tok[slot]; }
uint64_t ppsdh_prefix_digest(void* p, int n) { return ((HostSched*)p)->pdig[n]; }
int32_t ppsdh_token(void* p, int idx) { return ((HostSched*)p)->tokens[idx]; }

// out: [committed, ticks, accepts, rejects, error, trace_n]
void ppsdh_state(void* p, int64_t* out) {
  HostSched* h = (HostSched*)p;
  out[0] = h->s.committed;
  out[1] = h->s.t;
  out[2] = h->s.accepts;
  out[3] = h->s.rejects;
  out[4] = h->s.error;
  out[5] = h->s.trace_n;
}

int64_t ppsdh_trace(void* p, int32_t* rows, int64_t cap) {
  HostSched* h = (HostSched*)p;
  int64_t n = h->s.trace_n < cap ? h->s.trace_n : cap;
  if (h->trace) memcpy(rows, h->trace, n * sizeof(TraceRow));
  return n;
}
}
