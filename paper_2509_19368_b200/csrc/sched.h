// sched.h — the verify-while-draft tick machine, shared by the device
// scheduler kernel (sched.cu) and a host build used by the multi-rank CPU
// tests. It restates the reference machine `_ppsd_machine`
// (pkg/src/specpipe/pipesim.py:670-789) split at the point where model
// compute happens:
//
//   sched_plan(t)   : t += 1; deliver transit (pipesim.py:722-725); pick the
//                     chain each stage runs this tick (:729-733); launch a
//                     new chain at stage 1 if t == next_launch (:766-777).
//   ...model compute for every planned (stage, chain), exit head on the
//      chain at the exit stage, final head on the chain at stage S...
//   sched_finish(t) : verdict at stage S (:739-760), drafts at the exit stage
//                     (:709-719, :762-763), emissions into transit (:703-707),
//                     launch bookkeeping (:773-777), rollback (:779-786).
//
// Trace rows are written in exactly the reference's append order so the
// exported CSV is byte-identical (pipesim.py:175-189).
//
// Chain identity: an in-flight chain is named by its activation slot
// pos % nslot. In-flight positions are contiguous and at most (S-1)*per+1
// apart (one launch per tick at most, a chain lives (S-1)*per ticks), so the
// slot is unique while the chain lives; nslot = (S-1)*per + 2.
#pragma once
#include "hostdev.h"

namespace ppsd {

constexpr int kMaxStages = 96;
constexpr int kMaxSlots = 512;
constexpr int kTransitCap = 512;

enum : int { kKindAct = 0, kKindDraft = 1, kKindFinal = 2, kKindCheck = 3 };
enum : int { kVerdictNone = 0, kVerdictAccept = 1, kVerdictReject = 2 };
enum : int { kErrOrder = 1, kErrTrace = 2, kErrTransit = 4, kErrResidual = 8 };

struct TraceRow {
  int32_t tick, stage, kind, position, token, verdict;
};

struct SchedCfg {
  int32_t S, k, per, n_layers;
  int32_t model;        // 0: Bernoulli verdicts, 1: greedy model verdicts
  int32_t force_reject;
  int32_t stop;         // stop_commits (max_tokens / horizon)
  int32_t n_prompt;
  int32_t nslot;
  int32_t fold;         // 1: folded single-GPU execution (sched_fold_plan)
  int32_t rfold;        // 1: folded stage range rf_lo..rf_hi of one rank (sched_rfold_plan)
  int32_t rf_lo, rf_hi;
  double alpha;         // Bernoulli acceptance rate
  uint64_t verify_seed; // derive_seed(rng.seed, "verify") (pipesim.py:693)
  int32_t stage_layers[kMaxStages + 1];  // 1-based
  int32_t stage_first[kMaxStages + 1];   // global index of the stage's first layer
  int32_t shallow_layers;                // layers of stages 1..k (the exit layer k*E)
};

struct Sched {
  SchedCfg c;
  int32_t t, committed, accepts, rejects, draft_head, next_launch, done, error;
  uint64_t verify_counter;
  uint64_t draft_counter, commit_counter;  // sampling-mode streams (pipesim.py:339-344)
  int64_t trace_n;
  int32_t launched;     // the stage-1 chain this tick is a fresh launch
  int32_t exit_slot;    // chain whose exit head runs this tick, -1 none
  int32_t final_slot;   // chain whose final head runs this tick, -1 none
  int32_t tq_head, tq_n;
  int32_t cur[kMaxStages + 2];
  int32_t work[kMaxStages + 2];  // chain slot each stage runs this tick, -1 idle
  int32_t tq_ready[kTransitCap], tq_dest[kTransitCap], tq_slot[kTransitCap];
  int32_t ch_pos[kMaxSlots], ch_layer[kMaxSlots], ch_tok[kMaxSlots];
  // folded execution (sched_fold_plan): see the comment there
  int32_t deep_done;     // highest position whose deep stages + final head ran on the current prefix
  int32_t fold_base;     // first position of the latest deep batch
  int32_t fold_nb;       // vectors in this tick's deep batch, 0 = none
  int32_t fold_row;      // fold row of the chain launched this tick, -1 = none
  int32_t fold_batches;  // deep batches run so far
  int32_t rf_arrived;    // rank fold: highest position that reached stage rf_lo
  int64_t fold_vectors;  // chains that went through a deep batch
  int64_t fold_pos_sum;  // sum of their positions (attention context accounting)
  int64_t fold_comb;     // deep batches that also ran the launched chain's exit head (TickCtx.fold_comb)
  int32_t ch_draft[kMaxSlots];  // eager exit-head argmax per chain
};

constexpr int32_t kNone = -1;

PPSD_HD void sched_reset(Sched* s) {
  s->t = s->committed = s->accepts = s->rejects = s->draft_head = 0;
  s->next_launch = 1;
  s->done = (s->c.stop <= 0);
  s->error = 0;
  s->verify_counter = 0;
  s->draft_counter = s->commit_counter = 0;
  s->trace_n = 0;
  s->launched = 0;
  s->exit_slot = s->final_slot = kNone;
  s->tq_head = s->tq_n = 0;
  for (int i = 0; i <= s->c.S + 1; ++i) s->cur[i] = s->work[i] = kNone;
  s->deep_done = s->fold_base = 0;
  s->fold_nb = 0;
  s->fold_row = kNone;
  s->fold_batches = 0;
  s->rf_arrived = 0;
  s->fold_vectors = s->fold_pos_sum = 0;
  s->fold_comb = 0;
}

PPSD_HD void sched_trace(Sched* s, TraceRow* tr, int64_t cap, int st, int kind, int pos, int tok,
                         int verdict) {
  if (!tr) return;
  if (s->trace_n >= cap) {
    s->error |= kErrTrace;
    return;
  }
  TraceRow r;
  r.tick = s->t;
  r.stage = st;
  r.kind = kind;
  r.position = pos;
  r.token = tok;
  r.verdict = verdict;
  tr[s->trace_n++] = r;
}

// Beginning of tick t+1: returns 0 when the run is already done.
PPSD_HD int sched_plan(Sched* s) {
  const int S = s->c.S;
  for (int i = 0; i <= S + 1; ++i) s->work[i] = kNone;
  s->launched = 0;
  s->exit_slot = s->final_slot = kNone;
  if (s->done) return 0;
  s->t += 1;
  while (s->tq_n > 0 && s->tq_ready[s->tq_head] == s->t) {  // pipesim.py:723-725
    s->cur[s->tq_dest[s->tq_head]] = s->tq_slot[s->tq_head];
    s->tq_head = (s->tq_head + 1) % kTransitCap;
    s->tq_n -= 1;
  }
  for (int st = S; st >= 2; --st) {  // pipesim.py:729-733
    s->work[st] = s->cur[st];
    s->cur[st] = kNone;
  }
  if (s->next_launch != kNone && s->t == s->next_launch) {  // pipesim.py:766-772
    const int pos = s->draft_head + 1;
    const int slot = pos % s->c.nslot;
    s->ch_pos[slot] = pos;
    s->ch_layer[slot] = 0;
    s->ch_tok[slot] = kNone;
    s->work[1] = slot;
    s->launched = 1;
    s->draft_head = pos;
    if (s->c.k != 1) s->next_launch = kNone;  // pipesim.py:775-776
  }
  s->exit_slot = s->work[s->c.k];
  s->final_slot = s->work[S];
  return 1;
}

PPSD_HD void sched_push_token(const Sched* s, int32_t* tokens, uint64_t* pdig, int idx, int tok) {
  if (tokens) tokens[idx] = tok;
  if (pdig) pdig[idx + 1] = toy_extend(pdig[idx], tok);
  (void)s;
}

// make_draft (pipesim.py:709-719) for a chain at stage st with exit-head argmax tok
PPSD_HD void sched_draft(Sched* s, int slot, int st, int exit_tok, int32_t* tokens, uint64_t* pdig,
                         TraceRow* tr, int64_t cap) {
  int tok = kNone;
  if (s->c.model != 0) {
    tok = exit_tok;
    s->ch_tok[slot] = tok;
    sched_push_token(s, tokens, pdig, s->c.n_prompt + s->ch_pos[slot] - 1, tok);
  }
  sched_trace(s, tr, cap, st, kKindDraft, s->ch_pos[slot], tok, kVerdictNone);
  s->next_launch = s->t + (st == 1 ? 1 : s->c.per);
}

// emit_activation (pipesim.py:703-707)
PPSD_HD void sched_emit(Sched* s, int slot, int st, TraceRow* tr, int64_t cap) {
  sched_trace(s, tr, cap, st, kKindAct, s->ch_pos[slot], kNone, kVerdictNone);
  if (s->tq_n >= kTransitCap) {
    s->error |= kErrTransit;
    return;
  }
  const int tail = (s->tq_head + s->tq_n) % kTransitCap;
  s->tq_ready[tail] = s->t + s->c.per;
  s->tq_dest[tail] = st + 1;
  s->tq_slot[tail] = slot;
  s->tq_n += 1;
}

// End of tick t. exit_tok / final_tok are the exit and final heads' outputs for
// s->exit_slot / s->final_slot (ignored for Bernoulli). Greedy: final_ok < 0
// and the verdict is greedy_match. Sampling: the model side already ran
// accept_draft / the residual resample (pipesim.py:351-365) and passes the
// verdict in final_ok with the committed token in final_tok.
PPSD_HD void sched_finish(Sched* s, int exit_tok, int final_tok, int32_t* tokens, uint64_t* pdig,
                          TraceRow* tr, int64_t cap, int final_ok = -1) {
  // a tick that sched_plan declined (run already done) leaves work[] idle
  // and launched == 0, so nothing below fires.
  const int S = s->c.S, k = s->c.k;
  int rollback = kNone, corrected = kNone;
  for (int st = S; st >= 2; --st) {  // pipesim.py:729-764
    const int slot = s->work[st];
    if (slot == kNone) continue;
    s->ch_layer[slot] += s->c.stage_layers[st];
    if (st == S) {
      const int pos = s->ch_pos[slot];
      if (pos != s->committed + 1) s->error |= kErrOrder;  // pipesim.py:740-741
      bool ok;
      int tok;
      if (s->c.model != 0 && final_ok >= 0) {  // sampling verdict computed by the model side
        ok = final_ok != 0;
        tok = final_tok;
      } else if (s->c.model != 0) {  // greedy_match (speccore.py:116-126), pipesim.py:351-358
        ok = !s->c.force_reject && s->ch_tok[slot] == final_tok;
        tok = final_tok;  // == the draft when accepted
      } else {            // pipesim.py:749
        ok = false;
        if (!s->c.force_reject) ok = counter_uniform(s->c.verify_seed, s->verify_counter++) < s->c.alpha;
        tok = kNone;
      }
      s->committed += 1;
      if (ok) {
        s->accepts += 1;
        sched_trace(s, tr, cap, S, kKindFinal, pos, tok, kVerdictAccept);
      } else {
        s->rejects += 1;
        rollback = pos;
        corrected = tok;
        sched_trace(s, tr, cap, S, kKindCheck, pos, tok, kVerdictReject);
      }
    } else {
      if (st == k) sched_draft(s, slot, st, exit_tok, tokens, pdig, tr, cap);
      sched_emit(s, slot, st, tr, cap);
    }
  }
  if (s->launched) {  // pipesim.py:771-777
    const int slot = s->work[1];
    s->ch_layer[slot] = s->c.stage_layers[1];
    if (k == 1) sched_draft(s, slot, 1, exit_tok, tokens, pdig, tr, cap);
    sched_emit(s, slot, 1, tr, cap);
  }
  if (rollback != kNone) {  // pipesim.py:779-786
    if (s->c.fold || s->c.rfold) s->deep_done = rollback;  // deep results past the rollback belong to flushed chains
    if (s->c.rfold && s->rf_arrived > rollback) s->rf_arrived = rollback;
    s->tq_n = 0;
    for (int st = 1; st <= S; ++st) s->cur[st] = kNone;
    s->draft_head = rollback;
    if (s->c.model != 0) sched_push_token(s, tokens, pdig, s->c.n_prompt + rollback - 1, corrected);
    s->next_launch = s->t + s->c.per;
  }
  if (s->committed >= s->c.stop) s->done = 1;
}

// Folded execution of the machine on ONE device (SchedCfg.fold). Every stage
// shares one HBM, so time is bytes: instead of running each planned
// (stage, chain) forward in the tick it is planned (the pipelined schedule,
// one weight pass per stage per tick), the engine
//   * runs a chain's shallow stages 1..k (layers [0, k*E)) and its exit head
//     in the tick it is launched (the draft is then known early; the machine
//     still emits it at stage k, sched_finish, from ch_draft), and
//   * defers the deep stages k+1..S until a verdict needs them: in the tick the
//     chain at stage S has no deep result yet, ALL launched chains past
//     deep_done (positions deep_done+1 .. draft_head, consecutive, at most the
//     (S-1)*per+1 chains in flight) go through layers [k*E, N) and the final
//     head as ONE batch of vectors, i.e. one weight pass for up to S chains.
// Chains flushed by a rollback never run their deep stages unless they were
// already batched. Ticks, verdicts, tokens and the trace are exactly those of
// the machine: only WHEN a forward runs changes, and the batched GEMV rows are
// bit-identical to single-vector ones (gemv.cu), so the hidden states are too.
// Chain rows: the chain at position p lives in activation row
// p - deep_done - 1 (deep_done at its launch; a batch or rollback only moves
// deep_done past or back to chains no longer in flight), so a deep batch is
// rows 0 .. fold_nb-1 in position order.
PPSD_HD void sched_fold_plan(Sched* s) {
  s->fold_row = kNone;
  s->fold_nb = 0;
  if (s->launched) s->fold_row = s->ch_pos[s->work[1]] - s->deep_done - 1;
  if (s->final_slot != kNone && s->ch_pos[s->final_slot] > s->deep_done) {
    s->fold_base = s->deep_done + 1;
    s->fold_nb = s->draft_head - s->deep_done;
    s->deep_done = s->draft_head;
    s->fold_batches += 1;
    s->fold_vectors += s->fold_nb;
    s->fold_pos_sum += (int64_t)s->fold_nb * (s->fold_base + s->draft_head) / 2;
  }
}

// Largest fold row / batch the folded schedule can need: chains in flight.
PPSD_HD int sched_fold_width(const SchedCfg* c) { return (c->S - 1) * c->per + 1; }

// Folded execution of ONE RANK's stage range lo..hi (multi-rank, greedy;
// SchedCfg.rfold). The single-device fold above, restricted to a rank: the
// rank's stages up to the exit stage k ("eager": lo..k when lo <= k) run with
// the exit head in the tick the chain reaches stage lo, and the rest of its
// stages ("deferred": max(lo, k+1)..hi) run as ONE batch for every chain
// that has reached stage lo past deep_done, in the tick the oldest of them is
// due at stage hi (its activation goes into this tick's box, or its final
// head decides this tick's verdict). The rank streams its deferred weights
// once per batch instead of once per tick. Chains arrive at stage lo in
// position order, so a batch is the consecutive positions deep_done+1 ..
// rf_arrived; every chain of a batch is due at stage hi before the next batch
// is planned (the next batch is planned only when a chain past it is due), so
// the batch rows stay valid until then. Rollback: chains past the rejected
// position are flushed everywhere (sched_finish). Ticks, verdicts, tokens and
// the trace are the machine's; only WHEN a rank's forwards run changes.
PPSD_HD void sched_rfold_plan(Sched* s) {
  s->fold_nb = 0;
  const int lo = s->c.rf_lo, hi = s->c.rf_hi;
  const int a = s->work[lo];
  if (a != kNone && s->ch_pos[a] > s->rf_arrived) s->rf_arrived = s->ch_pos[a];
  const int due = s->work[hi];
  if (due != kNone && s->ch_pos[due] > s->deep_done) {
    s->fold_base = s->deep_done + 1;
    s->fold_nb = s->rf_arrived - s->deep_done;
    s->deep_done = s->rf_arrived;
    s->fold_batches += 1;
    s->fold_vectors += s->fold_nb;
    s->fold_pos_sum += (int64_t)s->fold_nb * (s->fold_base + s->rf_arrived) / 2;
  }
}

// First deferred stage of a rank fold, and the largest batch it can plan:
// chains reach stage lo at most one per tick and are due (hi - lo) * per
// ticks later.
PPSD_HD int sched_rfold_first(const SchedCfg* c, int lo) { return lo > c->k ? lo : c->k + 1; }
PPSD_HD int sched_rfold_width(const SchedCfg* c, int lo, int hi) { return (hi - lo) * c->per + 1; }
// A rank folds when it has deferred stages and more than one stage: a batch
// then holds up to (hi - lo) * per + 1 chains. (A one-stage rank past the
// exit is due the tick its chain arrives; a rank owning the exit stage
// batches even a single deferred stage, because the chain arriving this tick
// runs its eager stages before the batch.)
PPSD_HD bool sched_rfold_useful(const SchedCfg* c, int lo, int hi) {
  return sched_rfold_first(c, lo) <= hi && hi > lo;
}

// Host-side configuration helper (also used by the CPU test build).
PPSD_HD int sched_configure(SchedCfg* c, int n_layers, int exit_depth, int exit_stage,
                            int comm_latency) {
  if (n_layers < 1 || exit_depth < 1 || exit_depth > n_layers || comm_latency < 0) return -1;
  const int S = (n_layers + exit_depth - 1) / exit_depth;
  if (S < 2 || S > kMaxStages) return -1;
  const int k = exit_stage <= 0 ? 1 : exit_stage;
  if (k > S - 1) return -1;
  c->S = S;
  c->k = k;
  c->per = 1 + comm_latency;
  c->n_layers = n_layers;
  int first = 0;
  for (int st = 1; st <= S; ++st) {
    const int nl = (st < S) ? exit_depth : n_layers - (S - 1) * exit_depth;
    c->stage_layers[st] = nl;
    c->stage_first[st] = first;
    first += nl;
  }
  c->shallow_layers = c->stage_first[k] + c->stage_layers[k];
  c->fold = 0;
  c->rfold = c->rf_lo = c->rf_hi = 0;
  c->nslot = (S - 1) * c->per + 2;
  if (c->nslot > kMaxSlots || S * c->per + 2 > kTransitCap) return -1;
  return 0;
}

}  // namespace ppsd
