"""ctypes driver for libppsd_host.so (host build of csrc/sched.h) — test helper.

`run_toy` / `run_bernoulli` mimic what the GPU engine does each tick
(sched_plan -> per-stage compute + heads -> sched_finish) with the model
compute done by the oracle port, so the plan/finish split of the shipped
scheduler can be checked against the reference goldens on a CPU box.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from oracle import specpipe_port as sp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(ROOT, "paper_2509_19368_b200", "libppsd_host.so")
KINDS = ("ACTIVATION", "DRAFT_TOKEN", "FINAL_TOKEN", "CHECK_TOKEN")
VERDICTS = ("", "accept", "reject")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            import subprocess

            subprocess.check_call(["make", "-C", os.path.join(ROOT, "paper_2509_19368_b200", "csrc"),
                                   "host"])
        L = C.CDLL(LIB_PATH)
        L.ppsdh_create.restype = C.c_void_p
        L.ppsdh_create.argtypes = [C.c_int] * 7 + [C.POINTER(C.c_int32), C.c_int, C.c_int,
                                                  C.c_double, C.c_uint64, C.c_int, C.c_uint64,
                                                  C.c_int64]
        L.ppsdh_destroy.argtypes = [C.c_void_p]
        L.ppsdh_plan.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.ppsdh_finish.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ppsdh_finish_sampled.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.ppsdh_set_fold.argtypes = [C.c_void_p, C.c_int]
        L.ppsdh_fold_width.argtypes = [C.c_void_p]
        L.ppsdh_fold_plan.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        L.ppsdh_set_rfold.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ppsdh_rfold_first.argtypes = [C.c_void_p, C.c_int]
        L.ppsdh_rfold_useful.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ppsdh_rfold_plan.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
        L.ppsdh_chain_pos.argtypes = [C.c_void_p, C.c_int]
        L.ppsdh_chain_tok.argtypes = [C.c_void_p, C.c_int]
        L.ppsdh_prefix_digest.argtypes = [C.c_void_p, C.c_int]
        L.ppsdh_prefix_digest.restype = C.c_uint64
        L.ppsdh_token.argtypes = [C.c_void_p, C.c_int]
        L.ppsdh_state.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        L.ppsdh_trace.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int64]
        L.ppsdh_trace.restype = C.c_int64
        _lib = L
    return _lib


class HostSched:
    def __init__(self, n_layers, exit_depth, *, exit_stage=0, comm_latency=0, model=1,
                 force_reject=False, stop=0, prompt=(), alpha=0.0, verify_seed=0,
                 toy_seed=None, max_ctx=8192, trace_cap=1 << 20):
        L = lib()
        arr = (C.c_int32 * max(1, len(prompt)))(*prompt)
        self.h = L.ppsdh_create(n_layers, exit_depth, exit_stage or 0, comm_latency, model,
                                int(force_reject), stop, arr, len(prompt), max_ctx, alpha,
                                verify_seed, int(toy_seed is not None), toy_seed or 0, trace_cap)
        if not self.h:
            raise ValueError("bad pipeline config")
        self.n_prompt = len(prompt)
        self.layers = sp.stage_layers(n_layers, exit_depth)
        self.S = len(self.layers)
        self.per = 1 + comm_latency
        self.work = (C.c_int32 * (self.S + 2))()
        self.info = (C.c_int32 * 8)()

    def __del__(self):
        if getattr(self, "h", None):
            lib().ppsdh_destroy(self.h)
            self.h = None

    def plan(self):
        r = lib().ppsdh_plan(self.h, self.work, self.info)
        return r, list(self.work), list(self.info)

    def set_fold(self, on=True):
        lib().ppsdh_set_fold(self.h, int(on))

    def fold_width(self):
        return lib().ppsdh_fold_width(self.h)

    def fold_plan(self):
        out = (C.c_int32 * 6)()
        lib().ppsdh_fold_plan(self.h, out)
        return list(out)

    def finish(self, exit_tok=-1, final_tok=-1, final_ok=None):
        if final_ok is None:
            lib().ppsdh_finish(self.h, exit_tok, final_tok)
        else:
            lib().ppsdh_finish_sampled(self.h, exit_tok, final_tok, int(final_ok))

    def chain_pos(self, slot):
        return lib().ppsdh_chain_pos(self.h, slot)

    def chain_tok(self, slot):
        return lib().ppsdh_chain_tok(self.h, slot)

    def prefix_digest(self, n):
        return lib().ppsdh_prefix_digest(self.h, n)

    def state(self):
        out = (C.c_int64 * 6)()
        lib().ppsdh_state(self.h, out)
        return list(out)

    def tokens(self, n):
        return [lib().ppsdh_token(self.h, self.n_prompt + i) for i in range(n)]

    def trace_rows(self):
        n = self.state()[5]
        buf = (C.c_int32 * (6 * max(1, n)))()
        n = lib().ppsdh_trace(self.h, buf, n)
        a = np.frombuffer(buf, dtype=np.int32)[: 6 * n].reshape(n, 6)
        return [(int(t), int(s), KINDS[k], int(p), None if tok < 0 else int(tok), VERDICTS[v])
                for t, s, k, p, tok, v in a]

    def metrics(self):
        committed, ticks, acc, rej, err, _ = self.state()
        assert err == 0, f"scheduler error flags {err}"
        return sp.make_metrics(committed, ticks, acc, rej, acc + rej, self.S * self.per)


def _toy_heads(lm, n_layers, layers, k, S, digest_of, exit_slot, final_slot):
    exit_tok = final_tok = -1
    if exit_slot >= 0:
        d = digest_of[exit_slot]
        layer_after = sum(layers[:k])
        fin = lm.advance_digest(d, layer_after, n_layers)
        exit_tok = sp.first_argmax(lm.exit_logits(fin, d))
    if final_slot >= 0:
        final_tok = sp.first_argmax(lm.logits(digest_of[final_slot]))
    return exit_tok, final_tok


def run_toy(lm, n_layers, exit_depth, prompt, stop, *, exit_stage=0, comm_latency=0,
            force_reject=False):
    """Single-rank engine emulation: plan -> toy stage compute -> heads -> finish."""
    hs = HostSched(n_layers, exit_depth, exit_stage=exit_stage, comm_latency=comm_latency,
                   model=1, force_reject=force_reject, stop=stop, prompt=prompt, toy_seed=lm.seed)
    if stop == 0:
        return [], sp.make_metrics(0, 0, 0, 0, 0, hs.S * hs.per), []
    layers = hs.layers
    first = [sum(layers[:i]) for i in range(len(layers))]
    dig = {}
    while True:
        r, work, info = hs.plan()
        if not r:
            break
        k = info[6]
        for st in range(1, hs.S + 1):
            slot = work[st]
            if slot < 0:
                continue
            if st == 1 and info[1]:
                pos = hs.chain_pos(slot)
                dig[slot] = hs.prefix_digest(hs.n_prompt + pos - 1)
            a = first[st - 1]
            dig[slot] = lm.advance_digest(dig[slot], a, a + layers[st - 1])
        e, f = _toy_heads(lm, n_layers, layers, k, hs.S, dig, info[2], info[3])
        hs.finish(e, f)
    m = hs.metrics()
    return hs.tokens(m[0]), m, hs.trace_rows()


def run_toy_folded(lm, n_layers, exit_depth, prompt, stop, *, exit_stage=0, comm_latency=0,
                   force_reject=False, max_batch=16):
    """Folded single-device emulation (sched.h: sched_fold_plan), mirroring
    what sched_tick_kernel and the folded tick graph do: the launched chain's
    shallow stages + exit head run in its launch tick (the draft is kept per
    chain until the machine emits it at stage k); when the chain at stage S
    has no deep result, every chain past deep_done goes through the deep
    layers + final head as one batch in fold rows 0..nb-1. Checks the row and
    batch invariants the device kernels rely on. Returns (tokens, metrics,
    trace, batch sizes)."""
    hs = HostSched(n_layers, exit_depth, exit_stage=exit_stage, comm_latency=comm_latency,
                   model=1, force_reject=force_reject, stop=stop, prompt=prompt, toy_seed=lm.seed)
    hs.set_fold(True)
    if stop == 0:
        return [], sp.make_metrics(0, 0, 0, 0, 0, hs.S * hs.per), [], []
    width = hs.fold_width()
    assert width <= max_batch
    shallow = sum(hs.layers[:(exit_stage or 1)])
    draft = {}       # slot -> eager exit-head argmax
    row_pos = {}     # fold row -> position of the chain living there
    final = []       # final-head argmax per vector of the latest batch
    base = 0
    batches = []
    while True:
        r, work, info = hs.plan()
        if not r:
            break
        launched, exit_slot, final_slot = info[1], info[2], info[3]
        row, nb, fbase, deep_done, shallow_c, deep_before = hs.fold_plan()
        assert shallow_c == shallow
        if launched:  # shallow stages + exit head of the new chain, now
            slot = work[1]
            pos = hs.chain_pos(slot)
            assert row == pos - deep_before - 1 and 0 <= row < width, (row, pos, deep_before)
            row_pos[row] = pos
            d = hs.prefix_digest(hs.n_prompt + pos - 1)
            ex = lm.advance_digest(d, 0, shallow)
            draft[slot] = sp.first_argmax(lm.exit_logits(lm.advance_digest(ex, shallow, n_layers), ex))
        else:
            assert row == -1
        if nb > 0:  # deep batch over rows 0..nb-1 = positions fbase..fbase+nb-1
            assert 1 <= nb <= width and fbase == deep_before + 1 and deep_done == fbase + nb - 1
            for i in range(nb):
                assert row_pos.get(i) == fbase + i, (i, row_pos.get(i), fbase)
            base = fbase
            final = []
            for i in range(nb):
                d = hs.prefix_digest(hs.n_prompt + fbase + i - 1)
                final.append(sp.first_argmax(lm.logits(lm.advance_digest(d, 0, n_layers))))
            batches.append(nb)
        e = draft[exit_slot] if exit_slot >= 0 else -1
        f = -1
        if final_slot >= 0:
            p = hs.chain_pos(final_slot)
            assert base <= p < base + len(final), (p, base, len(final))
            f = final[p - base]
        hs.finish(e, f)
    m = hs.metrics()
    return hs.tokens(m[0]), m, hs.trace_rows(), batches


def run_bernoulli(n_layers, exit_depth, alpha, horizon, verify_seed, *, exit_stage=0,
                  comm_latency=0):
    hs = HostSched(n_layers, exit_depth, exit_stage=exit_stage, comm_latency=comm_latency,
                   model=0, stop=horizon, alpha=alpha, verify_seed=verify_seed)
    while hs.plan()[0]:
        hs.finish()
    return hs.metrics(), hs.trace_rows()


def run_toy_multirank_folded(lm, n_layers, exit_depth, prompt, stop, world, *, exit_stage=0,
                             comm_latency=0, force_reject=False, max_batch=16):
    """Multi-rank emulation with the per-rank fold (sched.h: sched_rfold_plan):
    `world` replicated schedulers, one per rank, each owning a contiguous stage
    range (distributed.stage_owner). A rank whose deferred part spans >= 2
    stages folds: its eager stages (lo..k) + exit head run when a chain
    reaches stage lo, its deferred stages run as one batch when the oldest
    unprocessed chain is due at stage hi; other ranks run every planned stage
    in its tick. Activations move between ranks only through the box of the
    tick the sender's stage hi is planned, and arrive at the end of that tick
    (the engine's exchange). Every input is checked to exist when used.
    Returns (tokens, metrics, trace, {rank: batch sizes})."""
    owner = [-1] + [(st - 1) * world // -(-n_layers // exit_depth) for st in
                    range(1, -(-n_layers // exit_depth) + 1)]
    ranks = []
    for r in range(world):
        hs = HostSched(n_layers, exit_depth, exit_stage=exit_stage, comm_latency=comm_latency,
                       model=1, force_reject=force_reject, stop=stop, prompt=prompt,
                       toy_seed=lm.seed)
        sts = [st for st in range(1, hs.S + 1) if owner[st] == r]
        lo, hi = sts[0], sts[-1]
        fold = bool(lib().ppsdh_rfold_useful(hs.h, lo, hi))
        width = 0
        if fold:
            width = lib().ppsdh_set_rfold(hs.h, lo, hi)
            fold = width <= max_batch
            assert fold, "the engine runs such a rank pipelined"
        ranks.append(dict(hs=hs, lo=lo, hi=hi, fold=fold, width=width, dlo=lib().ppsdh_rfold_first(hs.h, lo),
                          act={}, draft={}, final={}, out={}, recv={}, batches=[]))
    hs0 = ranks[0]["hs"]
    if stop == 0:
        return [], sp.make_metrics(0, 0, 0, 0, 0, hs0.S * hs0.per), [], {}
    layers = hs0.layers
    S = hs0.S
    first = [0] + [sum(layers[:i]) for i in range(S)]  # 1-based: first[st] = first layer of stage st
    last = [0] + [sum(layers[:i + 1]) for i in range(S)]
    while True:
        plans = [R["hs"].plan() for R in ranks]
        r0, work, info = plans[0]
        for p in plans[1:]:
            assert p == plans[0]  # replicated
        if not r0:
            break
        k = info[6]
        exit_slot, final_slot = info[2], info[3]
        sent = {}
        exit_tok = final_tok = -1
        for rank, R in enumerate(ranks):
            hs, lo, hi = R["hs"], R["lo"], R["hi"]
            pos_of = hs.chain_pos

            def stage_input(slot):
                pos = pos_of(slot)
                if lo == 1:
                    return hs.prefix_digest(hs.n_prompt + pos - 1)
                assert pos in R["recv"], f"rank {rank}: chain {pos} used before its box arrived"
                return R["recv"][pos]

            if R["fold"]:
                out5 = (C.c_int32 * 5)()
                lib().ppsdh_rfold_plan(hs.h, out5)
                nb, base, deep_done, arrived, before = list(out5)
                a = work[lo]
                if a >= 0:  # arrival at stage lo: input now, eager stages + exit head
                    pos = pos_of(a)
                    d = stage_input(a)
                    if lo <= k:
                        d = lm.advance_digest(d, first[lo], last[k])
                        fin = lm.advance_digest(d, last[k], n_layers)
                        R["draft"][pos] = sp.first_argmax(lm.exit_logits(fin, d))
                    R["act"][pos] = d
                if nb > 0:
                    assert base == before + 1 and 1 <= nb <= R["width"] and deep_done == base + nb - 1
                    assert arrived == deep_done
                    for p in range(base, base + nb):
                        assert p in R["act"], f"rank {rank}: batch chain {p} has no input"
                        o = lm.advance_digest(R["act"][p], first[R["dlo"]], last[hi])
                        R["out"][p] = o
                        if hi == S:
                            R["final"][p] = sp.first_argmax(lm.logits(o))
                    R["batches"].append(nb)
                due = work[hi]
                if due >= 0:
                    p = pos_of(due)
                    assert p <= deep_done and p in R["out"], f"rank {rank}: chain {p} due without output"
                    if hi < S:
                        sent[rank] = (p, R["out"][p])
                    else:
                        final_tok = R["final"][p]
                if lo <= k <= hi and exit_slot >= 0:
                    exit_tok = R["draft"][pos_of(exit_slot)]
            else:  # pipelined rank: every planned stage in its tick
                for st in range(lo, hi + 1):
                    slot = work[st]
                    if slot < 0:
                        continue
                    pos = pos_of(slot)
                    d = stage_input(slot) if st == lo else R["act"][pos]
                    R["act"][pos] = lm.advance_digest(d, first[st], last[st])
                    if st == k:
                        fin = lm.advance_digest(R["act"][pos], last[k], n_layers)
                        exit_tok = sp.first_argmax(lm.exit_logits(fin, R["act"][pos]))
                    if st == hi and hi < S:
                        sent[rank] = (pos, R["act"][pos])
                    if st == S:
                        final_tok = sp.first_argmax(lm.logits(R["act"][pos]))
        for rank, (p, d) in sent.items():  # the exchange at the end of the tick
            ranks[rank + 1]["recv"][p] = d
        for R in ranks:
            R["hs"].finish(exit_tok, final_tok)
    ms = [R["hs"].metrics() for R in ranks]
    rows = [R["hs"].trace_rows() for R in ranks]
    for m, rw in zip(ms[1:], rows[1:]):
        assert m == ms[0] and rw == rows[0]
    m = ms[0]
    return hs0.tokens(m[0]), m, rows[0], {i: R["batches"] for i, R in enumerate(ranks) if R["fold"]}
