"""CPU oracle for the greedy PPSD decode path — TEST INFRASTRUCTURE ONLY.

This module is a from-scratch CPU restatement of the reference `specpipe`
decode semantics (the checker, never the product). Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import it. The shipped decode path runs on the GPU through
`paper_2509_19368_b200/libppsd.so` and never calls into this file.

Parity is PINNED: `tests/golden/make_golden.py` ran the real reference
(`/root/reference/pkg/src/specpipe`) in the build container and committed its
outputs under `tests/golden/`; `tests/test_oracle_golden.py` checks this port
against those fixtures token-for-token, metric-for-metric and trace-row-for-
trace-row.

What is restated (reference file:line each piece follows):

* splitmix64 finalizer, label-derived seeds, counter streams —
  `pkg/src/specpipe/rng.py:29-99`
* ToyLM digest chain, hashed logits and exit-head noise —
  `pkg/src/specpipe/toylm.py:72-130`
* greedy verification (first-index argmax on both sides) —
  `pkg/src/specpipe/speccore.py:116-126`, `pipesim.py:346-365`
* stage partition — `pkg/src/specpipe/pipesim.py:76-114`
* the verify-while-draft tick machine — `pkg/src/specpipe/pipesim.py:670-789`
* the Bernoulli schedule-only oracle — `pkg/src/specpipe/pipesim.py:636-667`
* the autoregressive oracle — `pkg/src/specpipe/pipesim.py:390-409`
* the EESD draft-then-verify rounds — `pkg/src/specpipe/pipesim.py:435-551`
* metrics — `pkg/src/specpipe/pipesim.py:256-275`

The model is reached only through the reference's 7-member duck-typed
protocol (`n_layers`, `vocab`, `empty_digest`, `extend_digest`,
`advance_digest`, `dist_from_final_state`, `exit_dist_from_states`), so the
same machine drives the ToyLM restatement below and the CPU transformer in
`oracle/transformer.py`. Distributions are plain float64 numpy vectors here.
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB
_LABEL_SALT = 0xA24BAED4963EE407

# ToyLM salts (toylm.py:25-29)
SEQ_SALT = 0x243F6A8885A308D3
TOKEN_SALT = 0x13198A2E03707344
LAYER_SALT = 0x452821E638D01377
LOGIT_SALT = 0xBE5466CF34E90C6C
NOISE_SALT = 0xC0AC29B7C97C50DD

ACTIVATION, DRAFT_TOKEN, FINAL_TOKEN, CHECK_TOKEN = (
    "ACTIVATION", "DRAFT_TOKEN", "FINAL_TOKEN", "CHECK_TOKEN")


# --------------------------------------------------------------------------
# rng.py:29-99


def mix64(x: int) -> int:
    x &= M64
    x = ((x ^ (x >> 30)) * _C1) & M64
    x = ((x ^ (x >> 27)) * _C2) & M64
    return x ^ (x >> 31)


def mix64_np(x: np.ndarray) -> np.ndarray:
    x = np.array(x, dtype=np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(_C1)
        x ^= x >> np.uint64(27)
        x *= np.uint64(_C2)
        x ^= x >> np.uint64(31)
    return x


def derive_seed(seed: int, label) -> int:
    h = mix64(seed ^ _LABEL_SALT)
    if isinstance(label, str):
        for byte in label.encode("utf-8"):
            h = mix64(h ^ (byte + 1))
        return h
    return mix64(h ^ mix64(label & M64))


class Stream:
    """Counter stream: draw i is mix64(seed + (i+1)*GOLDEN) >> 11 scaled."""

    def __init__(self, seed: int, counter: int = 0):
        self.seed = seed & M64
        self.counter = counter

    def uniform(self) -> float:
        self.counter += 1
        return (mix64((self.seed + self.counter * GOLDEN) & M64) >> 11) * 2.0 ** -53

    def randbelow(self, n: int) -> int:
        v = int(self.uniform() * n)
        return min(v, n - 1)

    def split(self, label) -> "Stream":
        return Stream(derive_seed(self.seed, label))


def default_prompt(vocab: int, rng_seed: int, length: int = 8) -> list[int]:
    """pipesim.py:290-294 (PROMPT_LEN = 8 at pipesim.py:45)."""
    s = Stream(rng_seed).split("prompt")
    return [s.randbelow(vocab) for _ in range(length)]


def first_argmax(v) -> int:
    """np.argmax semantics: lowest index among the maxima (speccore.py:116-126)."""
    return int(np.argmax(np.asarray(v)))


# speccore.py:76-113 — the sampling primitives


def sample_token(p: np.ndarray, stream: Stream) -> int:
    """Inverse CDF: first index whose running sum exceeds u (speccore.py:76-87)."""
    u = stream.uniform()
    idx = int(np.searchsorted(np.cumsum(p), u, side="right"))
    return min(idx, len(p) - 1)


def accept_draft(p_tok: float, q_tok: float, stream: Stream) -> bool:
    """r <= min(1, q/p), one draw; a token without target mass never passes (speccore.py:90-101)."""
    r = stream.uniform()
    if q_tok == 0.0:
        return False
    return r <= min(1.0, q_tok / p_tok)


def residual(p: np.ndarray, q: np.ndarray) -> np.ndarray:
    """Normalised positive part of q - p (speccore.py:104-113)."""
    diff = np.maximum(q - p, 0.0)
    z = float(diff.sum())
    if z <= 1e-12:
        raise ValueError("q <= p pointwise; residual has no mass")
    return diff / z


# --------------------------------------------------------------------------
# toylm.py:55-130, as a protocol object


class ToyLMPort:
    def __init__(self, n_layers: int, vocab: int, seed: int, misalignment: float = 0.0):
        self.n_layers, self.vocab = n_layers, vocab
        self.seed, self.misalignment = seed, float(misalignment)

    def empty_digest(self) -> int:
        return mix64(self.seed ^ SEQ_SALT)

    def extend_digest(self, d: int, tok: int) -> int:
        return mix64(d ^ ((TOKEN_SALT + tok) & M64))

    def advance_digest(self, d: int, a: int, b: int) -> int:
        for layer in range(a + 1, b + 1):
            d = mix64(d ^ ((layer * LAYER_SALT) & M64))
        return d

    def _unit(self, digest: int, salt: int) -> np.ndarray:
        ids = np.arange(self.vocab, dtype=np.uint64)
        with np.errstate(over="ignore"):
            keyed = (np.uint64(digest) ^ (ids * np.uint64(TOKEN_SALT | 1))) + np.uint64(salt)
        return (mix64_np(keyed) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def logits(self, final_digest: int) -> np.ndarray:
        return (self._unit(final_digest, LOGIT_SALT) - 0.5) * 8.0

    def exit_logits(self, final_digest: int, exit_digest: int) -> np.ndarray:
        z = self.logits(final_digest)
        if self.misalignment != 0.0:
            z = z + self.misalignment * (2.0 * self._unit(exit_digest, NOISE_SALT) - 1.0)
        return z

    @staticmethod
    def _softmax(z: np.ndarray) -> np.ndarray:
        w = np.exp(z - z.max())
        return w / w.sum()

    # protocol: digests wrapped as in the reference's PrefixState(.digest)
    def dist_from_final_state(self, state) -> np.ndarray:
        return self._softmax(self.logits(_dig(state)))

    def exit_dist_from_states(self, final, exit_state) -> np.ndarray:
        return self._softmax(self.exit_logits(_dig(final), _dig(exit_state)))


class _State:
    __slots__ = ("digest",)

    def __init__(self, digest):
        self.digest = digest


def _dig(s):
    return s.digest if hasattr(s, "digest") else s


def _probs(p) -> np.ndarray:
    return np.asarray(p.probs if hasattr(p, "probs") else p, dtype=np.float64)


# --------------------------------------------------------------------------
# pipesim.py:76-114


def stage_layers(n_layers: int, exit_depth: int) -> tuple[int, ...]:
    s = -(-n_layers // exit_depth)
    return (exit_depth,) * (s - 1) + (n_layers - (s - 1) * exit_depth,)


def make_metrics(committed, ticks, accepts, rejects, drafted, ar_ticks_per_token):
    """pipesim.py:256-275 — returns the RunMetrics field tuple."""
    assert committed == accepts + rejects
    thr = committed / ticks if ticks > 0 else 0.0
    alpha = (accepts / drafted) if drafted > 0 else None
    return (committed, ticks, accepts, rejects, alpha, thr, thr * ar_ticks_per_token)


# --------------------------------------------------------------------------
# pipesim.py:670-789 — the tick machine


class _Chain:
    __slots__ = ("pos", "layer", "digest", "token", "p")

    def __init__(self, pos, digest):
        self.pos, self.layer, self.digest = pos, 0, digest
        self.token = None
        self.p = None


def ppsd_machine(lm, n_layers, exit_depth, prompt, stop, *, exit_stage=None,
                 comm_latency=0, greedy=True, force_reject=False,
                 bernoulli_alpha=None, rng_seed=0, trace=True):
    """Returns (tokens, metrics_tuple, trace_rows). `lm` is None for the
    Bernoulli schedule-only oracle. trace rows are
    (tick, stage, kind, position, token_or_None, verdict)."""
    layers = stage_layers(n_layers, exit_depth)
    S = len(layers)
    k = exit_stage if exit_stage is not None else 1
    per = 1 + comm_latency
    rows = []
    rng = Stream(rng_seed)
    toy = lm is not None
    if toy:
        # _ToyVerifier streams (pipesim.py:339-344); greedy draws none
        s_draft, s_verify, s_commit = rng.split("draft"), rng.split("verify"), rng.split("commit")
        seq_tok = list(prompt)
        seq_dig = [lm.empty_digest()]
        for t in prompt:
            seq_dig.append(lm.extend_digest(seq_dig[-1], t))
        n_prompt = len(prompt)
    else:
        verify = rng.split("verify")

    def push(tok):
        seq_tok.append(tok)
        seq_dig.append(lm.extend_digest(seq_dig[-1], tok))

    cur = [None] * (S + 1)
    transit = []  # FIFO of (ready_tick, dest, chain)
    committed = accepts = rejects = 0
    draft_head, next_launch, t = 0, 1, 0

    def emit(ch, st, tick):
        if trace:
            rows.append((tick, st, ACTIVATION, ch.pos, None, ""))
        transit.append((tick + per, st + 1, ch))

    def draft(ch, st, tick):
        nonlocal next_launch
        if toy:
            fin = lm.advance_digest(ch.digest, ch.layer, n_layers)
            ch.p = _probs(lm.exit_dist_from_states(_State(fin), _State(ch.digest)))
            ch.token = first_argmax(ch.p) if greedy else sample_token(ch.p, s_draft)
            push(ch.token)
        if trace:
            rows.append((tick, st, DRAFT_TOKEN, ch.pos, ch.token, ""))
        next_launch = tick + (1 if st == 1 else per)

    while committed < stop:
        t += 1
        while transit and transit[0][0] == t:
            _, dest, ch = transit.pop(0)
            cur[dest] = ch
        rollback = corrected = None
        for st in range(S, 1, -1):
            ch, cur[st] = cur[st], None
            if ch is None:
                continue
            nl = layers[st - 1]
            if toy:
                ch.digest = lm.advance_digest(ch.digest, ch.layer, ch.layer + nl)
            ch.layer += nl
            if st == S:
                if ch.pos != committed + 1:
                    raise AssertionError("verdicts must land in position order")
                if toy:
                    q = _probs(lm.dist_from_final_state(_State(ch.digest)))
                    if greedy:
                        top_q = first_argmax(q)
                        if force_reject:
                            ok, tok = False, top_q
                        else:
                            ok = first_argmax(ch.p) == top_q
                            tok = ch.token if ok else top_q
                    elif force_reject:  # full_model_token (pipesim.py:360-365)
                        ok, tok = False, sample_token(q, s_commit)
                    elif accept_draft(ch.p[ch.token], q[ch.token], s_verify):  # pipesim.py:356-358
                        ok, tok = True, ch.token
                    else:
                        ok, tok = False, sample_token(residual(ch.p, q), s_commit)
                else:
                    ok = (not force_reject) and verify.uniform() < bernoulli_alpha
                    tok = None
                committed += 1
                if ok:
                    accepts += 1
                    if trace:
                        rows.append((t, S, FINAL_TOKEN, ch.pos, tok, "accept"))
                else:
                    rejects += 1
                    rollback, corrected = ch.pos, tok
                    if trace:
                        rows.append((t, S, CHECK_TOKEN, ch.pos, tok, "reject"))
            else:
                if st == k:
                    draft(ch, st, t)
                emit(ch, st, t)
        if next_launch is not None and t == next_launch:
            pos = draft_head + 1
            ch = _Chain(pos, seq_dig[n_prompt + pos - 1] if toy else None)
            if toy:
                ch.digest = lm.advance_digest(ch.digest, 0, layers[0])
            ch.layer = layers[0]
            draft_head = pos
            if k == 1:
                draft(ch, 1, t)
            else:
                next_launch = None
            emit(ch, 1, t)
        if rollback is not None:
            transit.clear()
            cur = [None] * (S + 1)
            draft_head = rollback
            if toy:
                idx = n_prompt + rollback - 1
                del seq_tok[idx:]
                del seq_dig[idx + 1:]
                push(corrected)
            next_launch = t + per
    tokens = seq_tok[n_prompt:n_prompt + committed] if toy else []
    m = make_metrics(committed, t, accepts, rejects, accepts + rejects, S * per)
    return tokens, m, rows


def decode_ppsd(lm, n_layers, exit_depth, prompt, max_tokens, **kw):
    """pipesim.py:595-633 (greedy): ([] , zero metrics, no rows) at max_tokens=0."""
    S = len(stage_layers(n_layers, exit_depth))
    per = 1 + kw.get("comm_latency", 0)
    if max_tokens == 0:
        return [], make_metrics(0, 0, 0, 0, 0, S * per), []
    return ppsd_machine(lm, n_layers, exit_depth, prompt, max_tokens, **kw)


def decode_autoregressive(lm, prompt, max_tokens, greedy=True, rng_seed=0):
    """pipesim.py:390-409."""
    commit = Stream(rng_seed).split("commit")
    seq = list(prompt)
    d = lm.empty_digest()
    digs = [d]
    for t in seq:
        digs.append(lm.extend_digest(digs[-1], t))
    out = []
    for _ in range(max_tokens):
        fin = lm.advance_digest(digs[-1], 0, lm.n_layers)
        q = _probs(lm.dist_from_final_state(_State(fin)))
        tok = first_argmax(q) if greedy else sample_token(q, commit)
        seq.append(tok)
        digs.append(lm.extend_digest(digs[-1], tok))
        out.append(tok)
    return out


def simulate_ppsd_bernoulli_fast(n_layers, exit_depth, alpha, horizon, rng_seed,
                                 exit_stage=None, comm_latency=0):
    """pipesim.py:636-667, the untraced O(1)-per-tick path."""
    S = len(stage_layers(n_layers, exit_depth))
    per = 1 + comm_latency
    k = exit_stage or 1
    age = (S - 1) * per
    gap = 1 if k == 1 else k * per
    verify = Stream(rng_seed).split("verify")
    pipe, committed, acc, rej, t, nxt = [], 0, 0, 0, 0, 1
    while committed < horizon:
        t += 1
        if t == nxt:
            pipe.append(t)
            nxt = t + gap
        if pipe and t - pipe[0] == age:
            pipe.pop(0)
            if verify.uniform() < alpha:
                acc += 1
            else:
                rej += 1
                pipe.clear()
                nxt = t + per
            committed += 1
    return make_metrics(committed, t, acc, rej, acc + rej, S * per)


# --------------------------------------------------------------------------
# pipesim.py:435-551 — EESD rounds, greedy toy oracle


def simulate_eesd(lm, n_layers, exit_depth, gamma, horizon, rng_seed, *,
                  exit_stage=None, comm_latency=0, bernoulli_alpha=None,
                  prompt=None, trace=True):
    layers = stage_layers(n_layers, exit_depth)
    S = len(layers)
    k = exit_stage or 1
    per = 1 + comm_latency
    dt = 1 if k == 1 else k * per
    round_ticks = gamma * dt + S * per
    exit_layer = k * exit_depth
    rows = []
    rng = Stream(rng_seed)
    toy = lm is not None
    if toy:
        if prompt is None:
            prompt = default_prompt(lm.vocab, rng_seed)
        seq = list(prompt)
        digs = [lm.empty_digest()]
        for tk in seq:
            digs.append(lm.extend_digest(digs[-1], tk))
        n_prompt = len(seq)
    else:
        verify = rng.split("verify")

    def push(tok):
        seq.append(tok)
        digs.append(lm.extend_digest(digs[-1], tok))

    committed = acc = rej = drafted = 0
    t = 0
    while committed < horizon:
        base = committed
        vt = t + gamma * dt + (S - 1) * per + 1
        drafts = []
        for h in range(1, gamma + 1):
            tok = None
            if toy:
                d0 = digs[len(seq)]
                fin = lm.advance_digest(d0, 0, n_layers)
                ex = lm.advance_digest(d0, 0, exit_layer)
                p = _probs(lm.exit_dist_from_states(_State(fin), _State(ex)))
                tok = first_argmax(p)
                push(tok)
                drafts.append((tok, p))
            if trace:
                rows.append((t + h * dt, k, DRAFT_TOKEN, base + h, tok, ""))
        if trace:
            for st in range(1, S):
                rows.append((t + gamma * dt + (st - 1) * per + 1, st, ACTIVATION, base + 1, None, ""))
        n_acc, corrected = 0, None
        for h in range(1, gamma + 1):
            if toy:
                tok, p = drafts[h - 1]
                fin = lm.advance_digest(digs[n_prompt + base + h - 1], 0, n_layers)
                top_q = first_argmax(_probs(lm.dist_from_final_state(_State(fin))))
                ok = first_argmax(p) == top_q
                ctok = tok if ok else top_q
            else:
                ok = verify.uniform() < bernoulli_alpha
                tok = ctok = None
            if ok:
                n_acc += 1
                if trace:
                    rows.append((vt, S, FINAL_TOKEN, base + h, tok, "accept"))
            else:
                corrected = ctok
                if trace:
                    rows.append((vt, S, CHECK_TOKEN, base + h, ctok, "reject"))
                break
        if n_acc == gamma:
            bonus = None
            if toy:
                fin = lm.advance_digest(digs[len(seq)], 0, n_layers)
                bonus = first_argmax(_probs(lm.dist_from_final_state(_State(fin))))
                push(bonus)
            if trace:
                rows.append((vt, S, FINAL_TOKEN, base + gamma + 1, bonus, ""))
        elif toy:
            idx = n_prompt + base + n_acc
            del seq[idx:]
            del digs[idx + 1:]
            push(corrected)
        drafted += gamma
        acc += n_acc
        rej += 1
        committed += n_acc + 1
        t += round_ticks
    m = make_metrics(committed, t, acc, rej, drafted, S * per)
    tokens = seq[n_prompt:] if toy else []
    return tokens, m, rows


def trace_csv(rows) -> str:
    """pipesim.py:175-189 format."""
    out = ["tick,stage,kind,position,token,verdict"]
    for tick, st, kind, pos, tok, verdict in rows:
        out.append(f"{tick},{st},{kind},{pos},{'' if tok is None else tok},{verdict}")
    return "\n".join(out) + "\n"
