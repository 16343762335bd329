"""The reference's decode entry points, executed by the B200 engine.

`decode_ppsd`, `decode_autoregressive`, `simulate_ppsd` keep the signatures,
argument checks, error types and return values of
pkg/src/specpipe/pipesim.py:390-409, 571-633; all compute goes through
libppsd.so (include/ppsd.h). Validation order mirrors the reference
(`_check_mode`, `_check_prompt`, depth, draft head) so errors surface the
same way.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from .models import ToyLM, TransformerLM
from .pipeline import (AcceptanceOracle, EventTrace, OracleMode, PipelineConfig, RunMetrics,
                       default_prompt, make_metrics)
from .rng import RngStream


def _check_mode(mode: str) -> None:
    if mode not in ("greedy", "sampling"):
        raise ValueError(f"mode must be 'greedy' or 'sampling', got {mode!r}")


def _check_prompt(lm, prompt) -> None:
    if len(prompt) == 0:
        raise ValueError("prompt must be non-empty")
    for t in prompt:
        if not 0 <= t < lm.vocab:
            raise ValueError(f"prompt token {t} outside vocab of {lm.vocab}")


def _require_draft_head(cfg: PipelineConfig) -> int:
    if cfg.exit_stage is None:
        raise ValueError("this schedule needs a draft head (at least 2 stages)")
    return cfg.exit_stage


class Engine:
    """One libppsd engine: a model (or the Bernoulli oracle) + a pipeline split."""

    def __init__(self, model_desc: _lib.ModelDesc, weights, cfg: PipelineConfig, device: int = 0,
                 stage_range: tuple[int, int] = (0, 0)):
        L = _lib.lib()
        self.cfg = cfg
        self.kind = model_desc.kind
        pd = _lib.PipelineDesc(n_layers=cfg.n_layers, exit_depth=cfg.exit_depth,
                               exit_stage=cfg.exit_stage or 0, comm_latency=cfg.comm_latency,
                               stage_lo=stage_range[0], stage_hi=stage_range[1], device=device)
        h = C.c_void_p()
        self._weights = weights  # keep pointer arrays alive
        _lib.check(L.ppsd_engine_create(C.byref(model_desc), C.byref(weights) if weights is not None
                                        else None, C.byref(pd), None, C.byref(h)), "engine_create")
        self.h = h
        self.max_ctx = model_desc.max_ctx
        self._vocab = model_desc.vocab
        self._d_model = model_desc.d_model
        self.last = None
        self._fin = weakref.finalize(self, L.ppsd_engine_destroy, h)

    def close(self):
        self._fin()

    def set_schedule(self, schedule: str) -> None:
        """'auto' | 'pipelined' | 'folded' (include/ppsd.h PPSD_SCHEDULE_*)."""
        if schedule not in _lib.SCHEDULES:
            raise ValueError(f"schedule must be one of {sorted(_lib.SCHEDULES)}, got {schedule!r}")
        _lib.check(_lib.lib().ppsd_set_schedule(self.h, _lib.SCHEDULES[schedule]), "set_schedule")

    def schedule(self, mode: str = "greedy") -> str:
        """The schedule a decode in `mode` runs on this engine."""
        out = C.c_int32()
        _lib.check(_lib.lib().ppsd_get_schedule(self.h, int(mode == "greedy"), C.byref(out)), "get_schedule")
        return {v: k for k, v in _lib.SCHEDULES.items()}[out.value]

    # -- helpers ---------------------------------------------------------
    def _trace_cap(self, stop: int) -> int:
        c = self.cfg
        return (stop * c.n_stages * c.hop_period + c.n_stages * c.hop_period + 8) * (c.n_stages + 2)

    def _finish(self, m: _lib.Metrics, rows: np.ndarray | None, n_rows: int):
        self.last = dict(decode_ms=m.decode_ms, prefill_ms=m.prefill_ms, gpu_launches=m.gpu_launches,
                         ticks=m.ticks, committed=m.committed_tokens,
                         schedule={v: k for k, v in _lib.SCHEDULES.items()}.get(m.schedule, "pipelined"),
                         deep_batches=m.deep_batches, deep_vectors=m.deep_vectors,
                         deep_pos_sum=m.deep_pos_sum, comb_heads=m.comb_heads)
        metrics = make_metrics(m.committed_tokens, m.ticks, m.accepts, m.rejects,
                               m.accepts + m.rejects, self.cfg.ar_ticks_per_token)
        trace = EventTrace.from_array(rows[:n_rows]) if rows is not None else EventTrace()
        return metrics, trace

    # -- entry points ----------------------------------------------------
    def decode(self, prompt, max_tokens: int, force_reject: bool = False, trace: bool = True,
               mode: str = "greedy", rng_seed: int = 0):
        L = _lib.lib()
        p = (C.c_int32 * len(prompt))(*[int(t) for t in prompt])
        out = np.zeros(max(1, max_tokens), dtype=np.int32)
        m = _lib.Metrics()
        rows = np.zeros((self._trace_cap(max_tokens), 6), dtype=np.int32) if trace else None
        n_rows = C.c_int64(0)
        greedy = int(mode == "greedy")
        _lib.check(L.ppsd_decode(self.h, greedy, rng_seed & ((1 << 64) - 1), p, len(prompt), max_tokens,
                                 int(bool(force_reject)),
                                 out.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(m),
                                 rows.ctypes.data_as(C.POINTER(_lib.TraceRowC)) if trace else None,
                                 rows.shape[0] if trace else 0, C.byref(n_rows)), "decode")
        metrics, tr = self._finish(m, rows, n_rows.value)
        return out[:max_tokens].tolist(), metrics, tr

    def decode_ar(self, prompt, max_tokens: int, mode: str = "greedy", rng_seed: int = 0):
        L = _lib.lib()
        p = (C.c_int32 * len(prompt))(*[int(t) for t in prompt])
        out = np.zeros(max(1, max_tokens), dtype=np.int32)
        m = _lib.Metrics()
        _lib.check(L.ppsd_decode_ar(self.h, int(mode == "greedy"), rng_seed & ((1 << 64) - 1), p, len(prompt),
                                    max_tokens,
                                    out.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(m)), "decode_ar")
        self.last = dict(decode_ms=m.decode_ms, prefill_ms=m.prefill_ms, gpu_launches=m.gpu_launches,
                         ticks=m.ticks, committed=m.committed_tokens)
        return out[:max_tokens].tolist()

    def simulate(self, alpha: float, verify_seed: int, horizon: int, force_reject=False, trace=True):
        L = _lib.lib()
        m = _lib.Metrics()
        rows = np.zeros((self._trace_cap(horizon), 6), dtype=np.int32) if trace else None
        n_rows = C.c_int64(0)
        _lib.check(L.ppsd_simulate(self.h, float(alpha), verify_seed & ((1 << 64) - 1), horizon,
                                   int(bool(force_reject)), C.byref(m),
                                   rows.ctypes.data_as(C.POINTER(_lib.TraceRowC)) if trace else None,
                                   rows.shape[0] if trace else 0, C.byref(n_rows)), "simulate")
        return self._finish(m, rows, n_rows.value)

    def _eesd_result(self, m: _lib.Metrics, rows, n_rows: int):
        self.last = dict(decode_ms=m.decode_ms, prefill_ms=m.prefill_ms, gpu_launches=m.gpu_launches,
                         ticks=m.ticks, committed=m.committed_tokens)
        thr = m.committed_tokens / m.ticks if m.ticks > 0 else 0.0
        metrics = RunMetrics(m.committed_tokens, m.ticks, m.accepts, m.rejects,
                             m.alpha_all_measured if m.alpha_valid else None, thr,
                             thr * self.cfg.ar_ticks_per_token)
        trace = EventTrace.from_array(rows[:n_rows]) if rows is not None else EventTrace()
        return metrics, trace

    def _eesd_rows(self, horizon: int, gamma: int):
        return np.zeros((horizon * (2 * gamma + self.cfg.n_stages + 1) + 8, 6), dtype=np.int32)

    def decode_eesd(self, prompt, horizon: int, gamma: int, trace: bool = True, mode: str = "greedy",
                    rng_seed: int = 0):
        L = _lib.lib()
        p = (C.c_int32 * len(prompt))(*[int(t) for t in prompt])
        cap_tok = horizon + gamma + 1
        out = np.zeros(cap_tok, dtype=np.int32)
        m = _lib.Metrics()
        rows = self._eesd_rows(horizon, gamma) if trace else None
        n_rows = C.c_int64(0)
        _lib.check(L.ppsd_decode_eesd_mode(self.h, gamma, int(mode == "greedy"), rng_seed & ((1 << 64) - 1), p,
                                           len(prompt), horizon, out.ctypes.data_as(C.POINTER(C.c_int32)), cap_tok,
                                           C.byref(m),
                                           rows.ctypes.data_as(C.POINTER(_lib.TraceRowC)) if trace else None,
                                           rows.shape[0] if trace else 0, C.byref(n_rows)), "decode_eesd")
        metrics, tr = self._eesd_result(m, rows, n_rows.value)
        return out[:metrics.committed_tokens].tolist(), metrics, tr

    def simulate_eesd(self, gamma: int, alpha: float, verify_seed: int, horizon: int, trace: bool = True):
        L = _lib.lib()
        m = _lib.Metrics()
        rows = self._eesd_rows(horizon, gamma) if trace else None
        n_rows = C.c_int64(0)
        _lib.check(L.ppsd_simulate_eesd(self.h, gamma, float(alpha), verify_seed & ((1 << 64) - 1), horizon,
                                        C.byref(m),
                                        rows.ctypes.data_as(C.POINTER(_lib.TraceRowC)) if trace else None,
                                        rows.shape[0] if trace else 0, C.byref(n_rows)), "simulate_eesd")
        return self._eesd_result(m, rows, n_rows.value)

    def read_logits(self, which: int) -> np.ndarray:
        V = self._vocab
        out = np.zeros(V, dtype=np.float32)
        _lib.check(_lib.lib().ppsd_read_logits(self.h, which, out.ctypes.data_as(C.POINTER(C.c_float))),
                   "read_logits")
        return out

    def debug_matvec(self, which: int, layer: int, x: np.ndarray, batched: bool) -> np.ndarray:
        """GEMV unit check: y = W x for the O (which=1) or down (which=3)
        projection of `layer`, x [nv][K] fp32 -> [nv][R] fp32, through the
        shipped kernel (parity tests)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        nv = x.shape[0]
        out = np.zeros((nv, self._d_model), dtype=np.float32)
        _lib.check(_lib.lib().ppsd_debug_matvec(self.h, which, layer, nv, int(batched),
                                                x.ctypes.data_as(C.POINTER(C.c_float)),
                                                out.ctypes.data_as(C.POINTER(C.c_float))), "debug_matvec")
        return out

    def set_logits_tap(self, tap=None) -> None:
        """Parity tests: while `tap` (a CUDA float32 tensor [P+1, 2, vocab]) is
        set, decode() leaves the exit (index 0) and final (index 1) logits row
        of the committed prefix at every generated position 1..P in it
        (include/ppsd.h ppsd_set_logits_tap). None clears it."""
        if tap is None:
            _lib.check(_lib.lib().ppsd_set_logits_tap(self.h, None, 0), "set_logits_tap")
            self._tap = None
            return
        if tap.dim() != 3 or tap.shape[1] != 2 or tap.shape[2] != self._vocab or not tap.is_contiguous():
            raise ValueError("tap must be a contiguous [P+1, 2, vocab] tensor")
        self._tap = tap  # keep alive while the engine holds the pointer
        _lib.check(_lib.lib().ppsd_set_logits_tap(self.h, C.c_void_p(tap.data_ptr()), tap.shape[0] - 1),
                   "set_logits_tap")

    def probe_attn(self, n_vec: int, ctx: int, reps: int = 20):
        ms, nbytes = C.c_double(), C.c_double()
        _lib.check(_lib.lib().ppsd_probe_attn(self.h, n_vec, ctx, reps, C.byref(ms), C.byref(nbytes)),
                   "probe_attn")
        return ms.value, nbytes.value

    def probe_gemv(self, which: int, n_groups: int, reps: int = 20):
        ms, nbytes = C.c_double(), C.c_double()
        _lib.check(_lib.lib().ppsd_probe_gemv(self.h, which, n_groups, reps, C.byref(ms), C.byref(nbytes)),
                   "probe")
        return ms.value, nbytes.value


# engines are cached per (model, pipeline split, device)
_ENGINES: dict = {}


def _cfg_key(cfg: PipelineConfig):
    return (cfg.n_layers, cfg.exit_depth, cfg.exit_stage, cfg.comm_latency)


def engine_for(lm, cfg: PipelineConfig) -> Engine:
    import torch

    if isinstance(lm, TransformerLM):
        cache = lm.__dict__.setdefault("_engines", {})
        key = _cfg_key(cfg)
        if key not in cache:
            cache[key] = Engine(lm.model_desc(), lm.weights_struct(), cfg, device=lm.device.index)
        cache[key].set_schedule(getattr(lm, "schedule", "auto"))
        return cache[key]
    if isinstance(lm, ToyLM):
        dev = _lib.require_cuda().index
        key = (lm, _cfg_key(cfg), dev)
        if key not in _ENGINES:
            _ENGINES[key] = Engine(lm.model_desc(max_ctx=4096), None, cfg, device=dev)
        return _ENGINES[key]
    raise TypeError(f"the B200 engine runs ToyLM or TransformerLM models, got {type(lm).__name__}")


def toy_alignment(lm: ToyLM, exit_depth: int, prefixes):
    """Per-prefix sum(min(p, q)) and argmax agreement of the ToyLM exit head
    at exit_depth, computed on the GPU (ppsd_toy_alignment)."""
    if not 1 <= exit_depth <= lm.n_layers:
        raise ValueError(f"exit_depth must lie in [1, {lm.n_layers}], got {exit_depth}")
    n, plen = len(prefixes), len(prefixes[0])
    cfg = PipelineConfig(lm.n_layers, max(1, lm.n_layers // 2)) if lm.n_layers >= 2 else None
    if cfg is None:
        raise NotImplementedError("single-layer models are not supported by the engine")
    eng = engine_for(lm, cfg)
    flat = np.ascontiguousarray(np.asarray(prefixes, dtype=np.int32).reshape(-1))
    minsum = np.zeros(n, dtype=np.float64)
    agree = np.zeros(n, dtype=np.int32)
    _lib.check(_lib.lib().ppsd_toy_alignment(eng.h, exit_depth, n, plen, flat.ctypes.data_as(C.POINTER(C.c_int32)),
                                             minsum.ctypes.data_as(C.POINTER(C.c_double)),
                                             agree.ctypes.data_as(C.POINTER(C.c_int32))), "toy_alignment")
    return minsum.tolist(), agree.tolist()


def _toy_ctx_for(lm: ToyLM, n_prompt: int, max_tokens: int, cfg: PipelineConfig) -> None:
    need = n_prompt + max_tokens + cfg.n_stages * cfg.hop_period + 2
    if need > 4096:
        raise ValueError("prompt + max_tokens exceeds the ToyLM engine context (4096)")


def decode_ppsd(lm, cfg: PipelineConfig, prompt: list[int], max_tokens: int, mode: str,
                rng: RngStream, *, force_reject: bool = False
                ) -> tuple[list[int], RunMetrics, EventTrace]:
    """Verify-while-draft decode on the GPU (pipesim.py:595-633)."""
    _check_mode(mode)
    _check_prompt(lm, prompt)
    if cfg.n_layers != lm.n_layers:
        raise ValueError(f"pipeline is {cfg.n_layers} layers deep but the model has {lm.n_layers}")
    _require_draft_head(cfg)
    if max_tokens == 0:
        return [], make_metrics(0, 0, 0, 0, 0, cfg.ar_ticks_per_token), EventTrace()
    if isinstance(lm, ToyLM):
        _toy_ctx_for(lm, len(prompt), max_tokens, cfg)
    return engine_for(lm, cfg).decode(prompt, max_tokens, force_reject, mode=mode, rng_seed=rng.seed)


def decode_autoregressive(lm, prompt: list[int], max_tokens: int, mode: str, rng: RngStream) -> list[int]:
    """Full-model decode on the GPU (pipesim.py:390-409); sampling draws one
    commit-stream uniform per token."""
    _check_mode(mode)
    _check_prompt(lm, prompt)
    if max_tokens == 0:
        return []
    n = lm.n_layers
    if n < 2:
        raise NotImplementedError("single-layer models are not supported by the engine")
    cfg = PipelineConfig(n, max(1, n // 2))
    if isinstance(lm, ToyLM):
        _toy_ctx_for(lm, len(prompt), max_tokens, cfg)
        return engine_for(lm, cfg).decode_ar(prompt, max_tokens, mode=mode, rng_seed=rng.seed)
    cached = getattr(lm, "_engines", None)
    eng = next(iter(cached.values())) if cached else engine_for(lm, cfg)  # reuse the KV pool
    return eng.decode_ar(prompt, max_tokens, mode=mode, rng_seed=rng.seed)


def simulate_ppsd(cfg: PipelineConfig, oracle: AcceptanceOracle, horizon: int, rng: RngStream, *,
                  trace: EventTrace | None = None) -> RunMetrics:
    """Pipelined schedule with a verdict oracle (pipesim.py:571-592), on the GPU tick machine."""
    if horizon < 1:
        raise ValueError("horizon must be >= 1")
    _require_draft_head(cfg)
    if oracle.mode is OracleMode.BERNOULLI:
        m, tr = _bernoulli_engine(cfg).simulate(oracle.alpha, rng.split("verify").seed, horizon,
                                                trace=trace is not None)
    else:
        lm = oracle.lm
        prompt = default_prompt(lm.vocab, rng)
        _, m, tr = engine_for(lm, cfg).decode(prompt, horizon, trace=trace is not None,
                                              mode="greedy" if oracle.greedy else "sampling", rng_seed=rng.seed)
    if trace is not None:
        trace._rows.extend(tr.rows())
    return m


def simulate_autoregressive(cfg: PipelineConfig, horizon: int, *, trace: EventTrace | None = None
                            ) -> RunMetrics:
    """Sequential baseline tick arithmetic (pipesim.py:372-387); host-side, no model."""
    from .pipeline import ACTIVATION, FINAL_TOKEN, StageMessage

    if horizon < 1:
        raise ValueError("horizon must be >= 1")
    s, per = cfg.n_stages, cfg.hop_period
    if trace is not None:
        for i in range(1, horizon + 1):
            start = 1 + (i - 1) * s * per
            for st in range(1, s):
                trace.add(start + (st - 1) * per, st, StageMessage(ACTIVATION, i))
            trace.add(start + (s - 1) * per, s, StageMessage(FINAL_TOKEN, i))
    ticks = 1 + (horizon - 1) * s * per + (s - 1) * per
    return make_metrics(horizon, ticks, 0, horizon, 0, cfg.ar_ticks_per_token)


def _bernoulli_engine(cfg: PipelineConfig) -> Engine:
    dev = _lib.require_cuda().index
    key = ("bernoulli", _cfg_key(cfg), dev)
    if key not in _ENGINES:
        _ENGINES[key] = Engine(_lib.ModelDesc(kind=_lib.MODEL_BERNOULLI, n_layers=cfg.n_layers), None, cfg,
                               device=dev)
    return _ENGINES[key]


def simulate_eesd(cfg: PipelineConfig, gamma: int, oracle: AcceptanceOracle, horizon: int, rng: RngStream, *,
                  trace: EventTrace | None = None) -> RunMetrics:
    """Draft-then-verify rounds (pipesim.py:435-551) on the GPU: gamma drafts
    through the exit layers, one batched verify, acceptance scan."""
    if horizon < 1:
        raise ValueError("horizon must be >= 1")
    if gamma < 1:
        raise ValueError("gamma must be >= 1")
    _require_draft_head(cfg)
    if oracle.mode is OracleMode.BERNOULLI:
        m, tr = _bernoulli_engine(cfg).simulate_eesd(gamma, oracle.alpha, rng.split("verify").seed, horizon,
                                                      trace=trace is not None)
    else:
        lm = oracle.lm
        prompt = default_prompt(lm.vocab, rng)
        _, m, tr = engine_for(lm, cfg).decode_eesd(prompt, horizon, gamma, trace=trace is not None,
                                                   mode="greedy" if oracle.greedy else "sampling",
                                                   rng_seed=rng.seed)
    if trace is not None:
        trace._rows.extend(tr.rows())
    return m


def decode_eesd(lm, cfg: PipelineConfig, prompt: list[int], horizon: int, gamma: int, mode: str = "greedy",
                rng: RngStream | None = None) -> tuple[list[int], RunMetrics, EventTrace]:
    """EESD with an explicit prompt, returning the committed tokens as well
    (the baseline next to decode_ppsd / decode_autoregressive in bench tools)."""
    _check_mode(mode)
    _check_prompt(lm, prompt)
    if cfg.n_layers != lm.n_layers:
        raise ValueError(f"pipeline is {cfg.n_layers} layers deep but the model has {lm.n_layers}")
    _require_draft_head(cfg)
    return engine_for(lm, cfg).decode_eesd(prompt, horizon, gamma, mode=mode,
                                           rng_seed=rng.seed if rng is not None else 0)
