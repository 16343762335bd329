"""Host-side mirror of the reference's decode-path types.

Names, fields, validation and error types follow
pkg/src/specpipe/pipesim.py (PipelineConfig :60-114, StageMessage :122-142,
TraceRow/EventTrace :145-189, AcceptanceOracle :192-232, RunMetrics
:235-275, default_prompt :290-294), so code written against the reference
keeps working. The schedule itself runs on the GPU (csrc/sched.h).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from enum import Enum
from typing import Iterator, NamedTuple

from .rng import RngStream

PROMPT_LEN = 8
ACTIVATION = "ACTIVATION"
DRAFT_TOKEN = "DRAFT_TOKEN"
FINAL_TOKEN = "FINAL_TOKEN"
CHECK_TOKEN = "CHECK_TOKEN"
KINDS = (ACTIVATION, DRAFT_TOKEN, FINAL_TOKEN, CHECK_TOKEN)  # index = PPSD_* kind code
VERDICTS = ("", "accept", "reject")
TRACE_HEADER = "tick,stage,kind,position,token,verdict"


@dataclass(frozen=True)
class PipelineConfig:
    """ceil(N/E) stages of E layers (remainder last); draft head at exit_stage."""

    n_layers: int
    exit_depth: int
    exit_stage: int | None = None
    comm_latency: int = 0
    n_stages: int = field(init=False)
    stage_layers: tuple[int, ...] = field(init=False)

    def __post_init__(self):
        n, e = self.n_layers, self.exit_depth
        if n < 1:
            raise ValueError("n_layers must be >= 1")
        if not 1 <= e <= n:
            raise ValueError(f"exit_depth must lie in [1, n_layers], got {e} with n_layers={n}")
        if self.comm_latency < 0:
            raise ValueError("comm_latency must be non-negative")
        s = -(-n // e)
        object.__setattr__(self, "n_stages", s)
        object.__setattr__(self, "stage_layers", tuple([e] * (s - 1) + [n - (s - 1) * e]))
        k = self.exit_stage
        if k is None:
            object.__setattr__(self, "exit_stage", 1 if s >= 2 else None)
        elif s < 2:
            raise ValueError("a draft head needs at least 2 stages")
        elif not 1 <= k <= s - 1:
            raise ValueError(f"exit_stage must lie in [1, {s - 1}], got {k}")

    @property
    def exit_layer(self) -> int:
        if self.exit_stage is None:
            raise ValueError("single-stage pipeline has no draft head")
        return self.exit_stage * self.exit_depth

    @property
    def hop_period(self) -> int:
        return 1 + self.comm_latency

    @property
    def ar_ticks_per_token(self) -> int:
        return self.n_stages * self.hop_period


def partition_stages(n_layers: int, exit_depth: int) -> tuple[int, ...]:
    return PipelineConfig(n_layers, exit_depth).stage_layers


@dataclass(frozen=True)
class StageMessage:
    kind: str
    position: int
    token: int | None = None
    payload: object | None = None

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown message kind {self.kind!r}")
        if self.position < 1:
            raise ValueError("position must be >= 1")
        if self.payload is not None and self.kind != ACTIVATION:
            raise ValueError("only ACTIVATION messages carry a state payload")


class TraceRow(NamedTuple):
    tick: int
    stage: int
    kind: str
    position: int
    token: int | None
    verdict: str


class EventTrace:
    """Chronological message log; rows come back from the device trace ring."""

    __slots__ = ("_list", "_arr")

    def __init__(self, rows=None):
        self._list: list[TraceRow] = list(rows or [])
        self._arr = None

    @classmethod
    def from_array(cls, arr) -> "EventTrace":
        """arr: int32 [n, 6] of (tick, stage, kind, position, token|-1, verdict),
        the rows the device trace ring returned; the TraceRow objects are built
        on first use (a 512-token decode returns ~4k rows: ~4 ms of Python the
        decode call itself does not need to pay)."""
        tr = cls()
        tr._arr = arr
        return tr

    @property
    def _rows(self) -> list[TraceRow]:
        if self._arr is not None:
            self._list = [TraceRow(int(t), int(s), KINDS[k], int(p), None if tok < 0 else int(tok), VERDICTS[v])
                          for t, s, k, p, tok, v in self._arr.tolist()] + self._list
            self._arr = None
        return self._list

    def add(self, tick: int, stage: int, message: StageMessage, verdict: str = "") -> None:
        self._rows.append(TraceRow(tick, stage, message.kind, message.position, message.token, verdict))

    @property
    def records(self):
        return [(r.tick, r.stage, StageMessage(r.kind, r.position, r.token), r.verdict) for r in self._rows]

    def rows(self) -> Iterator[TraceRow]:
        return iter(self._rows)

    __iter__ = rows

    def __len__(self) -> int:
        return len(self._list) + (0 if self._arr is None else len(self._arr))

    def write_csv(self, dest) -> None:
        if hasattr(dest, "write"):
            dest.write(self.to_csv())
        else:
            with open(dest, "w", newline="") as fh:
                fh.write(self.to_csv())

    def to_csv(self) -> str:
        lines = [TRACE_HEADER]
        for r in self._rows:
            lines.append(f"{r.tick},{r.stage},{r.kind},{r.position},{'' if r.token is None else r.token},{r.verdict}")
        return "\n".join(lines) + "\n"


class OracleMode(str, Enum):
    BERNOULLI = "bernoulli"
    TOYLM_SAMPLING = "toylm-sampling"
    TOYLM_GREEDY = "toylm-greedy"


@dataclass(frozen=True)
class AcceptanceOracle:
    mode: OracleMode
    alpha: float | None = None
    lm: object | None = None

    def __post_init__(self):
        if self.mode is OracleMode.BERNOULLI:
            if self.alpha is None or not 0.0 <= self.alpha <= 1.0:
                raise ValueError("BERNOULLI oracle needs alpha in [0, 1]")
            if self.lm is not None:
                raise ValueError("BERNOULLI oracle does not take a model")
        else:
            if self.lm is None:
                raise ValueError(f"{self.mode.value} oracle needs a ToyLM")
            if self.alpha is not None:
                raise ValueError("toy-LM oracles measure alpha, do not set it")

    @classmethod
    def bernoulli(cls, alpha: float) -> "AcceptanceOracle":
        return cls(OracleMode.BERNOULLI, alpha=alpha)

    @classmethod
    def toylm_sampling(cls, lm) -> "AcceptanceOracle":
        return cls(OracleMode.TOYLM_SAMPLING, lm=lm)

    @classmethod
    def toylm_greedy(cls, lm) -> "AcceptanceOracle":
        return cls(OracleMode.TOYLM_GREEDY, lm=lm)

    @property
    def greedy(self) -> bool:
        return self.mode is OracleMode.TOYLM_GREEDY


@dataclass(frozen=True)
class RunMetrics:
    committed_tokens: int
    ticks: int
    accepts: int
    rejects: int
    alpha_all_measured: float | None
    throughput: float
    speedup_vs_ar: float


def make_metrics(committed, ticks, accepts, rejects, drafted, ar_ticks_per_token) -> RunMetrics:
    """The RunMetrics arithmetic of pipesim.py:256-275."""
    if committed != accepts + rejects:
        raise AssertionError("commit accounting out of balance")
    thr = committed / ticks if ticks > 0 else 0.0
    return RunMetrics(committed, ticks, accepts, rejects,
                      (accepts / drafted) if drafted > 0 else None, thr, thr * ar_ticks_per_token)


def steady_state_view(metrics: RunMetrics, cfg: PipelineConfig) -> RunMetrics:
    ticks = max(1, metrics.ticks - cfg.n_stages * cfg.hop_period)
    thr = metrics.committed_tokens / ticks
    return replace(metrics, ticks=ticks, throughput=thr, speedup_vs_ar=thr * cfg.ar_ticks_per_token)


def default_prompt(vocab: int, rng: RngStream) -> list[int]:
    stream = rng.split("prompt")
    return [stream.randbelow(vocab) for _ in range(PROMPT_LEN)]
