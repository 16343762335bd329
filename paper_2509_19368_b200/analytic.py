"""Closed-form throughput laws the measured speedups are reported against.

Host-side report columns only (no kernel). Formulas follow
pkg/src/specpipe/analytic.py:72-206 (paper Eqs. 4-7).
"""

from __future__ import annotations

from dataclasses import dataclass


def _alpha(a: float) -> None:
    if not 0.0 <= a <= 1.0:
        raise ValueError(f"alpha must lie in [0, 1], got {a!r}")


def _depths(n: int, e: int) -> None:
    if n < 1:
        raise ValueError("n_layers must be >= 1")
    if not 1 <= e <= n:
        raise ValueError(f"exit_depth must lie in [1, n_layers], got {e} with N={n}")


def _gamma(g) -> None:
    if not isinstance(g, int) or isinstance(g, bool) or g < 1:
        raise ValueError(f"gamma must be an integer >= 1, got {g!r}")


@dataclass(frozen=True)
class SpeedupParams:
    alpha: float
    gamma: int
    n_layers: int
    exit_depth: int

    def __post_init__(self):
        _alpha(self.alpha)
        _gamma(self.gamma)
        _depths(self.n_layers, self.exit_depth)


def n_stages(n_layers: int, exit_depth: int) -> int:
    _depths(n_layers, exit_depth)
    return -(-n_layers // exit_depth)


def expected_accept_len(alpha: float, gamma: int) -> float:
    _alpha(alpha)
    _gamma(gamma)
    return float(gamma) if alpha == 1.0 else alpha * (1.0 - alpha ** gamma) / (1.0 - alpha)


def ppsd_speedup(alpha: float, n_layers: int, exit_depth: int) -> float:
    """Eq. 7: N / (alpha*E + (1-alpha)*ceil(N/E)*E)."""
    _alpha(alpha)
    s = n_stages(n_layers, exit_depth)
    return n_layers / (alpha * exit_depth + (1.0 - alpha) * s * exit_depth)


def ppsd_reference_speedup(alpha: float, n_layers: int, exit_depth: int, exit_stage: int) -> float:
    _alpha(alpha)
    s = n_stages(n_layers, exit_depth)
    if not 1 <= exit_stage <= s - 1:
        raise ValueError(f"exit_stage must lie in [1, {s - 1}], got {exit_stage}")
    return n_layers / (alpha * exit_stage * exit_depth + (1.0 - alpha) * s * exit_depth)


def eesd_speedup(params: SpeedupParams, cache_reuse: bool = False) -> float:
    """Eq. 5: (1-a^(g+1))/(1-a) * N / (g*E + N [- E])."""
    a, g, n, e = params.alpha, params.gamma, params.n_layers, params.exit_depth
    per_round = float(g + 1) if a == 1.0 else (1.0 - a ** (g + 1)) / (1.0 - a)
    return per_round * n / (g * e + n - (e if cache_reuse else 0))


def ppsd_over_eesd_lambda(params: SpeedupParams) -> float:
    a, g, n, e = params.alpha, params.gamma, params.n_layers, params.exit_depth
    if a == 1.0:
        return (g + n / e) / (g + 1.0)
    s = n_stages(n, e)
    return (1.0 - a) * (g * e + n) / ((a * e + (1.0 - a) * s * e) * (1.0 - a ** (g + 1)))



@dataclass(frozen=True)
class CostModel:
    """Wall-clock cost of one full-model forward and one draft forward
    (analytic.py:22-36); t_draft = 0 is the free-drafts limit."""

    t_target: float
    t_draft: float

    def __post_init__(self):
        if self.t_target <= 0.0:
            raise ValueError("t_target must be positive")
        if self.t_draft < 0.0:
            raise ValueError("t_draft must be non-negative")


def overall_acceptance(alpha: float, gamma: int) -> float:
    """expected_accept_len / gamma: accepted fraction of all drafted tokens."""
    return expected_accept_len(alpha, gamma) / gamma


def sd_gain(cost: CostModel, alpha: float, gamma: int) -> float:
    """t_target / (gamma*t_draft + t_target) * (expected_accept_len + 1)."""
    _alpha(alpha)
    _gamma(gamma)
    return cost.t_target / (gamma * cost.t_draft + cost.t_target) * (expected_accept_len(alpha, gamma) + 1.0)


def eesd_best_gamma(alpha: float, n_layers: int, exit_depth: int, gamma_max: int = 64) -> int:
    """Draft length in 1..gamma_max maximising eesd_speedup (first maximum)."""
    _alpha(alpha)
    best_g, best_v = 1, float("-inf")
    for g in range(1, gamma_max + 1):
        v = eesd_speedup(SpeedupParams(alpha, g, n_layers, exit_depth))
        if v > best_v:
            best_g, best_v = g, v
    return best_g
