"""Seeds and counter streams with the reference's exact bit semantics.

Host-side: the decode path only needs these to derive seeds (model seeds,
`default_prompt`, the Bernoulli verify stream) — the per-draw stream math
also lives on the device (`csrc/hostdev.h:counter_uniform`).
Follows pkg/src/specpipe/rng.py:29-99.
"""

from __future__ import annotations

_MASK = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
_M1, _M2 = 0xBF58476D1CE4E5B9, 0x94D049BB133111EB
_LABEL = 0xA24BAED4963EE407


def mix64(x: int) -> int:
    """splitmix64 finalizer (rng.py:29-37)."""
    x &= _MASK
    x = ((x ^ (x >> 30)) * _M1) & _MASK
    x = ((x ^ (x >> 27)) * _M2) & _MASK
    return x ^ (x >> 31)


def derive_seed(seed: int, label) -> int:
    """Child seed of (seed, label); string labels fold byte-wise (rng.py:51-63)."""
    h = mix64(seed ^ _LABEL)
    if isinstance(label, str):
        for b in label.encode("utf-8"):
            h = mix64(h ^ (b + 1))
    else:
        h = mix64(h ^ mix64(label & _MASK))
    return h


class RngStream:
    """Counter stream: draw c is splitmix64(seed + (c+1)*gamma) >> 11 / 2^53."""

    __slots__ = ("seed", "counter")

    def __init__(self, seed: int, counter: int = 0):
        if counter < 0:
            raise ValueError("counter must be non-negative")
        self.seed = seed & _MASK
        self.counter = counter

    def uniform(self) -> float:
        self.counter += 1
        return (mix64(self.seed + self.counter * _GAMMA) >> 11) * 2.0 ** -53

    def randbelow(self, n: int) -> int:
        if n < 1:
            raise ValueError("n must be positive")
        return min(int(self.uniform() * n), n - 1)

    def split(self, label) -> "RngStream":
        return RngStream(derive_seed(self.seed, label))

    def __repr__(self) -> str:
        return f"RngStream(seed={self.seed:#018x}, counter={self.counter})"
