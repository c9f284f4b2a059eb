"""Lattice-size selection for the randomized MR1L construction (host side).

Restates reference construct.py:50-136: the L_max smallest primes above
lambda = c (|I| - 1) that keep the target set distinct componentwise mod p,
and the MLConfig formulas for L_max and lambda.  These are O(L_max) scalar
computations per step; the data-parallel part of the construction (alias
histograms over all candidates) runs in the CUDA library (K3, csrc/alias.cu,
driven by mr1l.build_scheme).
"""

from __future__ import annotations

import math
from functools import lru_cache
from dataclasses import dataclass

import numpy as np

__all__ = ["MLConfig", "candidate_primes", "primes_above"]


class _Sieve:
    """Grow-only table of primes (Eratosthenes on a bool array)."""

    def __init__(self):
        self.limit = 0
        self.primes = np.empty(0, dtype=np.int64)

    def cover(self, limit: int) -> None:
        if limit <= self.limit:
            return
        limit = max(limit, 2 * self.limit, 1024)
        flags = np.ones(limit + 1, dtype=bool)
        flags[:2] = False
        flags[4::2] = False
        for p in range(3, math.isqrt(limit) + 1, 2):
            if flags[p]:
                flags[p * p::2 * p] = False
        self.primes = np.flatnonzero(flags).astype(np.int64)
        self.limit = limit


_SIEVE = _Sieve()


def primes_above(bound: float, count: int) -> list[int]:
    """The ``count`` smallest primes strictly greater than ``bound``."""
    return list(_primes_above(max(int(math.floor(bound)), 0), int(count)))


@lru_cache(maxsize=1024)
def _primes_above(start: int, count: int) -> tuple:
    return tuple(_primes_above_list(start, count))


def _primes_above_list(start: int, count: int) -> list[int]:
    out: list[int] = []
    while True:
        _SIEVE.cover(max(2 * (start + 1), 2 * start + 64))
        pos = int(np.searchsorted(_SIEVE.primes, start, side="right"))
        avail = _SIEVE.primes[pos:pos + count - len(out)]
        out.extend(int(p) for p in avail)
        if len(out) >= count:
            return out
        start = _SIEVE.limit
        _SIEVE.cover(2 * _SIEVE.limit)


def _distinct_mod(freqs: np.ndarray, p: int) -> bool:
    reduced = np.mod(freqs, p)
    return len(np.unique(reduced, axis=0)) == len(freqs)


def candidate_primes(I, lam: float, count: int, *, spread: int | None = None, rows=None) -> list[int]:
    """``count`` smallest primes p > lam such that the rows of I stay distinct
    mod p (automatic once p exceeds the expansion of I; reference
    construct.py:85-102).

    ``I`` may be a FrequencyIndexSet, or None together with ``spread`` (the
    set's expansion, or an upper bound of it) and a ``rows`` callable that
    materialises the (n, d) rows on the host only when a prime p <= spread
    actually needs the explicit check.
    """
    if count < 1:
        raise ValueError("count must be >= 1")
    if I is not None:
        if not len(I):
            raise ValueError("candidate primes need a nonempty frequency set")
        spread = I.expansion() if len(I) > 1 else 0
        rows = (lambda: I.freqs)
    out: list[int] = []
    host_rows = None
    want = count
    while True:
        for p in primes_above(lam, want):
            if p in out:
                continue
            if p > spread:
                ok = True
            else:
                if host_rows is None:
                    host_rows = rows()
                ok = _distinct_mod(host_rows, p)
            if ok:
                out.append(p)
                if len(out) == count:
                    return out
        want *= 2


@dataclass(frozen=True)
class MLConfig:
    """Oversampling factor c > 1 and failure bound gamma in (0, 1) of the
    randomized multi-lattice search (reference construct.py:108-136)."""

    c: float = 2.0
    gamma: float = 0.5
    rng_seed: int = 0

    def __post_init__(self):
        if not self.c > 1.0:
            raise ValueError("oversampling factor c must be > 1")
        if not 0.0 < self.gamma < 1.0:
            raise ValueError("gamma must lie in (0, 1)")

    def max_lattices(self, set_size: int) -> int:
        if set_size < 1:
            raise ValueError("set_size must be >= 1")
        factor = self.c ** 2 / (self.c - 1.0) ** 2
        return math.ceil(factor * (math.log(set_size) - math.log(self.gamma)) / 2.0)

    def size_lower_bound(self, set_size: int) -> float:
        return self.c * (set_size - 1)
