"""Seeded synthetic inputs of the five BASELINE.json configurations.

Seeds follow the reference CLI's protocol (cli.py:254-262):
SeedSequence([seed, config, trial]).spawn(3) -> (truth, detection, noise),
with the detection seed collapsed to one uint64 (cli.py:254-255).  No public
dataset is involved; every input is generated here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import SearchBox, SparseSpectrum
from .engine import DetectionConfig
from .oracles import (BSplineOracle, RelativeNoisyOracle, SparsePolynomialOracle,
                      gen_random_sparse_poly)

__all__ = ["Workload", "StepWorkload", "config0", "config1", "config2", "config3", "config4",
           "seeds_for", "distinct_rows"]


def seeds_for(seed: int, config: int, trial: int = 0):
    truth, detect, noise = np.random.SeedSequence([seed, config, trial]).spawn(3)
    return truth, int(detect.generate_state(1, np.uint64)[0]), noise


def distinct_rows(rng: np.random.Generator, n: int, dims: int, N: int) -> np.ndarray:
    """n distinct rows uniform on [-N, N]^dims (batched rejection, draw order kept)."""
    seen: set = set()
    rows = []
    while len(rows) < n:
        block = rng.integers(-N, N + 1, size=(max(n, 64), dims))
        for row in map(tuple, block.tolist()):
            if row not in seen:
                seen.add(row)
                rows.append(row)
                if len(rows) == n:
                    break
    return np.asarray(rows, dtype=np.int64)


@dataclass
class Workload:
    name: str
    oracle: object
    cfg: DetectionConfig
    truth: SparseSpectrum | None


@dataclass
class StepWorkload:
    """BASELINE config 1: one MR1L step with a known candidate set."""

    name: str
    cand: np.ndarray            # (|J|, d) int64, lexicographically sorted
    oracle: SparsePolynomialOracle
    truth_coef: np.ndarray      # length |J| complex (zeros off the support)
    b: int
    lattice_seed: int
    delta: float


def config0(seed: int = 0, trial: int = 0, d: int = 5, N: int = 16, s: int = 100, r: int = 2) -> Workload:
    ts, rs, _ = seeds_for(seed, 0, trial)
    truth, oracle = gen_random_sparse_poly(d, N, s, "box", seed=ts, min_magnitude=1e-3)
    cfg = DetectionConfig(box=SearchBox.centered(d, N), delta=1e-12, s=s, r=r, b=10, rng_seed=rs)
    return Workload("config0 d=5 N=16 s=100 r=2", oracle, cfg, truth)


def config1(seed: int = 0, n: int = 100_000, d: int = 10, N: int = 32, nnz: int = 2000) -> StepWorkload:
    ts, rs, _ = seeds_for(seed, 1)
    rng = np.random.default_rng(ts)
    rows = distinct_rows(rng, n, d, N)
    rows = rows[np.lexsort(rows.T[::-1])]
    support = np.sort(rng.choice(n, size=nnz, replace=False))
    coef = np.zeros(n, dtype=np.complex128)
    coef[support] = rng.uniform(-1, 1, nnz) + 1j * rng.uniform(-1, 1, nnz)
    oracle = SparsePolynomialOracle(rows[support], coef[support], d)
    return StepWorkload(f"config1 MR1L step |J|={n} d={d} nnz={nnz}", rows, oracle, coef, 10, rs, 1e-12)


def config2(seed: int = 0, trial: int = 0, r: int = 5) -> Workload:
    ts, rs, _ = seeds_for(seed, 2, trial)
    truth, oracle = gen_random_sparse_poly(10, 32, 1000, "box", seed=ts, min_magnitude=1e-3)
    cfg = DetectionConfig(box=SearchBox.centered(10, 32), delta=1e-12, s=1000, r=r, b=10, rng_seed=rs)
    return Workload(f"config2 d=10 N=32 s=1000 r={r}", oracle, cfg, truth)


def config3(seed: int = 0, trial: int = 0, d: int = 20, s: int = 10_000, r: int = 5,
            device_rng: bool = False) -> Workload:
    """``device_rng``: GPU-generated noise (same distribution, not the numpy
    realisation); the default draws the reference-compatible numpy stream."""
    ts, rs, ns = seeds_for(seed, 3, trial)
    truth, poly = gen_random_sparse_poly(d, 32, s, "polar", seed=ts)
    oracle = RelativeNoisyOracle(poly, 1e-2, seed=ns, device_rng=device_rng)
    box = SearchBox.centered(d, 32, check_cardinality=False)
    cfg = DetectionConfig(box=box, delta=1e-1, s=s, r=r, b=10, rng_seed=rs)
    return Workload(f"config3 d={d} N=32 s={s} r={r} noisy 1e-2", oracle, cfg, truth)


def bspline_partition(seed_seq) -> tuple:
    perm = np.random.default_rng(seed_seq).permutation(10)
    return ((2, tuple(sorted(int(c) for c in perm[:3]))),
            (4, tuple(sorted(int(c) for c in perm[3:7]))),
            (6, tuple(sorted(int(c) for c in perm[7:]))))


def config4(seed: int = 0, trial: int = 0, N: int = 64, s: int = 2000, r: int = 5) -> Workload:
    ts, rs, _ = seeds_for(seed, 4, trial)
    oracle = BSplineOracle(bspline_partition(ts), 10)
    box = SearchBox.centered(10, N, check_cardinality=False)
    cfg = DetectionConfig(box=box, delta=1e-6, s=s, r=r, b=10, rng_seed=rs)
    return Workload(f"config4 B-spline d=10 N={N} s={s} r={r}", oracle, cfg, None)
