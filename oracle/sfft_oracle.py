"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain-numpy restatement of the reference's MR1L path (arXiv 1711.05152
package `sfft`, /root/reference/pkg/src/sfft), used as the parity checker by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg.  Nothing in the product package imports this module.

Pinned: tests/test_oracle_golden.py checks every function here against
golden vectors produced by the unmodified reference (tests/golden/
make_golden.py, run in the build container where /root/reference exists).

Third-party arithmetic: the reference's DFT is scipy.fft (ducc0/pocketfft,
scipy 1.18.1 here); this restatement uses numpy.fft (pocketfft C), both
pinned by the same known-answer vectors.  numpy RNG (PCG64 / SeedSequence)
is the reference's own dependency and is used identically.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# residues / nodes (reference lattice.py:505-517)


def residues(freqs: np.ndarray, z: np.ndarray, m: int) -> np.ndarray:
    """k . z mod M with componentwise reduction (lattice.py:511-517)."""
    zm = np.asarray(z, dtype=np.int64) % m
    acc = np.zeros(len(freqs), dtype=np.int64)
    for t in range(freqs.shape[1]):
        acc = (acc + (freqs[:, t] % m) * zm[t]) % m
    return acc


def lattice_nodes(z: np.ndarray, m: int) -> np.ndarray:
    """(j z mod M) / M, j = 0..M-1 (lattice.py:505-508)."""
    j = np.arange(m, dtype=np.int64)
    return (j[:, None] * (np.asarray(z, dtype=np.int64) % m)[None, :] % m) / m


def alias_free_mask(freqs: np.ndarray, z: np.ndarray, m: int) -> np.ndarray:
    """counts[res] == 1 (construct.py:139-143)."""
    res = residues(freqs, z, m)
    return np.bincount(res, minlength=m)[res] == 1


# ---------------------------------------------------------------------------
# primes and Algorithm 1 (construct.py:50-206)


def primes_above(bound: float, count: int) -> list[int]:
    start = max(int(math.floor(bound)), 0)
    hi = max(2 * start + 64, 1024)
    while True:
        sieve = np.ones(hi + 1, dtype=bool)
        sieve[:2] = False
        for p in range(2, math.isqrt(hi) + 1):
            if sieve[p]:
                sieve[p * p::p] = False
        ps = np.flatnonzero(sieve)
        ps = ps[ps > start]
        if len(ps) >= count:
            return [int(p) for p in ps[:count]]
        hi *= 2


def candidate_primes(freqs: np.ndarray, lam: float, count: int) -> list[int]:
    """construct.py:85-102: primes > lam keeping rows distinct mod p."""
    spread = int((freqs.max(axis=0) - freqs.min(axis=0)).max()) if len(freqs) > 1 else 0
    out: list[int] = []
    want = count
    while True:
        for p in primes_above(lam, want):
            if p in out:
                continue
            if p > spread or len(np.unique(freqs % p, axis=0)) == len(freqs):
                out.append(p)
                if len(out) == count:
                    return out
        want *= 2


def max_lattices(n: int, c: float = 2.0, gamma: float = 0.5) -> int:
    """construct.py:127-131."""
    return math.ceil(c * c / (c - 1.0) ** 2 * (math.log(n) - math.log(gamma)) / 2.0)


@dataclass
class Scheme:
    ms: list[int]
    zs: list[np.ndarray]
    masks: list[np.ndarray]
    attempts: int = 1

    @property
    def covered(self) -> np.ndarray:
        return np.logical_or.reduce(self.masks)

    @property
    def total_size(self) -> int:
        return int(sum(self.ms))


def build_multiple_lattice(freqs: np.ndarray, rng: np.random.Generator) -> Scheme:
    """One randomized pass with early exit (construct.py:146-182), c=2, gamma=0.5."""
    n, d = freqs.shape
    primes = candidate_primes(freqs, 2.0 * (n - 1), max_lattices(n))
    ms, zs, masks = [], [], []
    covered = np.zeros(n, dtype=bool)
    for m in primes:
        z = rng.integers(0, m, size=d, dtype=np.int64)
        mk = alias_free_mask(freqs, z, m)
        ms.append(m)
        zs.append(z)
        masks.append(mk)
        covered |= mk
        if covered.all():
            break
    return Scheme(ms, zs, masks)


def build_with_retries(freqs: np.ndarray, b: int, seed_seq: np.random.SeedSequence) -> Scheme:
    """construct.py:185-206."""
    sch = None
    for attempt, child in enumerate(seed_seq.spawn(b), start=1):
        sch = build_multiple_lattice(freqs, np.random.default_rng(child))
        sch.attempts = attempt
        if sch.covered.all():
            return sch
    return sch


# ---------------------------------------------------------------------------
# single lattice, component by component (construct.py:212-278)


def cbc(freqs: np.ndarray) -> tuple[np.ndarray, int]:
    """Smallest odd M >= |I| and smallest z_t per component separating all
    distinct prefixes (construct.py:254-278); freqs lexicographically sorted."""
    n, d = freqs.shape
    if n == 1:
        return np.zeros(d, dtype=np.int64), 1
    m = n if n % 2 == 1 else n + 1
    while True:
        z = np.zeros(d, dtype=np.int64)
        z[0] = 1 % m
        ok = True
        if d == 1:
            ok = len(np.unique(freqs[:, 0] % m)) == n
        for t in range(1, d):
            rows = np.unique(freqs[:, :t + 1], axis=0)
            pres = residues(rows[:, :t], z[:t], m)
            col = rows[:, t] % m
            found = None
            for start in range(0, m, 4096):
                cand = np.arange(start, min(start + 4096, m), dtype=np.int64)
                res = np.sort((pres[:, None] + col[:, None] * cand[None, :]) % m, axis=0)
                good = np.flatnonzero(np.all(res[1:] != res[:-1], axis=0))
                if len(good):
                    found = int(cand[good[0]])
                    break
            if found is None:
                ok = False
                break
            z[t] = found
        if ok:
            return z, m
        m += 2


def invert_single(freqs: np.ndarray, z: np.ndarray, m: int, values: np.ndarray) -> np.ndarray:
    """transform.py:83-96: X[k.z mod M] / M for every k."""
    return (np.fft.fft(values) / m)[residues(freqs, z, m)]


# ---------------------------------------------------------------------------
# inversion (transform.py:99-127) and selection (detect.py:197-212)


def invert_multiple(freqs: np.ndarray, sch: Scheme, values: list[np.ndarray]):
    """Averaged inversion; returns (covered mask, coefficients of covered rows)."""
    n = len(freqs)
    sums = np.zeros(n, dtype=np.complex128)
    counts = np.zeros(n, dtype=np.int64)
    for v, m, z, mk in zip(values, sch.ms, sch.zs, sch.masks):
        if not mk.any():
            continue
        spec = np.fft.fft(v) / m
        sums[mk] += spec[residues(freqs[mk], z, m)]
        counts[mk] += 1
    cov = counts > 0
    return cov, sums[cov] / counts[cov]


def select(freqs: np.ndarray, coeffs: np.ndarray, cap: int, delta: float):
    """|c| >= delta, then up to cap by (|c| desc, lexicographic freq asc)."""
    mags = np.abs(coeffs)
    keep = mags >= delta
    freqs, coeffs, mags = freqs[keep], coeffs[keep], mags[keep]
    if len(freqs) > cap:
        keys = tuple(freqs[:, c] for c in range(freqs.shape[1] - 1, -1, -1)) + (-mags,)
        order = np.lexsort(keys)[:cap]
        freqs, coeffs = freqs[order], coeffs[order]
    return freqs, coeffs


def lexsort_rows(rows: np.ndarray) -> np.ndarray:
    if len(rows) <= 1:
        return rows
    return rows[np.lexsort(rows.T[::-1])]


def unique_rows(rows: np.ndarray) -> np.ndarray:
    rows = lexsort_rows(rows)
    if len(rows) <= 1:
        return rows
    keep = np.ones(len(rows), dtype=bool)
    keep[1:] = np.any(rows[1:] != rows[:-1], axis=1)
    return rows[keep]


# ---------------------------------------------------------------------------
# signals (testbed.py:116-182, 198-244)


def poly_eval(freqs: np.ndarray, coeffs: np.ndarray, points: np.ndarray, chunk_budget: int = 1 << 21,
              threads: int = 1) -> np.ndarray:
    """p(x) = sum_h c_h exp(2 pi i h.x) in phase-matrix chunks (testbed.py:116-127)."""
    ft = freqs.T.astype(np.float64)
    out = np.empty(len(points), dtype=np.complex128)
    chunk = max(1, chunk_budget // max(len(coeffs), 1))

    def work(i):
        ph = points[i:i + chunk] @ ft
        out[i:i + chunk] = np.exp(2j * np.pi * ph) @ coeffs

    starts = range(0, len(points), chunk)
    if threads > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(work, starts))
    else:
        for i in starts:
            work(i)
    return out


def gen_sparse_poly(dims: int, N: int, s: int, seed, coeff_model: str = "box", floor: float = 1e-6):
    """Draw sequence of testbed.py:130-182 (frequencies by batched rejection)."""
    rng = np.random.default_rng(seed)
    chosen, seen = [], set()
    while len(chosen) < s:
        batch = rng.integers(-N, N + 1, size=(max(s, 64), dims))
        for row in map(tuple, batch.tolist()):
            if row not in seen:
                seen.add(row)
                chosen.append(row)
                if len(chosen) == s:
                    break
    freqs = np.asarray(chosen, dtype=np.int64)
    if coeff_model == "box":
        c = rng.uniform(-1, 1, s) + 1j * rng.uniform(-1, 1, s)
        small = np.abs(c) < floor
        while small.any():
            k = int(small.sum())
            c[small] = rng.uniform(-1, 1, k) + 1j * rng.uniform(-1, 1, k)
            small = np.abs(c) < floor
    elif coeff_model == "unit_modulus":
        c = np.exp(2j * np.pi * rng.random(s))
    else:
        raise ValueError(coeff_model)
    order = np.lexsort(freqs.T[::-1])
    return freqs[order], c[order]


def bspline_constant(m: int) -> float:
    """testbed.py:198-212."""
    k = np.arange(1, 200_001)
    return float(1.0 / np.sqrt(1.0 + 2.0 * np.sum(np.sinc(k / m) ** (2 * m))))


def cardinal_bspline(m: int, u: np.ndarray) -> np.ndarray:
    """Order-m cardinal B-spline on knots 0..m, Cox-de Boor (the function
    scipy BSpline.basis_element(arange(m+1)) evaluates, testbed.py:214-229)."""
    u = np.asarray(u, dtype=np.float64)
    iv = np.clip(np.floor(u).astype(np.int64), 0, m - 1)
    N = [(iv == j).astype(np.float64) for j in range(m)]
    for k in range(2, m + 1):
        N = [((u - j) * N[j] + ((j + k) - u) * N[j + 1]) / (k - 1) for j in range(m - k + 1)]
    out = N[0]
    return np.where((u >= 0) & (u <= m), out, 0.0)


def bspline_eval(groups, points: np.ndarray) -> np.ndarray:
    """testbed.py:232-244."""
    total = np.zeros(len(points), dtype=np.complex128)
    for m, comps in groups:
        term = np.ones(len(points))
        for t in comps:
            term = term * (bspline_constant(m) * m * cardinal_bspline(m, m * np.mod(points[:, t], 1.0)))
        total += term
    return total


# ---------------------------------------------------------------------------
# the engine (detect.py:175-423)


def line_coefficients(fn, t: int, lows, highs, anchor: np.ndarray):
    """detect.py:175-194."""
    K = int(highs[t] - lows[t] + 1)
    pts = np.tile(np.asarray(anchor, dtype=np.float64), (K, 1))
    pts[:, t] = np.arange(K) / K
    bins = np.fft.fft(fn(pts)) / K
    ks = np.arange(lows[t], highs[t] + 1, dtype=np.int64)
    return ks, bins[ks % K]


@dataclass
class Report:
    freqs: np.ndarray
    coeffs: np.ndarray
    candidate_counts: list = field(default_factory=list)
    prefix_counts: list = field(default_factory=list)
    component_counts: list = field(default_factory=list)
    scheme_sizes: list = field(default_factory=list)
    attempts: list = field(default_factory=list)
    oracle_calls: int = 0
    wall_time: float = 0.0
    schemes: list = field(default_factory=list)


def sparse_fft(fn, lows, highs, delta: float, s: int, r: int = 1, b: int = 1, rng_seed: int = 0,
               s_local: int | None = None, zero_anchor: bool = False, component_delta: float | None = None,
               single: bool = False):
    """Algorithm 3 with the reference's RNG-stream contract (detect.py:305-423)."""
    t0 = time.perf_counter()
    lows = np.asarray(lows, dtype=np.int64)
    highs = np.asarray(highs, dtype=np.int64)
    d = len(lows)
    s_loc = s if s_local is None else s_local
    cdelta = delta if component_delta is None else component_delta
    root = np.random.SeedSequence(rng_seed)
    det_p, anc_p, lat_p = root.spawn(3)
    det_s, anc_s, lat_s = det_p.spawn(d), anc_p.spawn(d), lat_p.spawn(d)
    rep = Report(np.empty((0, d), np.int64), np.empty(0, np.complex128))
    for name in ("candidate_counts", "prefix_counts", "component_counts", "scheme_sizes", "attempts"):
        setattr(rep, name, [0] * d)
    calls = 0
    prefixes = None
    for t in range(d):
        rng = np.random.default_rng(det_s[t])
        found = []
        for _ in range(r):
            anchor = np.zeros(d) if zero_anchor else rng.random(d)
            ks, cf = line_coefficients(fn, t, lows, highs, anchor)
            calls += len(ks)
            kept, _ = select(ks[:, None], cf, s_loc, cdelta)
            found.append(kept[:, 0])
        comp = np.unique(np.concatenate(found))
        rep.component_counts[t] = len(comp)
        if t == 0:
            prefixes = comp[:, None]
            rep.candidate_counts[0] = rep.prefix_counts[0] = len(comp)
            if d > 1:
                continue
            cand = prefixes
        else:
            left = np.repeat(prefixes, len(comp), axis=0)
            right = np.tile(comp, len(prefixes))
            cand = unique_rows(np.column_stack([left, right]).astype(np.int64))
            rep.candidate_counts[t] = len(cand)
        last = t == d - 1
        rt = 1 if last else r
        st = s if last else s_loc
        if not len(cand):
            prefixes = cand
            continue
        if single:
            zc, mc = cbc(cand)
            sch = Scheme([mc], [zc], [np.ones(len(cand), dtype=bool)])
        else:
            sch = build_with_retries(cand, b, lat_s[t])
        rep.schemes.append(sch)
        rep.scheme_sizes[t] = sch.total_size
        rep.attempts[t] = sch.attempts
        arng = np.random.default_rng(anc_s[t])
        kept_f, kept_c = [], []
        for _ in range(rt):
            tail = np.zeros(d - t - 1) if zero_anchor else arng.random(d - t - 1)
            vals = []
            for m, z in zip(sch.ms, sch.zs):
                pts = np.empty((m, d))
                pts[:, :t + 1] = lattice_nodes(z, m)
                pts[:, t + 1:] = tail
                vals.append(fn(pts))
                calls += m
            cov, coefs = invert_multiple(cand, sch, vals)
            f, c = select(cand[cov], coefs, st, delta)
            kept_f.append(f)
            kept_c.append(c)
        if last:
            order = np.lexsort(kept_f[0].T[::-1]) if len(kept_f[0]) > 1 else np.arange(len(kept_f[0]))
            rep.freqs, rep.coeffs = kept_f[0][order], kept_c[0][order]
            rep.prefix_counts[t] = len(rep.freqs)
        else:
            prefixes = unique_rows(np.concatenate(kept_f))
            rep.prefix_counts[t] = len(prefixes)
    rep.oracle_calls = calls
    rep.wall_time = time.perf_counter() - t0
    return rep


def mr1l_step(cand: np.ndarray, fn, b: int, seed_seq, delta: float, cap: int, d: int | None = None):
    """One MR1L reconstruction step with known candidate set (BASELINE config 1):
    construction, sampling (no anchor tail), averaged inversion, selection."""
    sch = build_with_retries(cand, b, seed_seq)
    vals = [fn(lattice_nodes(z, m)) for m, z in zip(sch.ms, sch.zs)]
    cov, coefs = invert_multiple(cand, sch, vals)
    return sch, cov, coefs, select(cand[cov], coefs, cap, delta)
