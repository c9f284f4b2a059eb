"""Public lattice / construction / transform functions of the reference
(lattice.py:505-551, construct.py:146-206, transform.py:34-127) on the device.

Inputs and outputs are host numpy objects so these are drop-in replacements;
the computation (residues, nodes, alias masks, Bluestein DFT, gather and
averaging) runs in libsfft_b200.so.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .core import (FrequencyIndexSet, MultipleRank1Lattice, Rank1Lattice, SparseSpectrum,
                   as_frequency_rows)
from .device import dptr, get_device, hptr
from .mr1l import DeviceFreqs, build_scheme, lattice_tables, scheme_to_host
from .primes import MLConfig, candidate_primes

__all__ = [
    "lattice_nodes",
    "residues",
    "project",
    "is_reconstructing_single",
    "build_multiple_lattice",
    "build_multiple_lattice_with_retries",
    "LatticeSamples",
    "dft_1d",
    "invert_multiple",
]


def _z32(z: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(z, dtype=np.int64).astype(np.int32))


def lattice_nodes(lat: Rank1Lattice) -> np.ndarray:
    """All M nodes (j z mod M) / M as an (M, d) float64 array (lattice.py:505-508)."""
    dev = get_device()
    ms = np.array([lat.m], dtype=np.int64)
    zs = _z32(lat.z.reshape(1, -1))
    pts = dev.empty((lat.m, lat.dim), dev.torch.float64)
    dummy = np.zeros(1)
    dev.call("sfft_lattice_nodes", hptr(ms), hptr(zs), 1, lat.dim, 0, lat.dim, hptr(dummy), dptr(pts),
             ctx="lattice nodes")
    return dev.download(pts)


def residues(I, z, m: int) -> np.ndarray:
    """k . z mod M per frequency, in set order (lattice.py:520-529)."""
    m = int(m)
    if m < 1:
        raise ValueError("modulus M must be >= 1")
    z = np.atleast_1d(np.asarray(z, dtype=np.int64))
    rows = I.freqs if isinstance(I, FrequencyIndexSet) else as_frequency_rows(I)
    if rows.shape[1] != len(z):
        raise ValueError("dimension mismatch between frequencies and z")
    if m > 2**31 - 1:
        raise ValueError("modulus M must be <= 2**31 - 1")
    if not len(rows):
        return np.zeros(0, dtype=np.int64)
    dev = get_device()
    cand = DeviceFreqs.from_host(dev, rows)
    out = dev.empty((len(rows),), dev.torch.int64)
    ms = np.array([m], dtype=np.int64)
    zs = _z32(np.mod(z, m).reshape(1, -1))
    dev.call("sfft_residues", dptr(cand.data), cand.n, rows.shape[1], cand.kmax, hptr(ms), hptr(zs), 1,
             dptr(out), ctx="residues")
    return dev.download(out)


def project(I: FrequencyIndexSet, comps: Sequence[int]) -> FrequencyIndexSet:
    return I.project(comps)


def is_reconstructing_single(lat: Rank1Lattice, I: FrequencyIndexSet) -> bool:
    if lat.dim != I.dim:
        raise ValueError("dimension mismatch between lattice and frequency set")
    if len(I) <= 1:
        return True
    res = residues(I, lat.z, lat.m)
    return len(np.unique(res)) == len(I)


# ---------------------------------------------------------------------------
# construction (Algorithm 1)

def build_multiple_lattice(I: FrequencyIndexSet, cfg: MLConfig,
                           rng: np.random.Generator | None = None) -> MultipleRank1Lattice:
    """One randomized pass (construct.py:146-182).  The caller's generator
    ends in exactly the state the reference leaves it in: the vectors are
    pre-drawn for the batched device pass, then the generator is rewound and
    only the L vectors the early exit uses are redrawn."""
    if not len(I):
        raise ValueError("cannot build a sampling scheme for an empty set")
    if rng is None:
        rng = np.random.default_rng(cfg.rng_seed)
    dev = get_device()
    n = len(I)
    l_max = cfg.max_lattices(n)
    primes = candidate_primes(I, cfg.size_lower_bound(n), l_max)
    saved = rng.bit_generator.state
    ms = np.asarray(primes, dtype=np.int64)
    z = rng.integers(0, ms[:, None], size=(len(ms), I.dim), dtype=np.int64)
    cand = DeviceFreqs.from_host(dev, I.freqs)
    sch = _masks_for(dev, cand, primes, z)
    rng.bit_generator.state = saved
    rng.integers(0, ms[: sch.L, None], size=(sch.L, I.dim), dtype=np.int64)
    return scheme_to_host(dev, I.freqs, sch)


def _masks_for(dev, cand, primes, z):
    from . import _native
    from .mr1l import DeviceScheme
    torch = dev.torch
    ms = np.asarray(primes, dtype=np.int64)
    words = int(_native.query("sfft_alias_scratch_words", hptr(ms), len(ms)))
    scratch = dev.empty((max(words, 1),), torch.int32)
    masks = dev.empty((cand.n,), torch.int64)
    stats = dev.empty((2,), torch.int32)
    zh = _z32(z)
    dev.call("sfft_alias_masks", dptr(cand.data), cand.n, cand.ncomp, cand.kmax, hptr(ms), hptr(zh),
             len(ms), dptr(scratch), words, dptr(masks), dptr(stats), ctx="alias masks")
    st = dev.download(stats)
    L = int(st[0]) if int(st[1]) == 0 else len(ms)
    return DeviceScheme(list(primes), z, L, masks, 1, int(st[1]))


def build_multiple_lattice_with_retries(I: FrequencyIndexSet, cfg: MLConfig, b: int,
                                        seed_seq: np.random.SeedSequence | None = None):
    """Up to b attempts with child streams of ``seed_seq`` (construct.py:185-206)."""
    if b < 1:
        raise ValueError("retry cap b must be >= 1")
    if seed_seq is None:
        seed_seq = np.random.SeedSequence(cfg.rng_seed)
    if not len(I):
        raise ValueError("cannot build a sampling scheme for an empty set")
    dev = get_device()
    cand = DeviceFreqs.from_host(dev, I.freqs)
    sch = build_scheme(dev, cand, b, seed_seq, cfg=cfg, box_extent=I.expansion() if len(I) > 1 else 0)
    return scheme_to_host(dev, I.freqs, sch), sch.attempts


# ---------------------------------------------------------------------------
# one MR1L reconstruction step with a known candidate set (BASELINE config 1)

@dataclass
class StepReport:
    coeffs: np.ndarray        # (n,) complex; 0 where uncovered
    covered: np.ndarray       # (n,) bool
    kept: np.ndarray          # (n,) bool: |c| >= delta (and within the cap)
    lattice_sizes: list
    generating_vectors: np.ndarray
    attempts: int
    oracle_calls: int
    h2d_bytes: int = 0
    d2h_bytes: int = 0


def reconstruct_step(candidates, oracle, *, b: int = 10, seed_seq=None, delta: float = 0.0,
                     cap: int | None = None, anchor_tail=None, device=None, group=None,
                     shard: bool | None = None) -> StepReport:
    """Build the MR1L scheme for ``candidates``, sample ``oracle`` on it,
    invert and threshold: the composition build_multiple_lattice_with_retries
    -> oracle(lattice nodes) -> invert_multiple -> _select of the reference
    (construct.py:185-206, detect.py:290-299, transform.py:99-127,
    detect.py:197-212) as one device pipeline.  Under torch.distributed the
    step's lattices are sharded over the ranks of ``group`` (parallel.py)
    unless ``shard=False``; every rank returns the same report."""
    from .mr1l import prepare_step, run_step, speculate_scheme
    from .parallel import Shard, run_step_sharded
    sh = Shard(group)
    sharded = sh.active and shard is not False
    dev = device or get_device()
    torch = dev.torch
    if isinstance(candidates, torch.Tensor):
        host_rows = candidates.to(torch.int64) if candidates.dtype != torch.int64 else candidates
    else:
        host_rows = torch.from_numpy(np.ascontiguousarray(np.asarray(candidates, dtype=np.int64)))
    if host_rows.dim() != 2 or not host_rows.shape[0]:
        raise ValueError("candidates must be a nonempty (n, d) integer array")
    d_rows = DeviceFreqs.upload_rows(dev, host_rows)  # the largest input first: its DMA starts now
    n, t1 = (int(x) for x in host_rows.shape)
    d = oracle.dim
    tail = np.zeros(d - t1) if anchor_tail is None else np.asarray(anchor_tail, dtype=np.float64)
    fresh = not isinstance(seed_seq, np.random.SeedSequence)
    if fresh:
        seed_seq = np.random.SeedSequence(0 if seed_seq is None else seed_seq)
    h2d = n * t1 * 8
    if hasattr(oracle, "device_terms"):
        # the oracle's terms are inputs of the call too: copied every call
        # (asynchronously, behind the candidate rows)
        oracle._dev_cache.pop(dev.index, None)
        hf, cf = oracle.device_terms(dev)
        h2d += hf.numel() * 4 + cf.numel() * 8
    spec, early = [], {}

    def ahead():
        """While the rows are in flight: the first attempt's primes and draw
        (valid unless the set's spread exceeds lambda; lazy streams only) and
        the alias buffers.  The step preparation follows the alias kernel
        (build_scheme's ``prepare``), so the alias kernel runs as soon as the
        rows have arrived while the host prepares."""
        from . import _native
        g = speculate_scheme(n, t1, seed_seq, b)
        spec.append(g)
        ms = np.asarray(g.primes, dtype=np.int64)
        words = int(_native.query("sfft_alias_scratch_words", hptr(ms), len(ms)))
        early["bufs"] = (dev.empty((max(words, 1),), torch.int32), dev.empty((n,), torch.int64),
                         dev.empty((2,), torch.int32))
        early["cov_h"] = torch.empty((max(n, 8),), dtype=torch.uint8, pin_memory=True)
        early["cov_d"] = dev.empty((max(n, 8),), torch.uint8)

    def defer_extent():
        """Skip the read-back of the rows' extent before the alias kernel when
        the guessed lattices make the exact double-quotient residue path valid
        for ANY int32 component (t+1 * (2^31 - 1) * max M < 2^52); the extent
        then comes back with the alias stats and is checked there."""
        return bool(spec) and t1 * float(2**31 - 1) * float(max(spec[0].primes)) < 4503599627370496.0

    cand, lo, hi = DeviceFreqs.from_rows_tensor(dev, host_rows, before_sync=ahead if fresh else None,
                                                defer=defer_extent, d_rows=d_rows)
    guess = spec[0] if spec else None
    prepare = lambda ms, z: prepare_step(dev, oracle, cand, 1, ms, z, tails=[tail], d=d)  # noqa: E731
    if hi is None:  # deferred: alias with the guess, extent read back with the stats
        sch = build_scheme(dev, cand, b, seed_seq, box_extent=0, lazy_streams=fresh, guess=guess,
                           bufs=early.get("bufs"), also=lo, prepare=prepare)
        lo, hi, kmax = DeviceFreqs.extent_of(sch.extra.view(np.int32), t1, n)
        cand.kmax = kmax
        if not (sch.attempts == 1 and sch.z is guess.z and guess.primes[0] > int((hi - lo).max())):
            # the guess did not hold (spread >= lambda): the reference's construction
            sch = build_scheme(dev, cand, b, seed_seq, box_extent=int((hi - lo).max()), lazy_streams=fresh,
                               prepare=prepare)
    else:
        sch = build_scheme(dev, cand, b, seed_seq, box_extent=int((hi - lo).max()), lazy_streams=fresh,
                           prepare=prepare, guess=guess, bufs=early.get("bufs"))
    # the masks are final once the scheme is built: their copy to the host runs
    # on a side stream while the sampling kernel runs (enqueued after the
    # sampling launch, so the launch is not delayed by it)
    ready = torch.cuda.Event()
    ready.record(dev.stream)
    if sharded:
        res = run_step_sharded(dev, oracle, cand, sch, [tail], d, delta, n if cap is None else int(cap), sh,
                               prep=sch.prep, need_coef=True)
    else:
        res = run_step(dev, oracle, cand, sch, [tail], d, delta, n if cap is None else int(cap),
                       defer_cap=True, prep=sch.prep)
    cov_h, cov_d = early.get("cov_h"), early.get("cov_d")
    if cov_h is None:
        cov_h = torch.empty((max(n, 8),), dtype=torch.uint8, pin_memory=True)
        cov_d = dev.empty((max(n, 8),), torch.uint8)
    # the coverage flags (masks != 0) on the device and their n bytes back, on
    # a side stream while the sampling kernel runs
    side = dev.copy_stream()
    side.wait_event(ready)
    from . import _native
    _native.call("sfft_masks_covered", sch.masks.data_ptr(), n, cov_d.data_ptr(), side.cuda_stream,
                 ctx="coverage flags")
    _native.call("sfft_copy_async", cov_h.data_ptr(), cov_d.data_ptr(), n, side.cuda_stream,
                 ctx="coverage read-back")
    sch.masks.record_stream(side)
    cov_d.record_stream(side)
    res.finalize()  # cap applied (if binding) before the results are read
    coef, keep = dev.download_many(res.coef[0], res.keep[0])
    side.synchronize()
    covered = cov_h.numpy()[:n].view(bool)
    d2h = coef.nbytes + keep.nbytes + n
    coef = coef.view(np.complex128).reshape(n)  # views of fresh pinned buffers: no host copy
    return StepReport(coef, covered, keep.view(bool),
                      sch.primes[: sch.L], sch.z[: sch.L], sch.attempts, res.nodes, h2d, d2h)


# ---------------------------------------------------------------------------
# transforms

@dataclass(frozen=True)
class LatticeSamples:
    """Sample values of a signal at the M nodes of one rank-1 lattice (transform.py:34-47)."""

    lattice: Rank1Lattice
    values: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.values, dtype=np.complex128)
        if v.shape != (self.lattice.m,):
            raise ValueError(f"expected {self.lattice.m} sample values, got shape {v.shape}")
        object.__setattr__(self, "values", v)


def _c2(v: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.stack([v.real, v.imag], axis=-1))


def dft_1d(values, direction: str = "forward") -> np.ndarray:
    """Unnormalised forward DFT / 1/K-scaled inverse of any length K >= 1
    (transform.py:50-64) by the device Bluestein kernels."""
    v = np.asarray(values, dtype=np.complex128)
    if v.ndim != 1 or not len(v):
        raise ValueError("dft_1d expects a nonempty 1-D vector")
    if direction not in ("forward", "inverse"):
        raise ValueError("direction must be 'forward' or 'inverse'")
    dev = get_device()
    K = len(v)
    tabs = lattice_tables(dev, np.array([K], dtype=np.int64), None, ctx="dft_1d tables")
    buf = dev.zeros((1, tabs.P, 2), dev.torch.float64)
    with dev.torch.cuda.stream(dev.stream):
        buf[0, :K].copy_(dev.torch.from_numpy(_c2(v)))
    inv = direction == "inverse"
    if inv:
        dev.call("sfft_cscale", dptr(buf), K, 1.0, 1, ctx="dft_1d conj")
    dev.call("sfft_finish_samples", hptr(tabs.ms), 1, 1, dptr(tabs.chirp), dptr(buf), tabs.P, 0, 0, 0, 0, 0,
             ctx="dft_1d pre-chirp")
    dev.call("sfft_bluestein", hptr(tabs.ms), 1, 1, tabs.P, dptr(tabs.ftab), dptr(tabs.bhat),
             dptr(tabs.chirp), dptr(buf), 0, 0, ctx="dft_1d")
    if inv:
        dev.call("sfft_cscale", dptr(buf), K, 1.0 / K, 1, ctx="dft_1d scale")
    out = dev.download(buf[0, :K])
    return out[:, 0] + 1j * out[:, 1]


def invert_multiple(samples: Sequence[LatticeSamples], ml: MultipleRank1Lattice) -> SparseSpectrum:
    """Averaged inversion over the lattices of a scheme (transform.py:99-127)."""
    samples = list(samples)
    if len(samples) != len(ml.lattices):
        raise ValueError("need exactly one sample vector per lattice")
    for got, lat in zip(samples, ml.lattices):
        if got.lattice.m != lat.m or not np.array_equal(got.lattice.z, lat.z):
            raise ValueError("sample vectors are not aligned with the scheme's lattices")
    target = ml.target
    L = len(ml.lattices)
    if L > 64:
        raise ValueError("at most 64 lattices per scheme")
    dev = get_device()
    torch = dev.torch
    n = len(target)
    if n == 0:
        return SparseSpectrum(target.freqs, np.zeros(0, dtype=np.complex128), target.dim)
    words = np.zeros(n, dtype=np.uint64)
    for l, mk in enumerate(ml.recon_masks):
        words |= mk.astype(np.uint64) << np.uint64(l)
    ms = np.array([lat.m for lat in ml.lattices], dtype=np.int64)
    zs = _z32(np.stack([lat.z for lat in ml.lattices]))
    tabs = lattice_tables(dev, ms, zs, ctx="invert_multiple tables")
    buf = dev.zeros((L, tabs.P, 2), torch.float64)
    host = np.zeros((L, int(ms.max()), 2))
    for l, got in enumerate(samples):
        host[l, : got.lattice.m] = _c2(got.values)
    with torch.cuda.stream(dev.stream):
        buf[:, : host.shape[1]].copy_(torch.from_numpy(host))
    dev.call("sfft_finish_samples", hptr(ms), L, 1, dptr(tabs.chirp), dptr(buf), tabs.P, 0, 0, 0, 0, 0,
             ctx="invert_multiple pre-chirp")
    dev.call("sfft_bluestein", hptr(ms), L, 1, tabs.P, dptr(tabs.ftab), dptr(tabs.bhat), dptr(tabs.chirp),
             dptr(buf), 0, 0, ctx="invert_multiple FFT")
    cand = DeviceFreqs.from_host(dev, target.freqs)
    d_masks = dev.upload(words.view(np.int64))
    coef = dev.empty((1, n, 2), torch.float64)
    keep = dev.empty((1, n), torch.uint8)
    counts = dev.zeros((1,), torch.int32)
    dev.call("sfft_gather_select", dptr(cand.data), n, target.dim, cand.kmax, hptr(ms), hptr(zs), L,
             dptr(d_masks), dptr(buf), tabs.P, 1, 0, 0.0, dptr(coef), dptr(keep), dptr(counts),
             ctx="invert_multiple gather")
    c = dev.download(coef[0])
    covered = words != 0
    vals = c[:, 0] + 1j * c[:, 1]
    return SparseSpectrum(target.freqs[covered], vals[covered], target.dim)
