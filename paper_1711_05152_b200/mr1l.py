"""The multiple-rank-1-lattice (MR1L) reconstruction step on the device.

One step, for a candidate set J (sorted, on the device) and r~ anchors:

  construction  K3  alias histograms of all L_max pre-drawn lattices of an
                     attempt, masks, first-covering L        (construct.py:146-206)
  sampling      K1  the oracle at every node of every (iteration, lattice)
                     unit, written pre-chirped                (detect.py:280-299)
  FFT           K2  batched Bluestein DFT of each unit        (transform.py:121)
  gather        K4  alias-free bins, lattice average, delta threshold, cap
                                                              (transform.py:99-127,
                                                               detect.py:197-212)

The host replays the reference's RNG consumption exactly (primes, generating
vectors, anchors), so schemes are identical to the reference's on the same
seeds; the host only ever synchronises to read a handful of counters.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .core import FrequencyIndexSet, MultipleRank1Lattice, Rank1Lattice
from .device import Device, dptr, hptr
from .oracles import BSplineOracle, NoisyOracle, SparsePolynomialOracle
from .primes import MLConfig, candidate_primes

__all__ = ["DeviceFreqs", "DeviceScheme", "build_scheme", "clear_caches", "speculate_scheme", "SchemeGuess", "run_step",
           "prepare_step", "StepPrep", "StepResult", "first_attempt_rng", "compact_start", "compact_finish",
           "compact_count", "PendingScheme",
           "OracleInterrupt", "OracleError", "evaluate_callback"]

UMAX = 256      # (iteration, lattice) units per launch (plan.cuh SFFT_UMAX)
RBMAX = 8       # iterations per gather launch


class OracleInterrupt(Exception):
    """Deliberate abort signalled by an oracle; propagates unwrapped
    (reference detect.py:55-61)."""


class OracleError(RuntimeError):
    pass


def evaluate_callback(oracle, points: np.ndarray, step: int, iteration: int) -> np.ndarray:
    """Host-callback evaluation with the reference's error contract (detect.py:157-172)."""
    try:
        values = oracle(points)
    except OracleInterrupt:
        raise
    except Exception as exc:
        raise OracleError(f"oracle evaluation failed at step {step}, iteration {iteration}: {exc}") from exc
    values = np.asarray(values, dtype=np.complex128)
    if values.shape != (len(points),):
        raise OracleError(
            f"oracle returned shape {values.shape} for {len(points)} points "
            f"at step {step}, iteration {iteration}"
        )
    return values


@dataclass
class DeviceFreqs:
    """A lexicographically sorted candidate set on the device, component-major int32."""

    data: object          # torch int32 tensor (ncomp, n)
    n: int
    kmax: int             # bound on |k_c|

    @property
    def ncomp(self) -> int:
        return int(self.data.shape[0])

    @classmethod
    def from_host(cls, dev: Device, rows: np.ndarray) -> "DeviceFreqs":
        rows = np.asarray(rows, dtype=np.int64)
        kmax = int(np.abs(rows).max()) if rows.size else 0
        t = dev.upload(np.ascontiguousarray(rows.T.astype(np.int32)))
        return cls(t, rows.shape[0], kmax)

    @staticmethod
    def upload_rows(dev: Device, rows):
        """Start the copy of (n, d) int64 host rows (a CPU tensor) to the
        device on the engine stream (asynchronous DMA when pinned); the
        result goes to ``from_rows_tensor(d_rows=...)``."""
        torch = dev.torch
        n, d = (int(x) for x in rows.shape)
        if rows.is_pinned() and rows.is_contiguous() and rows.dtype == torch.int64:
            # one cudaMemcpyAsync of the library on the engine stream (asynchronous DMA)
            d_rows = torch.empty((n, d), dtype=torch.int64, device=dev.device)
            if n * d:
                _native.call("sfft_copy_async", d_rows.data_ptr(), rows.data_ptr(), n * d * 8, dev.sh,
                             ctx="row upload")
            return d_rows
        with torch.cuda.stream(dev.stream):
            return rows.to(dev.device, non_blocking=bool(rows.is_pinned()))

    @classmethod
    def from_rows_tensor(cls, dev: Device, rows, before_sync=None,
                         defer: bool = False, d_rows=None) -> tuple["DeviceFreqs", object, object]:
        """Upload (n, d) int64 rows (a CPU tensor; pinned memory makes the copy
        asynchronous DMA) and pack them on the device; also returns the
        per-component minima and maxima.  ``before_sync()`` runs while the
        copy is in flight.  ``d_rows``: the copy already started by
        ``upload_rows``.  ``defer``: no read-back; returns (set with kmax =
        the int32 bound, the device extent tensor, None) and the caller reads
        the extent later with ``extent_of`` (one synchronisation fewer)."""
        torch = dev.torch
        n, d = (int(x) for x in rows.shape)
        if d_rows is None:  # (a caller may have started the copy earlier: upload_rows)
            d_rows = cls.upload_rows(dev, rows)
        out = dev.empty((d, n), torch.int32)
        mm = dev.empty((2 * d + 1,), torch.int32)
        dev.call("sfft_pack_rows", dptr(d_rows), n, d, dptr(out), dptr(mm), ctx="pack rows")
        if before_sync is not None:
            before_sync()
        if defer() if callable(defer) else defer:
            return cls(out, n, 2**31 - 1), mm, None
        lo, hi, kmax = cls.extent_of(dev.download_small(mm), d, n)
        return cls(out, n, kmax), lo, hi

    @staticmethod
    def extent_of(mmh, d: int, n: int):
        """(minima, maxima, kmax) from sfft_pack_rows' extent words."""
        mmh = np.asarray(mmh).astype(np.int64)
        if mmh[2 * d]:
            raise ValueError("frequency components must satisfy |k_t| <= 2147483647")
        lo, hi = mmh[:d], mmh[d:2 * d]
        kmax = int(max(np.abs(lo).max(), np.abs(hi).max())) if n else 0
        return lo, hi, kmax

    def to_host(self, dev: Device) -> np.ndarray:
        return dev.download(self.data).T.astype(np.int64)


@dataclass
class DeviceScheme:
    primes: list[int]           # the L_max candidate primes
    z: np.ndarray               # (L_max, t1) int64 generating vectors of the chosen attempt
    L: int                      # lattices used (early exit) or L_max
    masks: object               # torch int64 (n,) alias-free bit masks (bit l = lattice l)
    attempts: int
    uncovered: int
    prep: object = None         # build_scheme(prepare=...) result
    extra: object = None        # build_scheme(also=...) read back with the first attempt's stats

    @property
    def m_used(self) -> np.ndarray:
        return np.asarray(self.primes[: self.L], dtype=np.int64)

    @property
    def z_used(self) -> np.ndarray:
        return np.ascontiguousarray(self.z[: self.L].astype(np.int32))

    @property
    def total_size(self) -> int:
        return int(sum(self.primes[: self.L]))


def _spread_bound(cand: DeviceFreqs, box_extent: int | None) -> int:
    if box_extent is not None:
        return int(box_extent)
    return 2 * cand.kmax


def _attempt_streams(seed_seq: np.random.SeedSequence, b: int, lazy: bool):
    """The b child streams of construct.py:202 (``seed_seq.spawn(b)``).

    ``lazy``: build each child only when its attempt runs (identical streams;
    ~10x cheaper, since one attempt is the norm) without advancing
    ``seed_seq``'s spawn counter — for parents that are never spawned again
    (the engine's per-step lattice streams, fresh per-call seeds)."""
    if not lazy:
        yield from seed_seq.spawn(b)
        return
    base = seed_seq.n_children_spawned
    for i in range(b):
        yield np.random.SeedSequence(seed_seq.entropy, spawn_key=seed_seq.spawn_key + (base + i,),
                                     pool_size=seed_seq.pool_size)


def first_attempt_rng(seed_seq: np.random.SeedSequence, b: int) -> np.random.Generator:
    """The generator of attempt 1 of ``build_scheme(..., lazy_streams=True)``
    (the first lazy child of ``seed_seq``), made ahead of time by a caller
    that has idle host time (``build_scheme(first_rng=...)``)."""
    return np.random.default_rng(next(_attempt_streams(seed_seq, b, True)))


# candidate primes by (n, L_max, lambda) when every prime exceeds the spread
# (the rows are then not needed): steps of equal |J_t| repeat them
_PRIMES_MEMO: dict = {}


@dataclass
class SchemeGuess:
    """The first attempt of ``build_scheme`` computed before the candidate
    set's spread is known (``speculate_scheme``): valid whenever every
    candidate prime exceeds the spread, i.e. the primes are simply the L_max
    smallest primes above lambda (construct.py:85-102)."""
    primes: list
    z: np.ndarray


def speculate_scheme(n: int, t1: int, seed_seq: np.random.SeedSequence, b: int,
                     cfg: MLConfig | None = None) -> SchemeGuess:
    """Primes and the first attempt's generating vectors for an n-row set,
    drawn from the same (lazy) child stream build_scheme would use."""
    from .primes import primes_above
    cfg = cfg or MLConfig(c=2.0, gamma=0.5)
    l_max = cfg.max_lattices(n)
    primes = primes_above(cfg.size_lower_bound(n), l_max)
    ms = np.asarray(primes, dtype=np.int64)
    child = next(_attempt_streams(seed_seq, b, True))
    z = np.random.default_rng(child).integers(0, ms[:, None], size=(l_max, t1), dtype=np.int64)
    return SchemeGuess(primes, z)


def first_chunk(n: int, ms, target: float = 0.05) -> int:
    key = (int(n), tuple(int(m) for m in ms), float(target))
    got = _FIRST_CHUNK.get(key)
    if got is None:
        if len(_FIRST_CHUNK) > 1024:
            _FIRST_CHUNK.clear()
        got = _FIRST_CHUNK[key] = _first_chunk(*key)
    return got


_FIRST_CHUNK: dict = {}


def _first_chunk(n: int, ms, target: float = 0.05) -> int:
    """Primes of an attempt whose alias masks are evaluated before the first
    coverage check: the fewest for which the expected number of candidates
    not yet alias-free on any of them, n * prod_l (1 - (1 - 1/M_l)^(n-1))
    (residues of distinct frequencies collide with probability 1/M_l for a
    uniform generating vector), falls below ``target``; all of them when
    that leaves at most one over.  The reference checks coverage after every
    prime (construct.py:173-181); evaluating a chunk and then the rest
    gives the same early-exit L and masks for the used lattices."""
    ms = [int(m) for m in ms]
    if n <= 1:
        return len(ms)
    log_unc = math.log(n)
    for L, m in enumerate(ms, start=1):
        free = math.exp((n - 1) * math.log1p(-1.0 / m)) if m > 1 else 0.0
        log_unc += math.log1p(-free) if free < 1.0 else -math.inf
        if log_unc < math.log(target):
            return L if L < len(ms) - 1 else len(ms)
    return len(ms)


def build_scheme(dev: Device, cand: DeviceFreqs, b: int, seed_seq: np.random.SeedSequence,
                 *, cfg: MLConfig | None = None, box_extent: int | None = None,
                 ctx: str = "", lazy_streams: bool = False, prepare=None,
                 guess: SchemeGuess | None = None, first_rng: np.random.Generator | None = None,
                 bufs: tuple | None = None, also=None, defer: bool = False):
    """Algorithm 1 with retries (reference construct.py:146-206) on the device.

    Every attempt pre-draws its L_max generating vectors (stream-identical to
    the reference's sequential draw, SURVEY §7 hard part 1) and evaluates the
    alias masks of a first chunk of them (``first_chunk``) in one pass, the
    rest only when that chunk leaves candidates uncovered; the early-exit L
    is the largest first-cover index over the candidates.  ``prepare(ms, z)``:
    called with the first chunk's primes once the first attempt's alias
    kernel is enqueued (host work that overlaps it); its result is returned
    as ``DeviceScheme.prep``.  ``guess``: the first attempt
    precomputed by ``speculate_scheme`` (used when its primes all exceed the
    spread; requires ``lazy_streams``).  ``bufs``: (scratch, masks, stats)
    allocated by the caller (used when large enough).  ``defer``: return a
    ``PendingScheme`` right after the first attempt's alias kernel is
    enqueued (when it comes from ``guess`` and neither ``prepare`` nor
    ``also`` is given; otherwise the search runs now); ``.finish()`` gives
    the DeviceScheme.
    """
    if b < 1:
        raise ValueError("retry cap b must be >= 1")
    n = cand.n
    if n < 1:
        raise ValueError("cannot build a sampling scheme for an empty set")
    cfg = cfg or MLConfig(c=2.0, gamma=0.5)
    l_max = cfg.max_lattices(n)
    if l_max > 64:
        raise ValueError(f"L_max = {l_max} lattices exceeds the 64-bit mask width")
    t1 = cand.ncomp
    spread = _spread_bound(cand, box_extent)
    if guess is not None and (not lazy_streams or len(guess.primes) != l_max or guess.primes[0] <= spread):
        guess = None
    lam = cfg.size_lower_bound(n)
    memo = _PRIMES_MEMO.get((n, l_max, lam))
    if guess is not None:
        primes = list(guess.primes)
    elif memo is not None and memo[0][0] > spread:
        primes = memo[0]
    else:
        primes = candidate_primes(None, lam, l_max, spread=spread, rows=lambda: cand.to_host(dev))
    ms = np.asarray(primes, dtype=np.int64)
    torch = dev.torch
    l_hi = first_chunk(n, ms)
    if memo is None and primes[0] > spread:
        if len(_PRIMES_MEMO) > 256:
            _PRIMES_MEMO.clear()
        _PRIMES_MEMO[(n, l_max, lam)] = (list(primes),)
    words = int(_native.query("sfft_alias_scratch_words", hptr(ms), l_max))
    if bufs is not None and bufs[0].numel() >= words and bufs[1].numel() == n:
        scratch, masks, stats = bufs  # allocated by the caller ahead of time
    else:
        scratch = dev.empty((max(words, 1),), torch.int32)
        masks = dev.empty((n,), torch.int64)
        stats = dev.empty((2,), torch.int32)
    streams = _attempt_streams(seed_seq, b, lazy_streams)

    def alias(zh, l0, l1):
        dev.call("sfft_alias_masks_range", dptr(cand.data), n, t1, cand.kmax, hptr(ms), hptr(zh), l0, l1,
                 dptr(scratch), words, dptr(masks), dptr(stats), ctx=ctx or "alias masks")

    def run(first=None):
        z = None
        stats_h = None
        attempt = 0
        prep = None
        extra = also
        for attempt, child in enumerate(streams, start=1):
            if first is not None and attempt == 1:
                z, zh, wait = first  # launched by the deferred call
                stats_h = wait()
            else:
                if attempt == 1 and guess is not None:
                    z = guess.z
                else:
                    rng = first_rng if (attempt == 1 and first_rng is not None and lazy_streams) \
                        else np.random.default_rng(child)
                    # one vectorised draw with per-row bounds == the reference's per-prime
                    # rng.integers(0, m, size=d) calls, element for element (tests/test_host.py)
                    z = rng.integers(0, ms[:, None], size=(l_max, t1), dtype=np.int64)
                zh = np.ascontiguousarray(z.astype(np.int32))
                alias(zh, 0, l_hi)
                if prepare is not None and attempt == 1:
                    # read the stats (and ``also``) back through events, so the
                    # preparation kernels queued behind the alias kernel run while
                    # the host continues
                    wait = dev.download_async(stats)
                    wait_x = dev.download_async(extra) if extra is not None else None
                    prep = prepare(ms[:l_hi], zh[:l_hi])
                    stats_h = wait()
                    if wait_x is not None:
                        extra = wait_x()  # handed back in DeviceScheme.extra
                elif extra is not None and attempt == 1:
                    stats_h, extra = dev.download_many(stats, extra)  # extra handed back in DeviceScheme.extra
                    stats_h = stats_h.view(np.int32)
                else:
                    stats_h = dev.download_small(stats)
            if int(stats_h[1]) != 0 and l_hi < l_max:
                # not covered by the first chunk: the remaining primes of the attempt
                alias(zh, l_hi, l_max)
                stats_h = dev.download_small(stats)
            if int(stats_h[1]) == 0:
                return DeviceScheme(primes, z, int(stats_h[0]), masks, attempt, 0, prep,
                                    extra=extra if isinstance(extra, np.ndarray) else None)
        return DeviceScheme(primes, z, l_max, masks, attempt, int(stats_h[1]), prep,
                            extra=extra if isinstance(extra, np.ndarray) else None)

    if defer:
        if guess is not None and prepare is None and also is None:
            # the first attempt's alias kernel now, its stats (and everything
            # after them) when the caller finishes
            zh = np.ascontiguousarray(guess.z.astype(np.int32))
            alias(zh, 0, l_hi)
            wait = dev.download_async(stats)
            return PendingScheme(lambda: run((guess.z, zh, wait)))
        done = run()
        return PendingScheme(lambda: done)
    return run()


class PendingScheme:
    """``build_scheme(defer=True)``: the first attempt's alias kernel is
    enqueued; ``finish()`` reads its stats back and completes the search
    (further chunks / attempts) exactly as the undeferred call."""

    def __init__(self, fn):
        self._fn = fn
        self._done = None

    def finish(self) -> DeviceScheme:
        if self._done is None:
            self._done = self._fn()
        return self._done


def scheme_to_host(dev: Device, cand_rows: np.ndarray, sch: DeviceScheme) -> MultipleRank1Lattice:
    """Host MultipleRank1Lattice view of a device scheme (bool masks per lattice)."""
    target = FrequencyIndexSet(cand_rows, cand_rows.shape[1], _presorted=True)
    words = dev.download(sch.masks).view(np.uint64)
    lattices, recon, masks = [], [], []
    for l in range(sch.L):
        mk = ((words >> np.uint64(l)) & np.uint64(1)).astype(bool)
        lattices.append(Rank1Lattice(sch.z[l], sch.primes[l]))
        recon.append(FrequencyIndexSet(cand_rows[mk], cand_rows.shape[1], _presorted=True))
        masks.append(mk)
    return MultipleRank1Lattice(lattices, recon, target, recon_masks=masks)


# ---------------------------------------------------------------------------
# step execution

def fft_size(m_max: int) -> int:
    """Bluestein convolution length for lattices of size <= m_max: the
    library's smallest supported P >= 2 m_max - 1 (powers of two, or
    f * 2^a * 2048 with f in {3, 5, 7, 9, 25}; plan.cuh fft_geom)."""
    P = int(_native.query("sfft_fft_size", int(m_max)))
    if P < 0:
        raise ValueError(f"lattice size {m_max} needs an FFT of more than 2^24 points")
    return P


@dataclass
class LatticeTables:
    ms: np.ndarray
    zs: np.ndarray
    P: int           # Bluestein convolution length (fft_size)
    tw: object
    chirp: object
    bhat: object
    ftab: object
    _pcache: dict = field(default_factory=dict, repr=False, compare=False)  # shared with the LRU entry

    def prefix(self, L: int) -> "LatticeTables | None":
        """Tables of the first L lattices (twiddles/chirps are concatenated in
        lattice order, one Bhat row per lattice: a prefix is a view), or None
        when the first L sizes need a smaller FFT than this set's.  The views
        are cached with the tables (the step's host path after the alias
        read-back is on the critical path)."""
        got = self._pcache.get(L)
        if got is None:
            ms = self.ms[:L]
            if fft_size(int(ms.max())) != self.P:
                got = False
            else:
                tot = int(ms.sum())
                got = (ms, self.tw[:tot], self.chirp[:tot], self.bhat[:L])
            self._pcache[L] = got
        if got is False:
            return None
        ms, tw, chirp, bhat = got
        zs = self.zs[:L] if self.zs is not None else None
        return LatticeTables(ms, zs, self.P, tw, chirp, bhat, self.ftab)


class _TableCache:
    """LRU of per-size tables (twiddles, chirps, transformed Bluestein kernels).

    They depend only on the lattice sizes M_l — like FFT plans (the
    reference's scipy/pocketfft keeps an LRU plan cache too) — and consecutive
    steps of a run, or repeated steps on sets of equal size, reuse the same
    primes.  Bounded by SFFT_B200_TABLE_CACHE_BYTES (default 8 GiB per device).
    """

    def __init__(self):
        import os
        from collections import OrderedDict
        self.cap = int(os.environ.get("SFFT_B200_TABLE_CACHE_BYTES", 8 << 30))
        self.entries: "OrderedDict[tuple, tuple]" = OrderedDict()
        self.bytes = 0
        self.hits = 0
        self.misses = 0

    def get(self, key):
        got = self.entries.get(key)
        if got is not None:
            self.entries.move_to_end(key)
            self.hits += 1
        return got

    def put(self, key, val, nbytes: int):
        self.misses += 1
        if nbytes > self.cap:
            return
        while self.entries and self.bytes + nbytes > self.cap:
            _, old = self.entries.popitem(last=False)
            self.bytes -= old[-1]
        self.entries[key] = val + (nbytes,)
        self.bytes += nbytes


_TABLES: dict[int, _TableCache] = {}


def _table_cache(dev: Device) -> _TableCache:
    tc = _TABLES.get(dev.index)
    if tc is None:
        tc = _TABLES[dev.index] = _TableCache()
    return tc


def clear_caches(dev: Device | None = None) -> None:
    """Drop every size-keyed cache (per-size lattice tables, FFT twiddle
    tables, the candidate-prime memo) so the next step pays what a step with
    never-seen lattice sizes pays (the bench's cold-step figures)."""
    _TABLES.clear()
    _PRIMES_MEMO.clear()
    if dev is not None:
        dev._ftab.clear()


def lattice_tables(dev: Device, ms: np.ndarray, zs: np.ndarray | None, ctx: str = "",
                   cache: bool = True) -> LatticeTables:
    torch = dev.torch
    ms = np.ascontiguousarray(np.asarray(ms, dtype=np.int64))
    L = len(ms)
    P = fft_size(int(ms.max()))
    key = (P,) + tuple(int(m) for m in ms)
    tc = _table_cache(dev)
    got = tc.get(key) if cache else None
    ftab = dev.fft_tables(P)
    if got is not None:
        tw, chirp, bhat, pc, _ = got
        return LatticeTables(ms, zs, P, tw, chirp, bhat, ftab, pc)
    tot = int(ms.sum())
    tw = dev.empty((tot, 2), torch.float64)
    chirp = dev.empty((tot, 2), torch.float64)
    dev.call("sfft_lattice_tables", hptr(ms), L, dptr(tw), dptr(chirp), ctx=ctx)
    bhat = dev.empty((L, P, 2), torch.float64)
    dev.call("sfft_bluestein_bhat", hptr(ms), L, P, dptr(ftab), dptr(chirp), dptr(bhat), ctx=ctx)
    pc: dict = {}
    if cache:
        tc.put(key, (tw, chirp, bhat, pc), 32 * tot + 16 * L * P)
    return LatticeTables(ms, zs, P, tw, chirp, bhat, ftab, pc)


@dataclass
class StepResult:
    keep: object              # torch uint8 (r, n)
    coef: object              # torch float64 (r, n, 2)
    _counts: np.ndarray | None  # survivors per iteration after threshold and cap
    nodes: int                # oracle samples taken
    timings: dict = field(default_factory=dict)
    _finish: object = None    # pending cap check (run_step(defer_cap=True))
    _lazy: object = None      # counts read back only when asked for (the cap could not bind)

    def finalize(self) -> "StepResult":
        """Apply the cap (detect.py:205-211) if it is still pending: waits for
        this step's survivor counts and runs the exact cap selection on the
        iterations that exceed it.  Must precede any use of keep / coef."""
        if self._finish is not None:
            fin, self._finish = self._finish, None
            self._counts = fin()
        return self

    @property
    def counts(self) -> np.ndarray:
        self.finalize()
        if self._counts is None and self._lazy is not None:
            self._counts = self._lazy()
        return self._counts


def _unit_arg(units):
    """(host int32 array or None, count) for the C ABI's unit lists."""
    if units is None:
        return None, 0
    arr = np.ascontiguousarray(np.asarray(units, dtype=np.int32))
    return arr, len(arr)


def _sample_units(dev: Device, oracle, tabs: LatticeTables, t1: int, d: int,
                  tails: list[np.ndarray], buf, step: int, it0: int, units=None, scratch=None,
                  prepared: bool = False, panels_ready: bool = False):
    """Fill buffer slot j with the pre-chirped samples of unit units[j]
    (global id i * L + l within this chunk of iterations; all rb * L units in
    order when ``units`` is None).  Noise streams are consumed for every unit
    of the chunk in the reference's call order, whichever units are local."""
    torch = dev.torch
    L = len(tabs.ms)
    rb = len(tails)
    P = tabs.P
    tail = d - t1
    anchor = np.ascontiguousarray(np.asarray(tails, dtype=np.float64).reshape(rb, tail)) \
        if tail else np.zeros(1, dtype=np.float64)
    ulist = range(rb * L) if units is None else [int(u) for u in units]
    uarr, nu = _unit_arg(units)
    up = hptr(uarr) if uarr is not None else 0
    if units is None:
        nodes = rb * int(tabs.ms.sum())
    else:
        nodes = int(tabs.ms[np.asarray(ulist, dtype=np.int64) % L].sum()) if len(ulist) else 0
    base = oracle.inner if isinstance(oracle, NoisyOracle) else oracle
    device_inner = isinstance(base, (SparsePolynomialOracle, BSplineOracle))
    noisy = isinstance(oracle, NoisyOracle)
    chirp_now = 0 if noisy else 1
    if device_inner:
        if isinstance(base, SparsePolynomialOracle):
            hf, cf = base.device_terms(dev)
            s = base.s

            def launch(name, cprime, rres, rj, part, panels=False):
                extra = (1 if panels else 0,) if name == "sfft_sample_poly_run" else ()
                dev.call(name, dptr(hf), dptr(cf), s, d, t1, hptr(tabs.ms), hptr(tabs.zs), L,
                         hptr(anchor), rb, dptr(cprime), dptr(rres), dptr(rj), dptr(tabs.tw),
                         dptr(tabs.chirp), dptr(buf), P, chirp_now, dptr(part), int(part.shape[0]), up, nu,
                         *extra, ctx=f"sampling, step {step}")

            done = False
            if scratch is not None:
                # the library checks the scratch against this plan's need (E_2BIG if short)
                try:
                    if prepared:
                        launch("sfft_sample_poly_run", *scratch, panels=panels_ready)
                    else:
                        launch("sfft_sample_poly", *scratch)
                    done = True
                except _native.NativeError as exc:
                    if exc.code != _native.E_2BIG:
                        raise
                    if prepared:  # operands are ready; only the scratch is short (panels rebuilt)
                        need = int(_native.query("sfft_sample_poly_scratch", hptr(tabs.ms), L, rb, s, up, nu))
                        launch("sfft_sample_poly_run", *scratch[:3],
                               dev.empty((max(need, 1), 2), torch.float64))
                        done = True
            if not done:
                need = int(_native.query("sfft_sample_poly_scratch", hptr(tabs.ms), L, rb, s, up, nu))
                launch("sfft_sample_poly", dev.empty((rb, max(s, 1), 2), torch.float64),
                       dev.empty((L, max(s, 1)), torch.int32), dev.empty((L, max(s, 1)), torch.int32),
                       dev.empty((max(need, 1), 2), torch.float64))
        else:
            order, start, comps, scale = base.host_spec()
            dev.call("sfft_sample_bspline", len(base.groups), hptr(order), hptr(start), hptr(comps),
                     hptr(scale), d, t1, hptr(tabs.ms), hptr(tabs.zs), L, hptr(anchor), rb,
                     dptr(tabs.chirp), dptr(buf), P, chirp_now, up, nu, ctx=f"sampling, step {step}")
        if noisy:
            _add_lattice_noise(dev, oracle, tabs, rb, buf, ulist, uarr)
        else:
            base.count_samples(nodes)
        return nodes
    # host callback: nodes on the device, values from the callback
    pts = dev.empty((int(tabs.ms.max()), d), torch.float64)
    for j, u in enumerate(ulist):
        i, l = divmod(u, L)
        m = int(tabs.ms[l])
        tail_i = np.ascontiguousarray(anchor[i] if tail else np.zeros(1))
        dev.call("sfft_lattice_nodes", hptr(tabs.ms), hptr(tabs.zs), L, t1, l, d, hptr(tail_i),
                 dptr(pts), ctx=f"lattice nodes, step {step}")
        host_pts = dev.download(pts[:m])
        vals = evaluate_callback(oracle, host_pts, step, it0 + i)
        v2 = np.ascontiguousarray(np.stack([vals.real, vals.imag], axis=1))
        with torch.cuda.stream(dev.stream):
            buf[j, :m].copy_(torch.from_numpy(v2), non_blocking=False)
    dev.call("sfft_finish_samples", hptr(tabs.ms), L, rb, dptr(tabs.chirp), dptr(buf), P, 0, 0, 0, up, nu,
             ctx=f"pre-chirp, step {step}")
    return nodes


def _add_lattice_noise(dev: Device, oracle: NoisyOracle, tabs: LatticeTables, rb: int, buf,
                       ulist: list[int], uarr):
    """Noise in the reference's call order (iteration-major, then lattice),
    drawn from the oracle's numpy stream for every unit of the chunk, added on
    the device (local units only) together with the pre-chirp."""
    torch = dev.torch
    L = len(tabs.ms)
    P = tabs.P
    mmax = int(tabs.ms.max())
    nu = len(ulist)
    up = hptr(uarr) if uarr is not None else 0
    nuarg = len(uarr) if uarr is not None else 0
    if oracle.device_rng:
        base = oracle.reserve_calls(rb * L)
        nrm = None
        if oracle.needs_norm():
            nrm = dev.empty((nu,), torch.float64)
            dev.call("sfft_unit_norm2", hptr(tabs.ms), L, rb, dptr(buf), P, dptr(nrm), up, nuarg,
                     ctx="noise norm")
        dev.call("sfft_finish_devnoise", hptr(tabs.ms), L, rb, dptr(tabs.chirp), dptr(buf), P,
                 dptr(nrm) if nrm is not None else 0, getattr(oracle, "rel", 0.0), oracle.sigma,
                 oracle.device_key, base, 1, up, nuarg, ctx="device noise")
        oracle.count_samples(int(tabs.ms[np.asarray(list(ulist), dtype=np.int64) % L].sum()) if len(ulist) else 0)
        return
    norms = {}
    if oracle.needs_norm():
        nrm = dev.empty((nu,), torch.float64)
        dev.call("sfft_unit_norm2", hptr(tabs.ms), L, rb, dptr(buf), P, dptr(nrm), up, nuarg,
                 ctx="noise norm")
        norms = dict(zip(ulist, dev.download(nrm).tolist()))
    slot = {u: j for j, u in enumerate(ulist)}
    noise = np.zeros((nu, mmax, 2), dtype=np.float64)
    sig = np.zeros(nu, dtype=np.float64)
    for u in range(rb * L):
        m = int(tabs.ms[u % L])
        e = oracle.draw(m)
        oracle.count_samples(m)
        j = slot.get(u)
        if j is not None:
            noise[j, :m] = e
            sig[j] = oracle.scale_for(norms.get(u, 0.0), m)
    d_noise = dev.upload(noise)
    d_sig = dev.upload(sig)
    dev.call("sfft_finish_samples", hptr(tabs.ms), L, rb, dptr(tabs.chirp), dptr(buf), P,
             dptr(d_noise), mmax, dptr(d_sig), up, nuarg, ctx="noisy samples")


class StageTimer:
    """CUDA-event brackets around the stages of run_step (on the engine stream)."""

    def __init__(self, dev: Device):
        self.dev = dev
        self.marks: list[tuple[str, object, object]] = []

    def span(self, name: str):
        timer = self

        class _Span:
            def __enter__(self_inner):
                self_inner.a = timer.dev.torch.cuda.Event(enable_timing=True)
                self_inner.a.record(timer.dev.stream)

            def __exit__(self_inner, *exc):
                b = timer.dev.torch.cuda.Event(enable_timing=True)
                b.record(timer.dev.stream)
                timer.marks.append((name, self_inner.a, b))
                return False

        return _Span()

    def totals_ms(self) -> dict:
        self.dev.sync()
        out: dict = {}
        for name, a, b in self.marks:
            out.setdefault(name, []).append(a.elapsed_time(b))
        return out


class _NoTimer:
    def span(self, name):
        import contextlib
        return contextlib.nullcontext()


@dataclass
class StepPrep:
    """Everything of a single-chunk step that does not depend on the
    early-exit L, made while the alias kernel runs (``build_scheme(prepare=)``):
    the per-size tables of all L_max primes (cached; the used lattices' are a
    prefix), the output buffers, the transform buffer and the sampling scratch
    sized for L_max lattices."""
    tabs: LatticeTables | None  # None: not cached (run_step builds the L it uses)
    keep: object
    coef: object
    counts: object
    buf: object
    poly: tuple | None
    r: int
    n: int
    poly_ready: bool = False  # c' and residues of all L_max lattices computed (attempt 1's vectors)
    l_max: int = 0
    panels_ready: bool = False  # tensor-core B panels of all L_max lattices built in poly[3]


def prepare_step(dev: Device, oracle, cand: DeviceFreqs, r: int, ms_all, zs_all,
                 cached_tables_only: bool = False, tails=None, d: int | None = None) -> StepPrep | None:
    """Host work of ``run_step`` that can overlap the alias kernel (single
    chunk of iterations, r * L_max <= the unit capacity); None otherwise.
    ``cached_tables_only``: do not build the per-size tables of all L_max
    primes when they are not cached already (run_step then builds the L it
    uses), so a step with new sizes does no extra table work."""
    torch = dev.torch
    ms_all = np.ascontiguousarray(np.asarray(ms_all, dtype=np.int64))
    L_max = len(ms_all)
    if r * L_max > UMAX or r > RBMAX:
        return None
    zs32 = np.ascontiguousarray(np.asarray(zs_all).astype(np.int32))
    P_all = fft_size(int(ms_all.max()))
    tabs = None
    if not cached_tables_only or \
            _table_cache(dev).get((P_all,) + tuple(int(m) for m in ms_all)) is not None:
        tabs = lattice_tables(dev, ms_all, zs32, ctx="lattice tables (prepared)")
    n = cand.n
    keep = dev.empty((r, n), torch.uint8)
    coef = dev.empty((r, n, 2), torch.float64)
    counts = dev.zeros_fast((r,), torch.int32)
    # the transform buffer for all L_max lattices only while that is small
    # (the early-exit L is about half of L_max); otherwise run_step allocates
    buf = dev.empty((r * L_max, P_all, 2), torch.float64) \
        if r * L_max * 16 * P_all <= (1 << 30) else None
    poly = None
    ready = False
    built = np.zeros(1, dtype=np.int32)
    base = oracle.inner if isinstance(oracle, NoisyOracle) else oracle
    if isinstance(base, SparsePolynomialOracle):
        s = max(base.s, 1)
        # sized for L_max lattices (the rare smaller-L plan that needs more
        # partial-sum space allocates its own in _sample_units)
        need = int(_native.query("sfft_sample_poly_scratch", hptr(ms_all), L_max, r, base.s, 0, 0))
        poly = (dev.empty((r, s, 2), torch.float64), dev.empty((L_max, s), torch.int32),
                dev.empty((L_max, s), torch.int32), dev.empty((max(need, 1), 2), torch.float64))
        if tails is not None and d is not None and len(tails) == r and base.s > 0:
            # anchor-rotated coefficients and the residues of every candidate
            # lattice now; run_step then only launches the contraction
            t1 = cand.ncomp
            tail = d - t1
            anchor = np.ascontiguousarray(np.asarray(tails, dtype=np.float64).reshape(r, tail)) \
                if tail else np.zeros(1, dtype=np.float64)
            hf, cf = base.device_terms(dev)
            dev.call("sfft_sample_poly_prepare", dptr(hf), dptr(cf), base.s, d, t1, hptr(ms_all), hptr(zs32),
                     L_max, hptr(anchor), r, dptr(poly[0]), dptr(poly[1]), dptr(poly[2]),
                     dptr(tabs.tw) if tabs is not None else 0, dptr(poly[3]), int(poly[3].shape[0]),
                     hptr(built), ctx="sampling operands (prepared)")
            ready = True
    return StepPrep(tabs, keep, coef, counts, buf, poly, r, n, ready, L_max, bool(built[0]))


def run_step(dev: Device, oracle, cand: DeviceFreqs, sch: DeviceScheme, tails: list[np.ndarray],
             d: int, delta: float, cap: int, step: int = 0, tabs: LatticeTables | None = None,
             timer: StageTimer | None = None, defer_cap: bool = False,
             prep: StepPrep | None = None, device_cap: bool = False) -> StepResult:
    """Sample, transform and invert all r~ iterations of one step; threshold + cap.

    ``defer_cap``: return as soon as the work is enqueued; the survivor counts
    come back asynchronously and the cap is applied by ``StepResult.finalize()``
    (or the first ``.counts`` access), so the host can prepare the next
    independent step while this one runs.  ``prep``: buffers and tables made
    by ``prepare_step`` while the alias kernel ran.  ``device_cap``: the cap
    is decided and applied on the device for every iteration (no host
    read-back at all; ``.counts`` downloads on first use)."""
    torch = dev.torch
    tm = timer or _NoTimer()
    n = cand.n
    t1 = cand.ncomp
    L = sch.L
    r = len(tails)
    if prep is not None and (prep.r != r or prep.n != n or prep.l_max < L):
        prep = None
    if tabs is None and prep is not None and prep.tabs is not None:
        tabs = prep.tabs.prefix(L)
        if tabs is not None:
            tabs.zs = sch.z_used  # the accepted attempt's vectors
    if tabs is None:
        with tm.span("tables"):
            tabs = lattice_tables(dev, sch.m_used, sch.z_used, ctx=f"lattice tables, step {step}")
    P = tabs.P
    rb_max = max(1, min(RBMAX, UMAX // L))
    rb_alloc = min(rb_max, r)
    if prep is not None:
        keep, coef, counts, scratch = prep.keep, prep.coef, prep.counts, prep.poly
        if prep.buf is not None and prep.buf.shape[1] == P:
            buf = prep.buf[: rb_alloc * L]
        else:
            buf = dev.empty((rb_alloc * L, P, 2), torch.float64)
    else:
        keep = dev.empty((r, n), torch.uint8)
        coef = dev.empty((r, n, 2), torch.float64)
        counts = dev.zeros_fast((r,), torch.int32)
        buf = dev.empty((rb_alloc * L, P, 2), torch.float64)
        scratch = None
    nodes = 0
    for i0 in range(0, r, rb_max):
        rb = min(rb_max, r - i0)
        # the prepared operands and B panels belong to the first attempt's vectors
        prepared = prep is not None and prep.poly_ready and sch.attempts == 1 and i0 == 0 and rb == r
        with tm.span("sample"):
            nodes += _sample_units(dev, oracle, tabs, t1, d, tails[i0:i0 + rb], buf, step, i0,
                                   scratch=scratch, prepared=prepared,
                                   panels_ready=prepared and prep.panels_ready)
        with tm.span("fft"):
            dev.call("sfft_bluestein", hptr(tabs.ms), L, rb, tabs.P, dptr(tabs.ftab), dptr(tabs.bhat),
                     dptr(tabs.chirp), dptr(buf), 0, 0, ctx=f"Bluestein FFT, step {step}")
        with tm.span("gather"):
            dev.call("sfft_gather_select", dptr(cand.data), n, t1, cand.kmax, hptr(tabs.ms), hptr(tabs.zs), L,
                     dptr(sch.masks), dptr(buf), P, rb, i0, float(delta), dptr(coef), dptr(keep),
                     dptr(counts), ctx=f"gather/select, step {step}")
    def apply_cap(counts_h):
        return apply_cap_rows(dev, coef, keep, n, counts_h, cap, step)

    if cap >= n:  # the cap cannot bind: no selection, nothing to wait for
        return StepResult(keep, coef, None, nodes, _lazy=lambda: dev.download_small(counts).astype(np.int64))
    if device_cap:
        for c0 in range(0, r, 64):
            rows = np.arange(c0, min(r, c0 + 64), dtype=np.int32)
            sbytes = int(_native.query("sfft_select_rows_scratch_bytes", len(rows)))
            scratch_sel = dev.empty((max(sbytes, 1),), torch.uint8)
            dev.call("sfft_select_cap_rows", dptr(coef), dptr(keep), n, hptr(rows), len(rows), int(cap),
                     dptr(counts), dptr(scratch_sel), ctx=f"cap selection, step {step}")
        return StepResult(keep, coef, None, nodes,
                          _finish=lambda: dev.download_small(counts).astype(np.int64))

    if defer_cap:
        wait = dev.download_async(counts)
        return StepResult(keep, coef, None, nodes, _finish=lambda: apply_cap(wait()))
    return StepResult(keep, coef, apply_cap(dev.download_small(counts)), nodes)


def apply_cap_rows(dev: Device, coef, keep, n: int, counts_h: np.ndarray, cap: int, step: int = 0) -> np.ndarray:
    """The cap of detect.py:205-211 on every iteration whose survivor count
    exceeds it: the exact radix selection of all such rows in one batched
    launch sequence (sfft_select_cap_rows).  Returns the updated counts."""
    counts_h = np.asarray(counts_h).astype(np.int64)
    over = np.ascontiguousarray([i for i in range(len(counts_h)) if counts_h[i] > cap], dtype=np.int32)
    for c0 in range(0, len(over), 64):
        rows = np.ascontiguousarray(over[c0:c0 + 64])
        sbytes = int(_native.query("sfft_select_rows_scratch_bytes", len(rows)))
        scratch = dev.empty((max(sbytes, 1),), dev.torch.uint8)
        dev.call("sfft_select_cap_rows", dptr(coef), dptr(keep), n, hptr(rows), len(rows), int(cap), 0,
                 dptr(scratch), ctx=f"cap selection, step {step}")
    counts_h[over] = cap
    return counts_h


def compact(dev: Device, cand: DeviceFreqs, flags, nrows: int, coef=None):
    """Rows of ``cand`` whose flag (OR over ``nrows`` rows) is set, in order;
    optional coefficient gather.  Returns (DeviceFreqs, coef tensor | None)."""
    return compact_finish(compact_start(dev, cand, flags, nrows, coef))


def compact_start(dev: Device, cand: DeviceFreqs, flags, nrows: int, coef=None):
    """First half of ``compact``: the flag scan and the asynchronous read-back
    of the survivor count.  The caller may enqueue more device work and do
    host work before ``compact_finish`` waits for the count."""
    torch = dev.torch
    n = cand.n
    idx = dev.empty((max(n, 1),), torch.int32)
    total = dev.empty((1,), torch.int32)
    sl = int(_native.query("sfft_scan_scratch_len", n))
    scr = dev.empty((max(sl, 1),), torch.int32)
    dev.call("sfft_flag_indices", dptr(flags), n, nrows, dptr(idx), dptr(total), dptr(scr), ctx="compaction")
    return dev, cand, idx, total, coef, dev.download_async(total)


def compact_count(pending) -> int:
    """The survivor count of a ``compact_start`` (waits for its read-back)."""
    return int(pending[5]()[0])


def compact_finish(pending):
    dev, cand, idx, total, coef, wait = pending
    torch = dev.torch
    n = cand.n
    cnt = int(wait()[0])
    out = dev.empty((cand.ncomp, max(cnt, 1)), torch.int32)
    cout = dev.empty((max(cnt, 1), 2), torch.float64) if coef is not None else None
    dev.call("sfft_gather_rows", dptr(cand.data), n, cand.ncomp, dptr(idx), dptr(total), cnt, dptr(out),
             max(cnt, 1), dptr(coef) if coef is not None else 0, dptr(cout) if cout is not None else 0,
             ctx="row gather")
    res = DeviceFreqs(out[:, :cnt] if cnt else out[:, :0], cnt, cand.kmax)
    if cnt and out.shape[1] != cnt:
        res.data = out[:, :cnt].contiguous()
    return res, (cout[:cnt] if cout is not None else None)


def product(dev: Device, prefixes: DeviceFreqs, comp: np.ndarray) -> DeviceFreqs:
    """Candidate product prefixes x comp in row-major (hence lexicographic) order."""
    torch = dev.torch
    comp = np.ascontiguousarray(np.asarray(comp, dtype=np.int32))
    nc = len(comp)
    tot = prefixes.n * nc
    out = dev.empty((prefixes.ncomp + 1, max(tot, 1)), torch.int32)
    if tot:
        d_comp = dev.upload(comp, asynchronous=True)  # no stream drain per step
        dev.call("sfft_candidate_product", dptr(prefixes.data), prefixes.n, prefixes.ncomp,
                 dptr(d_comp), nc, dptr(out), ctx="candidate product")
    kmax = max(prefixes.kmax, int(np.abs(comp).max()) if nc else 0)
    data = out if tot == out.shape[1] else out[:, :tot].contiguous()
    return DeviceFreqs(data, tot, kmax)
