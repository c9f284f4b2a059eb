"""Dimension-incremental sparse FFT engine (Algorithm 3 of arXiv 1711.05152)
driving the device MR1L step — the public reconstruction API of the
reference's detect.py (sparse_fft, DetectionConfig, DetectionReport,
detect_component, projected_line_coefficients, planners and bounds).

Per component step t the engine
  1. detects the 1-D component set from r anchored lines (device line kernels),
  2. forms J_t = prefixes x component on the device (already sorted),
  3. builds the MR1L scheme on the device (alias histograms, K3),
  4. runs all r~ iterations of sampling + Bluestein + gather/threshold/cap,
  5. unions the kept sets by flag compaction into the next prefixes.
RNG consumption matches the reference stream for stream (detect.py:328-399),
so lattices, anchors and therefore the detected sets are the reference's.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace
from typing import Sequence

import numpy as np

from .core import FrequencyIndexSet, SearchBox, SparseSpectrum
from .device import Device, dptr, get_device, hptr
from .mr1l import (DeviceFreqs, OracleError, OracleInterrupt, build_scheme, compact, compact_count, compact_finish,
                   compact_start, prepare_step,
                   evaluate_callback, first_attempt_rng, product, run_step)
from .oracles import BSplineOracle, NoisyOracle, SparsePolynomialOracle
from .primes import MLConfig

__all__ = [
    "DetectionConfig",
    "DetectionReport",
    "OracleInterrupt",
    "projected_line_coefficients",
    "detect_component",
    "sparse_fft",
    "plan_r",
    "plan_b",
    "failure_bound_single_coeff",
    "union_failure_bound",
]


@dataclass(frozen=True)
class DetectionConfig:
    """Engine parameters (reference detect.py:64-127); same fields, defaults
    and validation errors."""

    box: SearchBox
    delta: float
    s: int
    s_local: int | None = None
    r: int = 1
    b: int = 1
    mode: str = "randomized"
    lattice_kind: str = "multiple"
    rng_seed: int = 0
    dimension_order: tuple[int, ...] | None = None
    component_delta: float | None = None

    def __post_init__(self):
        if not isinstance(self.box, SearchBox):
            raise TypeError("box must be a SearchBox")
        if not self.delta > 0:
            raise ValueError("delta must be > 0")
        if self.s < 1:
            raise ValueError("sparsity cap s must be >= 1")
        if self.s_local is not None and self.s_local < 1:
            raise ValueError("s_local must be >= 1")
        if self.r < 1:
            raise ValueError("detection iterations r must be >= 1")
        if self.b < 1:
            raise ValueError("lattice retry cap b must be >= 1")
        if self.mode not in ("randomized", "deterministic_zero_anchor"):
            raise ValueError("mode must be 'randomized' or 'deterministic_zero_anchor'")
        if self.lattice_kind not in ("multiple", "single"):
            raise ValueError("lattice_kind must be 'multiple' or 'single'")
        if self.rng_seed < 0:
            raise ValueError("rng_seed must be a nonnegative integer")
        if self.component_delta is not None and not self.component_delta > 0:
            raise ValueError("component_delta must be > 0")
        if self.dimension_order is not None:
            order = tuple(int(c) for c in self.dimension_order)
            if sorted(order) != list(range(self.box.dim)):
                raise ValueError("dimension_order must be a permutation of 0..d-1")
            object.__setattr__(self, "dimension_order", order)

    @property
    def local_sparsity(self) -> int:
        return self.s if self.s_local is None else self.s_local

    @property
    def component_threshold(self) -> float:
        return self.delta if self.component_delta is None else self.component_delta


@dataclass
class DetectionReport:
    """Result and exact accounting of one run (reference detect.py:130-150)."""

    detected: SparseSpectrum
    component_counts: list[int] = field(default_factory=list)
    prefix_counts: list[int] = field(default_factory=list)
    candidate_counts: list[int] = field(default_factory=list)
    scheme_sizes: list[int] = field(default_factory=list)
    lattice_attempts: list[int] = field(default_factory=list)
    detection_calls: list[int] = field(default_factory=list)
    inversion_calls: list[int] = field(default_factory=list)
    oracle_calls: int = 0
    warnings: list[str] = field(default_factory=list)
    wall_time: float = 0.0
    step_times: list[float] = field(default_factory=list)


# ---------------------------------------------------------------------------
# oracle plumbing

class _PermutedCallback:
    """Host-callback oracle seen through a coordinate permutation (detect.py:243-254)."""

    def __init__(self, inner, order: Sequence[int]):
        self._inner = inner
        self._order = np.asarray(order, dtype=np.intp)
        self.dim = len(self._order)

    def __call__(self, points: np.ndarray) -> np.ndarray:
        full = np.empty_like(points)
        full[:, self._order] = points
        return self._inner(full)


def _is_device_oracle(oracle) -> bool:
    base = oracle.inner if isinstance(oracle, NoisyOracle) else oracle
    return isinstance(base, (SparsePolynomialOracle, BSplineOracle))


def _permute_oracle(oracle, order):
    if _is_device_oracle(oracle):
        return oracle.permuted(order)
    return _PermutedCallback(oracle, order)


def _line_values(dev: Device, oracle, t: int, box: SearchBox, anchors: np.ndarray, step: int, it0: int,
                 out=None):
    """Samples of r anchored axis lines of component t -> device (r, K, 2)
    (into ``out`` when given)."""
    torch = dev.torch
    r, d = anchors.shape
    K = int(box.sizes[t])
    vals = dev.empty((r, K, 2), torch.float64) if out is None else out
    base = oracle.inner if isinstance(oracle, NoisyOracle) else oracle
    noisy = isinstance(oracle, NoisyOracle)
    if isinstance(base, SparsePolynomialOracle):
        hf, cf = base.device_terms(dev)
        per = max(1, 2048 // d)
        for i0 in range(0, r, per):
            a = np.ascontiguousarray(anchors[i0:i0 + per])
            dev.call("sfft_line_sample_poly", dptr(hf), dptr(cf), base.s, d, t, K, hptr(a), len(a),
                     dptr(vals[i0:]), ctx=f"line sampling, step {step}")
    elif isinstance(base, BSplineOracle):
        pts = np.repeat(anchors, K, axis=0)
        pts[:, t] = np.tile(np.arange(K) / K, r)
        d_pts = dev.upload(np.ascontiguousarray(pts), asynchronous=True)  # no stream drain per component
        order, start, comps, scale = base.host_spec()
        dev.call("sfft_eval_bspline_points", dptr(d_pts), r * K, d, len(base.groups), hptr(order),
                 hptr(start), hptr(comps), hptr(scale), dptr(vals), ctx=f"line sampling, step {step}")
    else:
        host = np.empty((r, K, 2))
        for i in range(r):
            pts = np.tile(anchors[i], (K, 1))
            pts[:, t] = np.arange(K) / K
            v = evaluate_callback(oracle, pts, step, it0 + i)
            host[i, :, 0], host[i, :, 1] = v.real, v.imag
        with torch.cuda.stream(dev.stream):
            vals.copy_(torch.from_numpy(host))
        return vals
    if noisy and oracle.device_rng:
        km = np.array([K], dtype=np.int64)
        base_call = oracle.reserve_calls(r)
        nrm = None
        if oracle.needs_norm():
            nrm = dev.empty((r,), torch.float64)
            dev.call("sfft_unit_norm2", hptr(km), 1, r, dptr(vals), K, dptr(nrm), 0, 0, ctx="line noise norm")
        dev.call("sfft_finish_devnoise", hptr(km), 1, r, dptr(vals), dptr(vals), K,
                 dptr(nrm) if nrm is not None else 0, getattr(oracle, "rel", 0.0), oracle.sigma,
                 oracle.device_key, base_call, 0, 0, 0, ctx="line device noise")
        oracle.count_samples(r * K)
    elif noisy:
        norms = None
        if oracle.needs_norm():
            nrm = dev.empty((r,), torch.float64)
            km = np.array([K], dtype=np.int64)
            dev.call("sfft_unit_norm2", hptr(km), 1, r, dptr(vals), K, dptr(nrm), 0, 0, ctx="line noise norm")
            norms = dev.download(nrm)
        for i in range(r):
            e = dev.upload(np.ascontiguousarray(oracle.draw(K)))
            sc = oracle.scale_for(float(norms[i]) if norms is not None else 0.0, K)
            dev.call("sfft_add_noise", dptr(vals[i]), dptr(e), K, sc, ctx="line noise")
            oracle.count_samples(K)
    else:
        base.count_samples(r * K)
    return vals


def _lines(dev: Device, oracle, t: int, box: SearchBox, anchors: np.ndarray, cap: int, delta: float,
           step: int):
    """Device line detection: (ks, coefs (r, K) complex, keep (r, K) bool)."""
    torch = dev.torch
    r = anchors.shape[0]
    K = int(box.sizes[t])
    lo = int(box.lows[t])
    vals = _line_values(dev, oracle, t, box, anchors, step, 0)
    coefs = dev.empty((r, K, 2), torch.float64)
    keep = dev.empty((r, K), torch.uint8)
    if K <= 1024:
        dev.call("sfft_line_select", dptr(vals), r, K, lo, int(cap), float(delta), dptr(coefs), dptr(keep),
                 ctx=f"line selection, step {step}")
    else:
        _long_line_select(dev, vals, r, K, lo, int(cap), float(delta), coefs, keep, step)
    return np.arange(lo, lo + K, dtype=np.int64), coefs, keep


def _long_line_select(dev: Device, vals, r: int, K: int, lo: int, cap: int, delta: float, coefs, keep,
                      step: int):
    """Lines longer than 1024 points: each line is one unit of a 'lattice'
    of size K through the MR1L step's own Bluestein kernels (dft_1d of
    detect.py:191), then bins/threshold (sfft_line_bins) and the exact row
    cap (sfft_select_cap_rows: |c| desc, then k asc — the lines' q order)."""
    from . import _native
    from .mr1l import UMAX, lattice_tables
    torch = dev.torch
    tabs = lattice_tables(dev, np.array([K], dtype=np.int64), None, ctx=f"line tables, step {step}")
    counts = dev.empty((r,), torch.int32)
    per = min(r, UMAX)
    buf = dev.zeros((per, tabs.P, 2), torch.float64)
    for i0 in range(0, r, per):
        nb = min(per, r - i0)
        with torch.cuda.stream(dev.stream):
            buf[:nb, :K].copy_(vals[i0:i0 + nb])
        dev.call("sfft_finish_samples", hptr(tabs.ms), 1, nb, dptr(tabs.chirp), dptr(buf), tabs.P, 0, 0, 0, 0, 0,
                 ctx=f"line pre-chirp, step {step}")
        dev.call("sfft_bluestein", hptr(tabs.ms), 1, nb, tabs.P, dptr(tabs.ftab), dptr(tabs.bhat),
                 dptr(tabs.chirp), dptr(buf), 0, 0, ctx=f"line DFT, step {step}")
        dev.call("sfft_line_bins", dptr(buf), tabs.P, nb, K, lo, delta, dptr(coefs[i0:]), dptr(keep[i0:]),
                 dptr(counts[i0:]), ctx=f"line bins, step {step}")
    for c0 in range(0, r, 64):
        rows = np.arange(c0, min(r, c0 + 64), dtype=np.int32)
        sbytes = int(_native.query("sfft_select_rows_scratch_bytes", len(rows)))
        scratch = dev.empty((max(sbytes, 1),), torch.uint8)
        dev.call("sfft_select_cap_rows", dptr(coefs), dptr(keep), K, hptr(rows), len(rows), cap, dptr(counts),
                 dptr(scratch), ctx=f"line cap, step {step}")


def projected_line_coefficients(oracle, t: int, box: SearchBox, anchor: np.ndarray,
                                *, _step_ctx: tuple[int, int] = (0, 0)):
    """Projected 1-D coefficients along component t at one anchor
    (reference detect.py:175-194), computed on the device."""
    dev = get_device()
    anchor = np.asarray(anchor, dtype=np.float64).reshape(1, -1)
    ks, coefs, _ = _lines(dev, oracle, t, box, anchor, 1 << 30, 1.0, _step_ctx[0])
    c = dev.download(coefs)[0]
    return ks, c[:, 0] + 1j * c[:, 1]


def _detect_launch(dev: Device, oracle, t: int, cfg: DetectionConfig, rng: np.random.Generator, step: int):
    box = cfg.box
    d = box.dim
    zero = cfg.mode == "deterministic_zero_anchor"
    anchors = np.stack([np.zeros(d) if zero else rng.random(d) for _ in range(cfg.r)])
    ks, _, keep = _lines(dev, oracle, t, box, anchors, cfg.local_sparsity, cfg.component_threshold, step)
    return ks, keep


def _detect(dev: Device, oracle, t: int, cfg: DetectionConfig, rng: np.random.Generator, step: int):
    ks, keep = _detect_launch(dev, oracle, t, cfg, rng, step)
    hit = dev.download(keep).astype(bool).any(axis=0)
    return ks[hit]


def _detect_all(dev: Device, oracle, cfg: DetectionConfig, streams) -> list[np.ndarray]:
    """Line detection of every component at once: each
    component's lines use their own stream (detect_streams[t]) and do not
    depend on the other steps, so for a noiseless device oracle all d
    detections are launched back to back and read back with one
    synchronisation.  (Noisy and host-callback oracles keep the reference's
    per-step call order.)"""
    return _detect_all_collect(dev, _detect_all_launch(dev, oracle, cfg, streams))


def _detect_all_launch(dev: Device, oracle, cfg: DetectionConfig, streams):
    """Launch the line detections of all components.  When every component
    has the same extent (a centred box), the r lines of all d components go
    through one sample buffer and ONE selection launch (rows are independent
    lines, detect.py:229-236 per line), and a B-spline oracle evaluates all
    d * r * K nodes in one launch from one upload."""
    box = cfg.box
    d = box.dim
    same = len({(int(k), int(lo)) for k, lo in zip(box.sizes, box.lows)}) == 1
    base = oracle.inner if isinstance(oracle, NoisyOracle) else oracle
    if not same or isinstance(oracle, NoisyOracle) or int(box.sizes[0]) > 1024 or \
            not isinstance(base, (SparsePolynomialOracle, BSplineOracle)):
        return [_detect_launch(dev, oracle, t, cfg, np.random.default_rng(streams[t]), t) for t in range(d)]
    torch = dev.torch
    zero = cfg.mode == "deterministic_zero_anchor"
    r, K, lo = cfg.r, int(box.sizes[0]), int(box.lows[0])
    anchors = []
    vals = dev.empty((d * r, K, 2), torch.float64)
    poly = isinstance(base, SparsePolynomialOracle)
    for t in range(d):
        rng = np.random.default_rng(streams[t])
        anchors.append(np.stack([np.zeros(d) if zero else rng.random(d) for _ in range(r)]))
    if poly and d * r * d <= 2048:
        # every component's r lines in one launch (line g = t r + i)
        hf, cf = base.device_terms(dev)
        a_all = np.ascontiguousarray(np.concatenate(anchors))
        dev.call("sfft_line_sample_poly_all", dptr(hf), dptr(cf), base.s, d, K, hptr(a_all), r, dptr(vals),
                 ctx="line sampling, all components")
        base.count_samples(d * r * K)  # the oracle's own call audit, as _line_values
    elif poly:
        for t in range(d):
            _line_values(dev, oracle, t, box, anchors[t], t, 0, out=vals[t * r:(t + 1) * r])
    if not poly:
        # the d r K line points built on the device from the d r anchors
        d_anchors = dev.upload(np.ascontiguousarray(np.concatenate(anchors)), asynchronous=True)
        d_pts = dev.empty((d * r * K, d), torch.float64)
        dev.call("sfft_line_points", dptr(d_anchors), d, r, K, dptr(d_pts), ctx="line points, all components")
        order, start, comps, scale = base.host_spec()
        dev.call("sfft_eval_bspline_points", dptr(d_pts), d * r * K, d, len(base.groups), hptr(order),
                 hptr(start), hptr(comps), hptr(scale), dptr(vals), ctx="line sampling, all components")
        base.count_samples(d * r * K)  # the oracle's own call audit, as _line_values
    coefs = dev.empty((d * r, K, 2), torch.float64)
    keep = dev.empty((d * r, K), torch.uint8)
    dev.call("sfft_line_select", dptr(vals), d * r, K, lo, int(cfg.local_sparsity), float(cfg.component_threshold),
             dptr(coefs), dptr(keep), ctx="line selection, all components")
    return ("batched", np.arange(lo, lo + K, dtype=np.int64), keep, r, d)


def _detect_all_collect(dev: Device, launched) -> list[np.ndarray]:
    if isinstance(launched, tuple):  # one (d * r, K) keep buffer
        _, ks, keep, r, d = launched
        raw = dev.download_many(keep)[0].view(np.uint8).reshape(d, r, -1).astype(bool).any(axis=1)
        return [ks[raw[t]] for t in range(d)]
    outs = dev.download_many(*[keep for _, keep in launched])
    comps = []
    for (ks, keep), raw in zip(launched, outs):
        hit = raw.view(np.uint8).reshape(tuple(keep.shape)).astype(bool).any(axis=0)
        comps.append(ks[hit])
    return comps


def detect_component(oracle, t: int, cfg: DetectionConfig, rng: np.random.Generator | None = None):
    """Candidate values of component t from r anchored lines (reference detect.py:215-240)."""
    d = cfg.box.dim
    if not 0 <= t < d:
        raise ValueError(f"component index t must lie in 0..{d - 1}")
    if rng is None:
        rng = np.random.default_rng(np.random.SeedSequence([cfg.rng_seed, t]))
    comp = _detect(get_device(), oracle, t, cfg, rng, t)
    return FrequencyIndexSet(comp[:, None], 1, _presorted=True)


# ---------------------------------------------------------------------------
# the engine

def _tables_cached_only() -> bool:
    """The step preparation builds the per-size tables of the first alias
    chunk's lattices when they are not cached, behind the alias kernel and
    off the host's critical path (a few more lattices than the early exit
    keeps; cold d = 10 runs 0.3 ms faster, `profiles/r02ax_cold_ab.jsonl`).
    SFFT_B200_PREP_TABLES=0: only cached tables there, run_step builds the
    L it uses after the alias read-back."""
    import os
    return os.environ.get("SFFT_B200_PREP_TABLES", "1") == "0"


def _overlap_enabled() -> bool:
    """SFFT_B200_ENGINE_OVERLAP=0 runs every step after its predecessor's
    synchronisation (the A/B of tools/run_configs.py)."""
    import os
    return os.environ.get("SFFT_B200_ENGINE_OVERLAP", "1") != "0"


@dataclass
class _NextStep:
    """Step t+1 started during step t for a guessed prefix count ``cnt``: the
    prefixes gathered with that count, their product with the next
    component, the first lattice-search attempt's alias kernel (pending) and
    the step preparation.  Valid when step t's compaction count equals
    ``cnt``; otherwise discarded (its kernels only wrote their own buffers)."""
    cnt: int
    prefixes: DeviceFreqs
    cand: DeviceFreqs
    pending: object
    guess: object
    prep: object


def _start_next_step(dev: Device, oracle, prefixes: DeviceFreqs | None, pend, cnt: int, comp, t_next: int,
                     tails, d: int, seed_seq, b: int, spread: int) -> "_NextStep | None":
    """Enqueue step t_next up to its first alias kernel without host
    synchronisation.  ``prefixes``: the exact prefix set (step 1), or None
    with ``pend`` (step t's pending compaction) and the guessed count."""
    from . import _native
    from .mr1l import first_chunk, product, speculate_scheme
    torch = dev.torch
    n = cnt * len(comp)
    if n < 1 or cnt < 1:
        return None
    g = speculate_scheme(n, t_next + 1, seed_seq, b)
    if g.primes[0] <= spread:  # build_scheme would not take the guessed attempt
        return None
    if prefixes is None:
        # the compaction's gather with the guessed count, into zeroed rows (a
        # wrong guess leaves valid, if meaningless, frequencies behind)
        _, prev, idx, total, _, _ = pend
        out = dev.zeros((prev.ncomp, cnt), torch.int32)
        dev.call("sfft_gather_rows", dptr(prev.data), prev.n, prev.ncomp, dptr(idx), dptr(total), cnt, dptr(out),
                 cnt, 0, 0, ctx="row gather (next step)")
        prefixes = DeviceFreqs(out, cnt, prev.kmax)
    cand = product(dev, prefixes, comp)
    ms = np.asarray(g.primes, dtype=np.int64)
    words = int(_native.query("sfft_alias_scratch_words", hptr(ms), len(ms)))
    bufs = (dev.empty((max(words, 1),), torch.int32), dev.empty((n,), torch.int64), dev.empty((2,), torch.int32))
    pending = build_scheme(dev, cand, b, seed_seq, box_extent=spread, ctx=f"lattice search, step {t_next}",
                           lazy_streams=True, guess=g, bufs=bufs, defer=True)
    lhi = first_chunk(n, ms)
    prep = prepare_step(dev, oracle, cand, len(tails), ms[:lhi], np.ascontiguousarray(g.z[:lhi].astype(np.int32)),
                        cached_tables_only=_tables_cached_only(), tails=tails, d=d)
    return _NextStep(cnt, prefixes, cand, pending, g, prep)


def sparse_fft(oracle, cfg: DetectionConfig, *, device: Device | None = None,
               group=None, shard: bool | None = None) -> DetectionReport:
    """Reconstruct support and coefficients of a sparse periodic signal
    (reference detect.py:305-423) on the GPU.

    Under torch.distributed (one process per GPU) the units of every MR1L step
    are sharded over the ranks of ``group`` (parallel.py) unless
    ``shard=False``; every rank returns the same, bit-identical report."""
    from .parallel import Shard, run_step_sharded
    start = time.perf_counter()
    sh = Shard(group)
    sharded = sh.active and shard is not False
    if getattr(oracle, "dim", cfg.box.dim) != cfg.box.dim:
        raise ValueError("oracle dimension does not match the search box")
    dev = device or get_device()
    box = cfg.box
    order = cfg.dimension_order
    if order is not None and order != tuple(range(box.dim)):
        oracle = _permute_oracle(oracle, order)
        box = box.permute(order)
        cfg = replace(cfg, box=box, dimension_order=None)
    else:
        order = None

    d = box.dim
    root = np.random.SeedSequence(cfg.rng_seed)
    detect_parent, anchor_parent, lattice_parent = root.spawn(3)
    detect_streams = detect_parent.spawn(d)

    rep = DetectionReport(detected=SparseSpectrum.from_dict({}, dim=d))
    for name in ("component_counts", "prefix_counts", "candidate_counts", "scheme_sizes",
                 "lattice_attempts", "detection_calls", "inversion_calls"):
        setattr(rep, name, [0] * d)
    zero = cfg.mode == "deterministic_zero_anchor"
    extents = (box.highs - box.lows)
    final_rows = np.empty((0, d), dtype=np.int64)
    final_coef = np.empty(0, dtype=np.complex128)
    prefixes: DeviceFreqs | None = None

    hoisted = None
    if _is_device_oracle(oracle) and not isinstance(oracle, NoisyOracle):
        hoisted = _detect_all_launch(dev, oracle, cfg, detect_streams)
    # the anchors' and lattice searches' streams after the line detections are
    # launched (each parent spawns its own children: the order between the
    # parents does not change any stream)
    anchor_streams = anchor_parent.spawn(d)
    lattice_streams = lattice_parent.spawn(d)
    # host work of every step that does not depend on the previous steps,
    # done while the line detections run: the anchors (their own streams) and
    # the first lattice-search attempt's generator of each step
    zero = cfg.mode == "deterministic_zero_anchor"
    all_tails = []
    first_rngs = []
    for t in range(d):
        r_t = 1 if t == d - 1 else cfg.r
        anchor_rng = np.random.default_rng(anchor_streams[t])
        all_tails.append([np.zeros(d - (t + 1)) if zero else anchor_rng.random(d - (t + 1)) for _ in range(r_t)])
        first_rngs.append(first_attempt_rng(lattice_streams[t], cfg.b) if cfg.lattice_kind != "single" else None)
    if hoisted is not None:
        hoisted = _detect_all_collect(dev, hoisted)
    # step t+1 is enqueued during step t, up to its first alias kernel, for
    # a guessed prefix count (this step's, exact for step 1): the compaction,
    # product, lattice search and preparation then follow each other on the
    # device without host synchronisation in between.  Device oracles with
    # hoisted line detections; nothing of it draws from a stream the steps
    # draw from (speculate_scheme uses each attempt's own lazy child).
    # (a replaced scheme builder — the reference tests' seam — sees every step)
    from . import mr1l as _mr1l
    can_start = (hoisted is not None and cfg.lattice_kind != "single" and box.member is None and not sharded
                 and build_scheme is _mr1l.build_scheme and _overlap_enabled())
    nxt = None
    prev_count = None  # the prefix count of the step before the current one

    def start_next(t_next: int, prefixes_exact, pend, cnt):
        if not can_start or t_next >= d:
            return None
        return _start_next_step(dev, oracle, prefixes_exact, pend, cnt, hoisted[t_next], t_next, all_tails[t_next],
                                d, lattice_streams[t_next], cfg.b, int(extents[: t_next + 1].max()))

    for t in range(d):
        t_step = time.perf_counter()
        if hoisted is not None:
            comp = hoisted[t]
        else:
            comp = _detect(dev, oracle, t, cfg, np.random.default_rng(detect_streams[t]), t)
        rep.component_counts[t] = len(comp)
        rep.detection_calls[t] = cfg.r * int(box.sizes[t])
        started, nxt = nxt, None
        if t == 0:
            prefixes = DeviceFreqs.from_host(dev, comp[:, None])
            rep.prefix_counts[0] = rep.candidate_counts[0] = len(comp)
            if d > 1:
                nxt = start_next(1, prefixes, None, prefixes.n)
                rep.step_times.append(time.perf_counter() - t_step)
                continue
            cand = prefixes
        elif started is not None:
            cand = started.cand  # enqueued during the previous step (its count was right)
            rep.candidate_counts[t] = cand.n
        else:
            cand = product(dev, prefixes, comp)
            if box.member is not None and cand.n:
                rows = cand.to_host(dev)
                rows = rows[box.contains_projected(tuple(range(t + 1)), rows)]
                cand = DeviceFreqs.from_host(dev, rows) if len(rows) else DeviceFreqs(cand.data[:, :0], 0, 0)
            rep.candidate_counts[t] = cand.n
        last = t == d - 1
        r_tilde = 1 if last else cfg.r
        s_tilde = cfg.s if last else cfg.local_sparsity
        if cand.n == 0:
            prefixes = cand
            rep.prefix_counts[t] = 0
            rep.step_times.append(time.perf_counter() - t_step)
            continue
        tails = all_tails[t]  # the anchors' own stream (independent of the lattice search)
        if cfg.lattice_kind == "single":
            from .single import single_scheme
            sch = single_scheme(dev, cand)  # CBC (reference detect.py:269-271), no RNG consumed
        else:
            # while the alias kernel runs: buffers, the sampling operands
            # (and the tables, when this step's sizes were seen before)
            prepare = lambda ms, z: prepare_step(dev, oracle, cand, r_tilde, ms, z,  # noqa: E731
                                                 cached_tables_only=_tables_cached_only(), tails=tails, d=d)
            if started is not None:
                sch = started.pending.finish()
                if sch.prep is None and sch.attempts == 1 and sch.z is started.guess.z:
                    sch.prep = started.prep  # made for exactly this attempt's lattices
            else:
                sch = build_scheme(dev, cand, cfg.b, lattice_streams[t], box_extent=int(extents[: t + 1].max()),
                                   ctx=f"lattice search, step {t}", lazy_streams=True, prepare=prepare,
                                   first_rng=first_rngs[t])
        rep.scheme_sizes[t] = sch.total_size
        rep.lattice_attempts[t] = sch.attempts
        rep.inversion_calls[t] = r_tilde * sch.total_size
        if sch.uncovered:
            rep.warnings.append(
                f"step {t}: sampling scheme covers only {cand.n - sch.uncovered}/{cand.n} "
                f"candidates after {sch.attempts} attempts"
            )
        if sharded:
            res = run_step_sharded(dev, oracle, cand, sch, tails, d, cfg.delta, s_tilde, sh, step=t,
                                   prep=sch.prep, need_coef=last)
        else:
            res = run_step(dev, oracle, cand, sch, tails, d, cfg.delta, s_tilde, step=t, prep=sch.prep,
                           device_cap=True)
        if last:
            rows_d, coef_d = compact(dev, cand, res.keep[0], 1, res.coef[0])
            final_rows = rows_d.to_host(dev)
            c = dev.download(coef_d) if coef_d is not None else np.zeros((0, 2))
            final_coef = c[:, 0] + 1j * c[:, 1]
            rep.prefix_counts[t] = len(final_rows)
        else:
            pend = compact_start(dev, cand, res.keep, r_tilde)
            # the next step for as many prefixes as this step had, once the
            # counts have settled (the last two steps' equal, as when the caps
            # bind); the host work hides behind this step's sampling
            settled = prev_count is not None and prev_count == prefixes.n
            nxt = start_next(t + 1, None, pend, prefixes.n) if settled else None
            prev_count = prefixes.n
            if nxt is not None and compact_count(pend) == nxt.cnt:
                prefixes = nxt.prefixes
            else:
                nxt = None
                prefixes, _ = compact_finish(pend)
            rep.prefix_counts[t] = prefixes.n
        rep.step_times.append(time.perf_counter() - t_step)

    if order is not None:
        unperm = np.empty_like(final_rows)
        unperm[:, list(order)] = final_rows
        final_rows = unperm
    rep.detected = SparseSpectrum(final_rows, final_coef, d)
    rep.oracle_calls = sum(rep.detection_calls) + sum(rep.inversion_calls)
    rep.wall_time = time.perf_counter() - start
    return rep


# ---------------------------------------------------------------------------
# planners and bounds (reference detect.py:429-486; closed-form host formulas)

def plan_r(sparsity: int, dims: int, eps: float, lattice_kind: str = "multiple") -> int:
    if sparsity < 1:
        raise ValueError("sparsity must be >= 1")
    if dims < 1:
        raise ValueError("dims must be >= 1")
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    consts = {"multiple": 3.0, "single": 2.0}
    if lattice_kind not in consts:
        raise ValueError("lattice_kind must be 'multiple' or 'single'")
    return math.ceil(2.0 * sparsity * (math.log(consts[lattice_kind]) + math.log(dims)
                                       + math.log(sparsity) - math.log(eps)))


def plan_b(dims: int, eps: float, gamma: float) -> int:
    if dims < 1:
        raise ValueError("dims must be >= 1")
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    if not 0.0 < gamma < 1.0:
        raise ValueError("gamma must lie in (0, 1)")
    return math.ceil((math.log(3.0) + math.log(dims) - math.log(eps)) / abs(math.log(gamma)))


def failure_bound_single_coeff(coeff_magnitudes, delta: float) -> float:
    mags = np.atleast_1d(np.asarray(coeff_magnitudes, dtype=np.float64))
    if not len(mags) or (mags < 0).any() or not np.isfinite(mags).all():
        raise ValueError("coefficient magnitudes must be finite and nonnegative")
    if delta < 0:
        raise ValueError("delta must be >= 0")
    top = float(mags.max())
    if top <= delta:
        raise ValueError("bound inapplicable: no magnitude exceeds delta")
    return 1.0 - (top - delta) / float(mags.sum())


def union_failure_bound(q: float, r: int, sparsity: int, bins: int) -> float:
    if not 0.0 <= q <= 1.0:
        raise ValueError("q must lie in [0, 1]")
    if r < 1:
        raise ValueError("r must be >= 1")
    if sparsity < 0 or bins < 0:
        raise ValueError("counts must be nonnegative")
    return min(1.0, min(sparsity, bins) * q ** r)
