"""Sampling oracles, signal generators and error metrics (mirror of the
reference's testbed.py public API).

Two kinds of oracle reach the engine:

* **device-oracle descriptors** — :class:`SparsePolynomialOracle`,
  :class:`BSplineOracle` and :class:`NoisyOracle` / :class:`RelativeNoisyOracle`
  wrapping one of them.  Their samples at lattice nodes are computed by the
  CUDA sampling kernels (K1) and never leave the device.
* **host callbacks** — :class:`SignalOracle` around an arbitrary Python
  function (reference testbed.py:40-73).  Lattice nodes are generated on the
  device, handed to the callback, and its values are uploaded again; the FFT,
  alias and selection stages still run on the GPU.

Calling any oracle on an explicit (n, d) point array evaluates it on the
device (descriptors) or through the callback.
"""

from __future__ import annotations

import math
import threading
from functools import lru_cache
from typing import Callable, Sequence

import numpy as np

from .core import SparseSpectrum, as_frequency_rows
from .device import dptr, get_device, hptr

__all__ = [
    "SignalOracle",
    "SparsePolynomialOracle",
    "BSplineOracle",
    "NoisyOracle",
    "RelativeNoisyOracle",
    "gen_random_sparse_poly",
    "bspline_test_function",
    "bspline_exact_coefficient",
    "bspline_exact_coefficients",
    "bspline_l2_constant",
    "bspline_norm_sq",
    "sigma_for_snr",
    "relative_l2_error",
    "relative_spectrum_l2_error",
    "DEFAULT_BSPLINE_GROUPS",
]


def _as_points(points, dim: int) -> np.ndarray:
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[None, :]
    if pts.ndim != 2 or pts.shape[1] != dim:
        raise ValueError(f"expected points of shape (n, {dim}), got {pts.shape}")
    return np.ascontiguousarray(pts)


class _Counter:
    """Lock-protected exact sample counter (reference testbed.py:53, 71-72)."""

    def __init__(self):
        self._lock = threading.Lock()
        self._n = 0

    def add(self, n: int) -> None:
        with self._lock:
            self._n += int(n)

    @property
    def value(self) -> int:
        return self._n


class SignalOracle:
    """Host-callback oracle: ``fn`` maps an (n, d) float64 array to n complex values."""

    def __init__(self, dim: int, fn: Callable[[np.ndarray], np.ndarray], concurrency_safe: bool = True):
        self.dim = int(dim)
        self.concurrency_safe = bool(concurrency_safe)
        self._fn = fn
        self._counter = _Counter()

    @property
    def call_count(self) -> int:
        return self._counter.value

    def count_samples(self, n: int) -> None:
        self._counter.add(n)

    def __call__(self, points) -> np.ndarray:
        pts = _as_points(points, self.dim)
        vals = np.asarray(self._fn(pts), dtype=np.complex128)
        if vals.shape != (len(pts),):
            raise ValueError(f"oracle function returned shape {vals.shape}, expected ({len(pts)},)")
        self._counter.add(len(pts))
        return vals


class _DeviceOracle:
    """Common part of the device-oracle descriptors."""

    dim: int
    concurrency_safe = True

    def __init__(self):
        self._counter = _Counter()

    @property
    def call_count(self) -> int:
        return self._counter.value

    def count_samples(self, n: int) -> None:
        self._counter.add(n)

    def _eval_device(self, dev, d_pts, n: int):
        raise NotImplementedError

    def __call__(self, points) -> np.ndarray:
        pts = _as_points(points, self.dim)
        dev = get_device()
        torch = dev.torch
        d_pts = dev.upload(pts)
        out = self._eval_device(dev, d_pts, len(pts))
        vals = dev.download(out)
        self._counter.add(len(pts))
        return vals[:, 0] + 1j * vals[:, 1]


class SparsePolynomialOracle(_DeviceOracle):
    """p(x) = sum_h c_h e^{2 pi i h.x} (reference testbed.py:116-127) as a
    device descriptor: terms are uploaded once per device (component-major
    int32 frequencies, complex128 coefficients)."""

    kind = "poly"

    def __init__(self, freqs, coeffs, dim: int | None = None, *, _counter=None):
        super().__init__()
        if _counter is not None:
            self._counter = _counter
        rows = as_frequency_rows(freqs, dim)
        self.dim = rows.shape[1]
        self.freqs = rows
        self.coeffs = np.asarray(coeffs, dtype=np.complex128).reshape(-1)
        if self.coeffs.shape != (rows.shape[0],):
            raise ValueError("coefficients must align one-to-one with frequencies")
        self._dev_cache: dict[int, tuple] = {}

    @property
    def s(self) -> int:
        return self.freqs.shape[0]

    @property
    def max_abs_freq(self) -> int:
        return int(np.abs(self.freqs).max()) if self.freqs.size else 0

    def permuted(self, order: Sequence[int]) -> "SparsePolynomialOracle":
        """The oracle seen through slot t <- component order[t] (detect.py:243-254)."""
        return SparsePolynomialOracle(self.freqs[:, list(order)], self.coeffs, _counter=self._counter)

    def device_terms(self, dev):
        got = self._dev_cache.get(dev.index)
        if got is None:
            torch = dev.torch
            host = getattr(self, "_pinned_terms", None)
            if host is None:
                # packed once into pinned host memory: every (re-)upload is an
                # asynchronous DMA on the engine stream
                hf = np.ascontiguousarray(self.freqs.T.astype(np.int32))
                cf = np.ascontiguousarray(np.stack([self.coeffs.real, self.coeffs.imag], axis=1))
                host = (torch.from_numpy(hf).pin_memory(), torch.from_numpy(cf).pin_memory())
                self._pinned_terms = host
            # asynchronous DMA from the persistent pinned copy (one library
            # cudaMemcpyAsync each, no framework stream switch)
            from . import _native
            got = tuple(torch.empty(h.shape, dtype=h.dtype, device=dev.device) for h in host)
            for g_, h in zip(got, host):
                if h.numel():
                    _native.call("sfft_copy_async", g_.data_ptr(), h.data_ptr(), h.numel() * h.element_size(),
                                 dev.sh, ctx="oracle terms")
            self._dev_cache[dev.index] = got
        return got

    def _eval_device(self, dev, d_pts, n: int):
        hf, cf = self.device_terms(dev)
        out = dev.empty((n, 2), dev.torch.float64)
        dev.call("sfft_eval_poly_points", dptr(d_pts), n, self.dim, dptr(hf), dptr(cf), self.s,
                 dptr(out), ctx="polynomial oracle")
        return out


# ---------------------------------------------------------------------------
# B-spline test function (reference testbed.py:188-290)

#: (spline order, 0-based components) of the reference's fixed 10-D function
DEFAULT_BSPLINE_GROUPS: tuple[tuple[int, tuple[int, ...]], ...] = (
    (2, (0, 2, 7)),
    (4, (1, 4, 5, 9)),
    (6, (3, 6, 8)),
)


@lru_cache(maxsize=None)
def bspline_l2_constant(m: int) -> float:
    """C_m with ||C_m * periodised B_m||_2 = 1 (reference testbed.py:198-212)."""
    if m < 1:
        raise ValueError("spline order must be >= 1")
    k = np.arange(1, 200_001)
    return float(1.0 / np.sqrt(1.0 + 2.0 * np.sum(np.sinc(k / m) ** (2 * m))))


def _normalise_groups(groups, dim: int) -> tuple[tuple[int, tuple[int, ...]], ...]:
    out = []
    for m, comps in groups:
        comps = tuple(int(c) for c in comps)
        if any(c < 0 or c >= dim for c in comps):
            raise ValueError("B-spline group component out of range")
        out.append((int(m), comps))
    return tuple(out)


class BSplineOracle(_DeviceOracle):
    """f(x) = sum_g prod_{t in A_g} C_m m B_m(m frac(x_t)) with cardinal
    B-splines B_m of order m (reference testbed.py:219-244)."""

    kind = "bspline"

    def __init__(self, groups=DEFAULT_BSPLINE_GROUPS, dim: int = 10, *, _counter=None):
        super().__init__()
        if _counter is not None:
            self._counter = _counter
        self.dim = int(dim)
        self.groups = _normalise_groups(groups, self.dim)
        if len(self.groups) > 8 or any(not 1 <= m <= 7 for m, _ in self.groups):
            raise ValueError("at most 8 groups of spline order 1..7 are supported")

    def permuted(self, order: Sequence[int]) -> "BSplineOracle":
        slot_of = {int(c): t for t, c in enumerate(order)}
        groups = tuple((m, tuple(slot_of[c] for c in comps)) for m, comps in self.groups)
        return BSplineOracle(groups, self.dim, _counter=self._counter)

    def host_spec(self):
        got = self.__dict__.get("_host_spec")
        if got is None:
            got = self.__dict__["_host_spec"] = self._make_host_spec()
        return got

    def _make_host_spec(self):
        order = np.array([m for m, _ in self.groups], dtype=np.int32)
        start = np.zeros(len(self.groups) + 1, dtype=np.int32)
        comps = []
        for g, (m, cs) in enumerate(self.groups):
            comps.extend(cs)
            start[g + 1] = len(comps)
        comps = np.array(comps if comps else [0], dtype=np.int32)
        scale = np.array([bspline_l2_constant(m) * m for m, _ in self.groups] or [0.0], dtype=np.float64)
        return order if len(order) else np.zeros(1, np.int32), start, comps, scale

    def _eval_device(self, dev, d_pts, n: int):
        order, start, comps, scale = self.host_spec()
        out = dev.empty((n, 2), dev.torch.float64)
        dev.call("sfft_eval_bspline_points", dptr(d_pts), n, self.dim, len(self.groups),
                 hptr(order), hptr(start), hptr(comps), hptr(scale), dptr(out), ctx="B-spline oracle")
        return out

    # exact Fourier data ------------------------------------------------
    def exact_coefficients(self, freqs) -> np.ndarray:
        return bspline_exact_coefficients(freqs, self.groups, self.dim)

    def norm_sq(self) -> float:
        return bspline_norm_sq(self.groups)


def bspline_test_function(groups=None) -> BSplineOracle:
    """The 10-D B-spline test signal; ``groups`` overrides the reference's fixed
    partition (BASELINE config 4 uses a seed-chosen 3/4/3 partition)."""
    return BSplineOracle(DEFAULT_BSPLINE_GROUPS if groups is None else groups, 10)


def bspline_exact_coefficients(freqs, groups=None, dim: int = 10) -> np.ndarray:
    """Closed-form Fourier coefficients (reference testbed.py:247-265)."""
    groups = DEFAULT_BSPLINE_GROUPS if groups is None else groups
    rows = np.asarray(freqs, dtype=np.int64)
    if rows.ndim == 1:
        rows = rows[None, :]
    if rows.shape[1] != dim:
        raise ValueError(f"frequencies must have {dim} components")
    out = np.zeros(len(rows), dtype=np.complex128)
    for m, comps in groups:
        others = [t for t in range(dim) if t not in comps]
        live = (rows[:, others] == 0).all(axis=1)
        if not live.any():
            continue
        k = rows[np.ix_(np.flatnonzero(live), list(comps))]
        fac = bspline_l2_constant(m) * np.sinc(k / m) ** m * np.where(k % 2 == 0, 1.0, -1.0)
        out[live] += fac.prod(axis=1)
    return out


def bspline_exact_coefficient(freq, groups=None) -> complex:
    return complex(bspline_exact_coefficients(np.asarray(freq).reshape(1, -1), groups)[0])


def bspline_norm_sq(groups=None) -> float:
    """||f||_2^2: unit-norm terms plus cross terms of 1-D means (testbed.py:276-290)."""
    groups = DEFAULT_BSPLINE_GROUPS if groups is None else groups
    means = [bspline_l2_constant(m) ** len(comps) for m, comps in groups]
    cross = sum(means[a] * means[b] for a in range(len(means)) for b in range(a + 1, len(means)))
    return float(len(means) + 2.0 * cross)


# ---------------------------------------------------------------------------
# noise

class NoisyOracle:
    """Inner oracle plus complex Gaussian noise of std sigma (reference
    testbed.py:76-106): each call draws ``standard_normal((n, 2))`` from a
    dedicated numpy stream, in call order, so a run is bit-compatible with the
    reference's noise realisation.  The draw is host-side; the addition runs on
    the device for device-oracle inners."""

    kind = "noisy"

    def __init__(self, inner, sigma: float, seed=0, *, device_rng: bool = False):
        """``device_rng=True`` generates the noise on the GPU (Philox keyed by
        the seed and the call index) instead of drawing the numpy stream: the
        same distribution, a different realisation, no host RNG or upload —
        for runs whose sample counts make the host stream the bottleneck
        (BASELINE config 3: 1.4e9 samples)."""
        if sigma < 0:
            raise ValueError("sigma must be >= 0")
        self.inner = inner
        self.sigma = float(sigma)
        self.dim = inner.dim
        self.concurrency_safe = getattr(inner, "concurrency_safe", True)
        self._rng = np.random.default_rng(seed)
        self._lock = threading.Lock()
        self._counter = _Counter()
        self.device_rng = bool(device_rng)
        ss = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
        self.device_key = int(ss.generate_state(1, np.uint64)[0])
        self._next_call = 0

    def reserve_calls(self, n: int) -> int:
        """Index of the first of the next n oracle calls (device-noise counter)."""
        with self._lock:
            base = self._next_call
            self._next_call += int(n)
        return base

    @property
    def call_count(self) -> int:
        return self._counter.value

    def count_samples(self, n: int) -> None:
        self._counter.add(n)
        if hasattr(self.inner, "count_samples"):
            self.inner.count_samples(n)

    def draw(self, n: int) -> np.ndarray:
        """(n, 2) standard normals of the next call (real, imag parts)."""
        with self._lock:
            return self._rng.standard_normal((n, 2))

    def scale_for(self, clean_norm2: float, n: int) -> float:
        """Multiplier of the (re, im) normals for one call."""
        return self.sigma / math.sqrt(2.0)

    def needs_norm(self) -> bool:
        return False

    def permuted(self, order):
        view = object.__new__(type(self))
        view.__dict__.update(self.__dict__)
        view.inner = self.inner.permuted(order) if hasattr(self.inner, "permuted") else self.inner
        return view

    def __call__(self, points) -> np.ndarray:
        vals = self.inner(points)
        n = len(vals)
        e = self.draw(n)
        self._counter.add(n)
        sc = self.scale_for(float(np.sum(np.abs(vals) ** 2)), n)
        return vals + sc * (e @ np.array([1.0, 1.0j]))


class RelativeNoisyOracle(NoisyOracle):
    """Noise whose l2 norm is ``rel`` times the noise-free sample vector's norm
    in expectation, per oracle call (BASELINE config 3: rel = 1e-2):
    sigma_call = rel * ||p(X)||_2 / sqrt(n)."""

    def __init__(self, inner, rel: float = 1e-2, seed=0, *, device_rng: bool = False):
        super().__init__(inner, 0.0, seed, device_rng=device_rng)
        if rel < 0:
            raise ValueError("rel must be >= 0")
        self.rel = float(rel)

    def needs_norm(self) -> bool:
        return True

    def scale_for(self, clean_norm2: float, n: int) -> float:
        sigma = self.rel * math.sqrt(clean_norm2) / math.sqrt(max(n, 1))
        return sigma / math.sqrt(2.0)


def sigma_for_snr(sparsity: int, snr_db: float) -> float:
    """sigma = sqrt(s) / sqrt(10^(SNR_dB / 10)) (reference testbed.py:109-113)."""
    if sparsity < 1:
        raise ValueError("sparsity must be >= 1")
    return float(np.sqrt(sparsity) / np.sqrt(10.0 ** (snr_db / 10.0)))


# ---------------------------------------------------------------------------
# generators

def gen_random_sparse_poly(dims: int, freq_limit: int, sparsity: int, coeff_model: str = "box",
                           seed=0, *, min_magnitude: float = 1e-6, magnitude_range=(1.0, 2.0)):
    """Random sparse trigonometric polynomial and its device oracle.

    Same draw sequence as the reference (testbed.py:130-182): frequencies
    uniform without replacement on [-N, N]^d by batched rejection, then
    coefficients.  ``coeff_model``: ``box`` (Re, Im ~ U[-1, 1), redrawn while
    |c| < ``min_magnitude``; the reference fixes 1e-6, BASELINE configs 0/2 use
    1e-3), ``unit_modulus`` (e^{2 pi i phi}), or ``polar`` (phase U[0, 1),
    magnitude U[magnitude_range]; BASELINE config 3).
    """
    if dims < 1:
        raise ValueError("dims must be >= 1")
    if freq_limit < 0:
        raise ValueError("freq_limit must be >= 0")
    if sparsity < 1:
        raise ValueError("sparsity must be >= 1")
    if sparsity > (2 * freq_limit + 1) ** dims:
        raise ValueError(f"sparsity {sparsity} exceeds the grid cardinality {(2 * freq_limit + 1) ** dims}")
    rng = np.random.default_rng(seed)
    picked: list[tuple[int, ...]] = []
    seen: set[tuple[int, ...]] = set()
    while len(picked) < sparsity:
        block = rng.integers(-freq_limit, freq_limit + 1, size=(max(sparsity, 64), dims))
        for row in map(tuple, block.tolist()):
            if row in seen:
                continue
            seen.add(row)
            picked.append(row)
            if len(picked) == sparsity:
                break
    freqs = np.asarray(picked, dtype=np.int64)
    if coeff_model == "box":
        coeffs = rng.uniform(-1, 1, sparsity) + 1j * rng.uniform(-1, 1, sparsity)
        low = np.abs(coeffs) < min_magnitude
        while low.any():
            k = int(low.sum())
            coeffs[low] = rng.uniform(-1, 1, k) + 1j * rng.uniform(-1, 1, k)
            low = np.abs(coeffs) < min_magnitude
    elif coeff_model == "unit_modulus":
        coeffs = np.exp(2j * np.pi * rng.random(sparsity))
    elif coeff_model == "polar":
        phase = rng.random(sparsity)
        mag = rng.uniform(magnitude_range[0], magnitude_range[1], sparsity)
        coeffs = mag * np.exp(2j * np.pi * phase)
    else:
        raise ValueError("coeff_model must be 'box', 'unit_modulus' or 'polar'")
    spectrum = SparseSpectrum(freqs, coeffs, dims)
    return spectrum, SparsePolynomialOracle(spectrum.freqs, spectrum.coeffs, dims)


# ---------------------------------------------------------------------------
# metrics (reference testbed.py:296-337)

def relative_l2_error(detected: SparseSpectrum, exact_coefficients, norm_sq: float) -> float:
    if not norm_sq > 0:
        raise ValueError("norm_sq must be positive")
    if not len(detected):
        return 1.0
    truth = np.asarray(exact_coefficients(detected.freqs), dtype=np.complex128)
    rad = norm_sq - float(np.sum(np.abs(truth) ** 2)) + float(np.sum(np.abs(detected.coeffs - truth) ** 2))
    if rad < -1e-12 * max(1.0, norm_sq):
        raise ValueError(f"negative error radicand {rad}: inconsistent inputs")
    return float(np.sqrt(max(rad, 0.0) / norm_sq))


def relative_spectrum_l2_error(detected: SparseSpectrum, truth: SparseSpectrum) -> float:
    if not len(truth):
        raise ValueError("truth spectrum must be nonempty")
    a, b = truth.as_dict(), detected.as_dict()
    err = sum(abs(b.get(k, 0.0) - a.get(k, 0.0)) ** 2 for k in a.keys() | b.keys())
    return float(np.sqrt(err / truth.energy()))
