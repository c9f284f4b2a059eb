"""Single rank-1 lattice path (Algorithm 5, ``lattice_kind="single"``) on the
device: the deterministic component-by-component search of reference
construct.py:212-278, and invert_single / eval_on_lattice of transform.py:67-96.

CBC: odd sizes M = |I|, |I|+2, ... are tried in order; for each, component t
gets the smallest z_t in [0, M) that keeps the distinct (t+1)-prefixes of I
pairwise separated.  Candidate values are tested in device batches (one
bitmap per value, atomicOr duplicate detection), so the result — the smallest
workable M and the smallest z_t at every step — is the reference's.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .core import FrequencyIndexSet, Rank1Lattice, SparseSpectrum
from .device import Device, dptr, get_device, hptr
from .mr1l import DeviceFreqs, DeviceScheme, compact, lattice_tables

__all__ = ["cbc_device", "single_scheme", "build_single_lattice_cbc", "invert_single", "eval_on_lattice"]

_SCAN_BUDGET_WORDS = 16 << 20  # bitmap words per batch (64 MB)


def _distinct_prefixes(dev: Device, cand: DeviceFreqs, t1: int) -> DeviceFreqs:
    """np.unique(freqs[:, :t1], axis=0) of a lexicographically sorted set."""
    torch = dev.torch
    flags = dev.empty((max(cand.n, 1),), torch.uint8)
    dev.call("sfft_prefix_flags", dptr(cand.data), cand.n, t1, dptr(flags), ctx="CBC prefixes")
    head = DeviceFreqs(cand.data[:t1], cand.n, cand.kmax)
    if not head.data.is_contiguous():
        head.data = head.data.contiguous()
    rows, _ = compact(dev, head, flags, 1)
    return rows


def _first_separating(dev: Device, prefix_res, col, n: int, m: int) -> int | None:
    """Smallest z in [0, m) with (prefix_res + col * z) mod m pairwise distinct."""
    torch = dev.torch
    words = (m + 31) // 32
    Z = int(max(1, min(4096, _SCAN_BUDGET_WORDS // words, m)))
    bits = dev.empty((Z * words,), torch.int32)
    dup = dev.empty((Z,), torch.int32)
    for z0 in range(0, m, Z):
        zc = min(Z, m - z0)
        dev.call("sfft_cbc_scan", dptr(prefix_res), dptr(col), n, m, z0, zc, dptr(bits), words, dptr(dup),
                 ctx="CBC scan")
        ok = np.flatnonzero(dev.download(dup[:zc]) == 0)
        if len(ok):
            return z0 + int(ok[0])
    return None


def cbc_device(dev: Device, cand: DeviceFreqs) -> tuple[np.ndarray, int]:
    """(z, M) of build_single_lattice_cbc for a sorted device candidate set."""
    torch = dev.torch
    n, d = cand.n, cand.ncomp
    if n < 1:
        raise ValueError("cannot build a lattice for an empty set")
    if n == 1:
        return np.zeros(d, dtype=np.int64), 1
    prefixes = {t: _distinct_prefixes(dev, cand, t + 1) for t in range(1, d)}
    zero_res = dev.zeros((n,), torch.int64)
    m = n if n % 2 == 1 else n + 1
    while True:
        z = np.zeros(d, dtype=np.int64)
        z[0] = 1 % m
        ok = True
        if d == 1:
            # distinct k mod m: the scan at the single value z = 1
            words = (m + 31) // 32
            bits = dev.empty((words,), torch.int32)
            dup = dev.empty((1,), torch.int32)
            dev.call("sfft_cbc_scan", dptr(zero_res), dptr(cand.data), n, m, 1, 1, dptr(bits), words,
                     dptr(dup), ctx="CBC scan")
            ok = int(dev.download(dup)[0]) == 0
        else:
            for t in range(1, d):
                rows = prefixes[t]
                nt = rows.n
                res = dev.empty((max(nt, 1),), torch.int64)
                ms = np.array([m], dtype=np.int64)
                zs = np.ascontiguousarray(z[:t].astype(np.int32)).reshape(1, t)
                head = rows.data[:t]
                dev.call("sfft_residues", dptr(head), nt, t, rows.kmax, hptr(ms), hptr(zs), 1, dptr(res),
                         ctx="CBC prefix residues")
                zt = _first_separating(dev, res, rows.data[t], nt, m)
                if zt is None:
                    ok = False
                    break
                z[t] = zt
        if ok:
            return z, m
        m += 2


def single_scheme(dev: Device, cand: DeviceFreqs) -> DeviceScheme:
    """The single CBC lattice as a one-lattice scheme (every candidate on it)."""
    z, m = cbc_device(dev, cand)
    masks = dev.torch.ones((cand.n,), dtype=dev.torch.int64, device=dev.device)
    return DeviceScheme([int(m)], z.reshape(1, -1), 1, masks, 1, 0)


def build_single_lattice_cbc(I: FrequencyIndexSet) -> Rank1Lattice:
    """Deterministic single-lattice search (reference construct.py:254-278)."""
    if not len(I):
        raise ValueError("cannot build a lattice for an empty set")
    dev = get_device()
    z, m = cbc_device(dev, DeviceFreqs.from_host(dev, I.freqs))
    return Rank1Lattice(z, m)


def invert_single(samples, I: FrequencyIndexSet) -> SparseSpectrum:
    """Coefficients of every k in I from one lattice: X[k.z mod M] / M
    (reference transform.py:83-96; aliased k get the sum of their collisions)."""
    lat = samples.lattice
    if I.dim != lat.dim:
        raise ValueError("dimension mismatch between samples and frequency set")
    dev = get_device()
    torch = dev.torch
    n = len(I)
    if n == 0:
        return SparseSpectrum(I.freqs, np.zeros(0, dtype=np.complex128), I.dim)
    ms = np.array([lat.m], dtype=np.int64)
    zs = np.ascontiguousarray(lat.z.astype(np.int32)).reshape(1, -1)
    tabs = lattice_tables(dev, ms, zs, ctx="invert_single tables")
    buf = dev.zeros((1, tabs.P, 2), torch.float64)
    v = np.ascontiguousarray(np.stack([samples.values.real, samples.values.imag], axis=1))
    with torch.cuda.stream(dev.stream):
        buf[0, : lat.m].copy_(torch.from_numpy(v))
    dev.call("sfft_finish_samples", hptr(ms), 1, 1, dptr(tabs.chirp), dptr(buf), tabs.P, 0, 0, 0, 0, 0,
             ctx="invert_single pre-chirp")
    dev.call("sfft_bluestein", hptr(ms), 1, 1, tabs.P, dptr(tabs.ftab), dptr(tabs.bhat), dptr(tabs.chirp),
             dptr(buf), 0, 0, ctx="invert_single FFT")
    cand = DeviceFreqs.from_host(dev, I.freqs)
    masks = torch.ones((n,), dtype=torch.int64, device=dev.device)
    coef = dev.empty((1, n, 2), torch.float64)
    keep = dev.empty((1, n), torch.uint8)
    counts = dev.zeros((1,), torch.int32)
    dev.call("sfft_gather_select", dptr(cand.data), n, I.dim, cand.kmax, hptr(ms), hptr(zs), 1, dptr(masks),
             dptr(buf), tabs.P, 1, 0, 0.0, dptr(coef), dptr(keep), dptr(counts), ctx="invert_single gather")
    c = dev.download(coef[0])
    return SparseSpectrum(I.freqs, c[:, 0] + 1j * c[:, 1], I.dim)


def eval_on_lattice(spectrum: SparseSpectrum, lat: Rank1Lattice):
    """Sparse polynomial at all lattice nodes by one inverse DFT of the
    residue-scattered coefficients (reference transform.py:67-80)."""
    from .api import LatticeSamples
    if spectrum.dim != lat.dim:
        raise ValueError("dimension mismatch between spectrum and lattice")
    dev = get_device()
    torch = dev.torch
    ms = np.array([lat.m], dtype=np.int64)
    zs = np.ascontiguousarray(lat.z.astype(np.int32)).reshape(1, -1)
    tabs = lattice_tables(dev, ms, zs, ctx="eval_on_lattice tables")
    buf = dev.zeros((1, tabs.P, 2), torch.float64)
    if len(spectrum):
        cand = DeviceFreqs.from_host(dev, spectrum.freqs)
        cf = dev.upload(np.ascontiguousarray(np.stack([spectrum.coeffs.real, spectrum.coeffs.imag], axis=1)))
        dev.call("sfft_scatter_residues", dptr(cand.data), cand.n, lat.dim, lat.m, hptr(zs), dptr(cf), dptr(buf),
                 ctx="eval_on_lattice scatter")
    # M * ifft(acc) = conj(fft(conj(acc)))
    dev.call("sfft_cscale", dptr(buf), lat.m, 1.0, 1, ctx="eval_on_lattice conj")
    dev.call("sfft_finish_samples", hptr(ms), 1, 1, dptr(tabs.chirp), dptr(buf), tabs.P, 0, 0, 0, 0, 0,
             ctx="eval_on_lattice pre-chirp")
    dev.call("sfft_bluestein", hptr(ms), 1, 1, tabs.P, dptr(tabs.ftab), dptr(tabs.bhat), dptr(tabs.chirp),
             dptr(buf), 0, 0, ctx="eval_on_lattice DFT")
    dev.call("sfft_cscale", dptr(buf), lat.m, 1.0, 1, ctx="eval_on_lattice conj")
    out = dev.download(buf[0, : lat.m])
    return LatticeSamples(lat, out[:, 0] + 1j * out[:, 1])
