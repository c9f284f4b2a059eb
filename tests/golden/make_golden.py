"""Generate golden vectors from the UNMODIFIED reference (run in the build
container, where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The fixtures pin the CPU oracle (oracle/sfft_oracle.py) and are the
known answers of the GPU parity tests; nothing at test time reads
/root/reference.  Inputs come from paper_1711_05152_b200.workloads (pure
numpy generators with the reference's draw sequences).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import sfft  # noqa: E402  (the reference)
import sfft.testbed as ref_testbed  # noqa: E402
from sfft.construct import _alias_free_mask  # noqa: E402
from sfft.detect import _select  # noqa: E402

from paper_1711_05152_b200 import workloads  # noqa: E402


def _poly_signal(freqs, coeffs):
    spec = sfft.SparseSpectrum(freqs, coeffs)
    return sfft.SignalOracle(spec.dim, ref_testbed._poly_oracle_fn(spec.freqs, spec.coeffs))


class _BigBox(sfft.SearchBox):
    """Reference SearchBox without the u64 cardinality guard."""

    def __init__(self, lows, highs, member=None):
        from sfft.lattice import _freeze
        self._lows = _freeze(np.asarray(lows, dtype=np.int64))
        self._highs = _freeze(np.asarray(highs, dtype=np.int64))
        self._member = member

    @classmethod
    def centered(cls, dim, n):
        return cls([-n] * dim, [n] * dim)

    def permute(self, order):
        return _BigBox(self._lows[list(order)], self._highs[list(order)], None)


def pack_masks(masks) -> np.ndarray:
    words = np.zeros(len(masks[0]), dtype=np.uint64)
    for l, mk in enumerate(masks):
        words |= np.asarray(mk, dtype=np.uint64) << np.uint64(l)
    return words


def residues_fixture(out):
    rng = np.random.default_rng(101)
    freqs = rng.integers(-50, 51, size=(300, 6))
    big = np.array([[2**31 - 1, -(2**31 - 1), 5, 0, -7, 2**30], [-(2**31 - 1), 2**31 - 1, 3, 1, 1, 1]])
    freqs = np.vstack([freqs, big]).astype(np.int64)
    ms = np.array([7, 13, 601, 1009, 2**31 - 1], dtype=np.int64)
    zs = np.stack([rng.integers(0, m, size=6, dtype=np.int64) for m in ms])
    res = np.stack([sfft.residues(freqs, z, m) for z, m in zip(zs, ms)])
    masks = np.stack([_alias_free_mask(freqs, z, m) for z, m in zip(zs, ms[:4])])
    nodes = sfft.lattice_nodes(sfft.Rank1Lattice(zs[3], ms[3]))
    out.update(res_freqs=freqs, res_ms=ms, res_zs=zs, res_values=res, res_masks=masks,
               nodes_1009=nodes[:64], nodes_z=zs[3])


def primes_fixture(out):
    I = sfft.FrequencyIndexSet(np.array([[0, 0], [40, 1], [-40, 2], [3, -40]]))
    out["primes_small"] = np.array(sfft.candidate_primes(I, 2 * (len(I) - 1), 6))
    rng = np.random.default_rng(5)
    J = sfft.FrequencyIndexSet(rng.integers(-32, 33, size=(5000, 10)))
    out["primes_5000"] = np.array(sfft.candidate_primes(J, 2 * (len(J) - 1), 19))
    out["lmax_pins"] = np.array([sfft.MLConfig().max_lattices(n) for n in (1, 2, 1000, 65000, 100000, 650000)])


def scheme_fixture(out):
    """MR1L step on a config-1-shaped instance (|J| = 3000, 60 nonzero)."""
    wl = workloads.config1(seed=7, n=3000, nnz=60)
    J = sfft.FrequencyIndexSet(wl.cand)
    scheme, attempts = sfft.build_multiple_lattice_with_retries(
        J, sfft.MLConfig(), wl.b, np.random.SeedSequence(wl.lattice_seed))
    oracle = _poly_signal(wl.oracle.freqs, wl.oracle.coeffs)
    samples = [sfft.LatticeSamples(lat, oracle(sfft.lattice_nodes(lat))) for lat in scheme.lattices]
    spec = sfft.invert_multiple(samples, scheme)
    sel_f, sel_c = _select(spec.freqs, spec.coeffs, len(J), wl.delta)
    out.update(step_cand=wl.cand.astype(np.int16), step_hf=wl.oracle.freqs, step_hc=wl.oracle.coeffs,
               step_seed=np.array([wl.lattice_seed], dtype=np.uint64), step_b=np.array([wl.b]),
               step_ms=np.array([lat.m for lat in scheme.lattices]),
               step_zs=np.stack([lat.z for lat in scheme.lattices]),
               step_masks=pack_masks(scheme.recon_masks), step_attempts=np.array([attempts]),
               step_coef=spec.coeffs, step_cov_freqs=spec.freqs.astype(np.int16),
               step_sel=sel_f.astype(np.int16), step_sel_coef=sel_c,
               step_first_samples=samples[0].values[:256])


def run_fixture(out, key, oracle, cfg, truth=None):
    rep = sfft.sparse_fft(oracle, cfg)
    out[f"{key}_freqs"] = rep.detected.freqs
    out[f"{key}_coef"] = rep.detected.coeffs
    out[f"{key}_counts"] = np.array([rep.candidate_counts, rep.prefix_counts, rep.component_counts,
                                     rep.scheme_sizes, rep.lattice_attempts, rep.inversion_calls])
    out[f"{key}_calls"] = np.array([rep.oracle_calls])
    print(f"{key}: detected {len(rep.detected)} calls {rep.oracle_calls} wall {rep.wall_time:.2f}s")
    if truth is not None:
        out[f"{key}_err"] = np.array([sfft.relative_spectrum_l2_error(rep.detected, truth)])


def runs_fixture(out):
    wl = workloads.config0()
    out.update(cfg0_hf=wl.truth.freqs, cfg0_hc=wl.truth.coeffs, cfg0_seed=np.array([wl.cfg.rng_seed], np.uint64))
    cfg = sfft.DetectionConfig(box=sfft.SearchBox.centered(5, 16), delta=1e-12, s=100, r=2, b=10,
                               rng_seed=wl.cfg.rng_seed)
    truth = sfft.SparseSpectrum(wl.truth.freqs, wl.truth.coeffs)
    run_fixture(out, "cfg0", _poly_signal(wl.truth.freqs, wl.truth.coeffs), cfg, truth)

    # small edge-case runs: caps binding, zero anchor, dimension order, 1-D, noisy
    rng = np.random.default_rng(42)
    truth, _ = sfft.gen_random_sparse_poly(3, 6, 25, "box", seed=rng)
    out.update(cap_hf=truth.freqs, cap_hc=truth.coeffs)
    run_fixture(out, "cap", _poly_signal(truth.freqs, truth.coeffs),
                sfft.DetectionConfig(box=sfft.SearchBox.centered(3, 6), delta=1e-12, s=10, s_local=12, r=2,
                                     b=5, rng_seed=7))
    rng = np.random.default_rng(47)
    freqs = np.unique(rng.integers(-5, 6, size=(12, 3)), axis=0)
    coeffs = rng.uniform(0.5, 2.0, size=len(freqs))
    out.update(zero_hf=freqs, zero_hc=coeffs.astype(np.complex128))
    run_fixture(out, "zero", _poly_signal(freqs, coeffs),
                sfft.DetectionConfig(box=sfft.SearchBox.centered(3, 5), delta=1e-12, s=len(freqs), r=1, b=10,
                                     mode="deterministic_zero_anchor"))
    rng = np.random.default_rng(46)
    truth, _ = sfft.gen_random_sparse_poly(3, 6, 8, "box", seed=rng)
    out.update(perm_hf=truth.freqs, perm_hc=truth.coeffs)
    run_fixture(out, "perm", _poly_signal(truth.freqs, truth.coeffs),
                sfft.DetectionConfig(box=sfft.SearchBox.centered(3, 6), delta=1e-12, s=8, r=1, b=10, rng_seed=11,
                                     dimension_order=(2, 0, 1)))
    out.update(one_hf=np.array([[-3], [0], [4]]), one_hc=np.array([1.0, 2.0, 3.0], dtype=np.complex128))
    run_fixture(out, "one", _poly_signal(np.array([[-3], [0], [4]]), np.array([1.0, 2.0, 3.0])),
                sfft.DetectionConfig(box=sfft.SearchBox.centered(1, 5), delta=1e-12, s=3, b=5))
    # noisy (reference NoisyOracle, fixed sigma, numpy noise stream)
    truth, _ = sfft.gen_random_sparse_poly(4, 8, 20, "unit_modulus", seed=np.random.default_rng(9))
    out.update(noisy_hf=truth.freqs, noisy_hc=truth.coeffs)
    noisy = sfft.NoisyOracle(_poly_signal(truth.freqs, truth.coeffs), sfft.sigma_for_snr(20, 30.0), seed=123)
    run_fixture(out, "noisy", noisy,
                sfft.DetectionConfig(box=sfft.SearchBox.centered(4, 8), delta=0.3, s=20, r=3, b=10, rng_seed=5))
    # B-spline (permuted partition, small N, guard bypass)
    groups = workloads.bspline_partition(np.random.SeedSequence([0, 4, 0]).spawn(3)[0])
    out["bs_groups"] = np.array([[m] + list(c) + [-1] * (4 - len(c)) for m, c in groups])
    saved = ref_testbed._BSPLINE_GROUPS
    ref_testbed._BSPLINE_GROUPS = groups
    try:
        run_fixture(out, "bs", sfft.bspline_test_function(),
                    sfft.DetectionConfig(box=_BigBox.centered(10, 8), delta=1e-4, s=200, r=2, b=10, rng_seed=3))
        out["bs_l2err"] = np.array([sfft.relative_l2_error(
            sfft.SparseSpectrum(out["bs_freqs"], out["bs_coef"]), sfft.bspline_exact_coefficients,
            sfft.bspline_norm_sq())])
    finally:
        ref_testbed._BSPLINE_GROUPS = saved


def transform_fixture(out):
    rng = np.random.default_rng(77)
    for K in (1, 2, 3, 5, 7, 33, 65, 97, 129, 1009, 6007):
        v = rng.normal(size=K) + 1j * rng.normal(size=K)
        out[f"dft_in_{K}"] = v
        out[f"dft_fwd_{K}"] = sfft.dft_1d(v, "forward")
        out[f"dft_inv_{K}"] = sfft.dft_1d(v, "inverse")
    spec = sfft.SparseSpectrum([(1, -2, 3), (0, 4, -1), (-3, 0, 0)], [1.0 + 0.5j, -2.0, 0.25j])
    oracle = _poly_signal(spec.freqs, spec.coeffs)
    box = sfft.SearchBox([-4, -5, -3], [4, 5, 3])
    anchor = np.array([0.3, 0.71, 0.05])
    for t in range(3):
        ks, c = sfft.projected_line_coefficients(oracle, t, box, anchor)
        out[f"line_{t}_ks"] = ks
        out[f"line_{t}_c"] = c
    out.update(line_hf=spec.freqs, line_hc=spec.coeffs, line_anchor=anchor)


def bspline_fixture(out):
    rng = np.random.default_rng(3)
    pts = rng.random((500, 10))
    f = sfft.bspline_test_function()
    out["bsv_pts"] = pts
    out["bsv_vals"] = f(pts)
    ks = rng.integers(-6, 7, size=(200, 10))
    ks[:100, 3:] = 0
    out["bsv_ks"] = ks
    out["bsv_exact"] = sfft.bspline_exact_coefficients(ks)
    out["bsv_norm_sq"] = np.array([sfft.bspline_norm_sq()])
    out["bsv_cm"] = np.array([sfft.bspline_l2_constant(m) for m in (2, 4, 6)])


def single_fixture(out):
    """Algorithm 5 path: CBC lattices, invert_single / eval_on_lattice, a run."""
    rng = np.random.default_rng(8)
    for i, (n, d, N) in enumerate(((1, 3, 4), (7, 1, 20), (40, 2, 6), (90, 3, 5), (60, 4, 3))):
        rows = np.unique(rng.integers(-N, N + 1, size=(n, d)), axis=0)
        lat = sfft.build_single_lattice_cbc(sfft.FrequencyIndexSet(rows))
        out[f"cbc{i}_rows"] = rows
        out[f"cbc{i}_z"] = lat.z
        out[f"cbc{i}_m"] = np.array([lat.m])
    rows = out["cbc3_rows"]
    lat = sfft.Rank1Lattice(out["cbc3_z"], int(out["cbc3_m"][0]))
    coef = rng.normal(size=len(rows)) + 1j * rng.normal(size=len(rows))
    spec = sfft.SparseSpectrum(rows, coef)
    samples = sfft.eval_on_lattice(spec, lat)
    out["single_eval"] = samples.values
    out["single_inv"] = sfft.invert_single(samples, spec.support()).coeffs
    out["single_coef"] = spec.coeffs
    rng = np.random.default_rng(45)
    truth, _ = sfft.gen_random_sparse_poly(3, 8, 15, "box", seed=rng)
    out.update(sk_hf=truth.freqs, sk_hc=truth.coeffs)
    run_fixture(out, "sk", _poly_signal(truth.freqs, truth.coeffs),
                sfft.DetectionConfig(box=sfft.SearchBox.centered(3, 8), delta=1e-12, s=15, r=1, b=10, rng_seed=9,
                                     lattice_kind="single"))


class _RelNoisy:
    """Per-call relative noise around a reference oracle (the
    harness adaptation of testbed.py:76-106 for BASELINE config 3): each call
    draws ``standard_normal((n, 2))`` from one numpy stream in call order and
    adds sigma_call / sqrt(2) * (e0 + i e1) with sigma_call = rel * ||p(X)|| / sqrt(n)."""

    def __init__(self, inner, rel, seed):
        self._inner = inner
        self.rel = float(rel)
        self.dim = inner.dim
        self.concurrency_safe = inner.concurrency_safe
        self._rng = np.random.default_rng(seed)
        self._calls = 0

    @property
    def call_count(self):
        return self._calls

    def __call__(self, points):
        values = self._inner(points)
        n = len(values)
        noise = self._rng.standard_normal((n, 2)) @ np.array([1.0, 1.0j])
        self._calls += n
        sigma = self.rel * np.sqrt(float(np.sum(np.abs(values) ** 2))) / np.sqrt(max(n, 1))
        return values + (sigma / np.sqrt(2.0)) * noise


def _store_run(out, key, rep, truth=None):
    out[f"{key}_freqs"] = rep.detected.freqs
    out[f"{key}_coef"] = rep.detected.coeffs
    out[f"{key}_counts"] = np.array([rep.candidate_counts, rep.prefix_counts, rep.component_counts,
                                     rep.scheme_sizes, rep.lattice_attempts, rep.inversion_calls])
    out[f"{key}_calls"] = np.array([rep.oracle_calls])
    out[f"{key}_warnings"] = np.array(rep.warnings if rep.warnings else [""])
    if truth is not None:
        out[f"{key}_err"] = np.array([sfft.relative_spectrum_l2_error(rep.detected, truth)])
    print(f"{key}: detected {len(rep.detected)} calls {rep.oracle_calls} attempts {rep.lattice_attempts} "
          f"warnings {rep.warnings} wall {rep.wall_time:.1f}s", flush=True)


def retry_fixture(out):
    """Retries and partial schemes: a first attempt that
    fails and is recovered by a retry (test_construct.py:178-190), sparse_fft
    runs whose steps need a second attempt (b = 10) or exhaust b = 1 and
    omit a candidate with the "covers only" warning (detect.py:385-392,
    test_detect.py:310-336).  Seeds found by a search over the reference."""
    rng = np.random.default_rng(19)
    for trial in range(300):
        rows = np.unique(rng.integers(-16, 17, size=(64, 4)), axis=0)
        I = sfft.FrequencyIndexSet(rows)
        cfg = sfft.MLConfig(c=2.0, gamma=0.5, rng_seed=trial)
        scheme, attempts = sfft.build_multiple_lattice_with_retries(I, cfg, b=20,
                                                                    seed_seq=np.random.SeedSequence(trial))
        if attempts >= 2:
            assert scheme.is_reconstructing
            out.update(rt_rows=I.freqs, rt_trial=np.array([trial]), rt_attempts=np.array([attempts]),
                       rt_ms=np.array([lat.m for lat in scheme.lattices]),
                       rt_zs=np.stack([lat.z for lat in scheme.lattices]),
                       rt_masks=pack_masks(scheme.recon_masks))
            print(f"retry scheme: trial {trial} attempts {attempts} L {len(scheme.lattices)}")
            break
    else:
        raise RuntimeError("no failing first attempt found")
    for key, seed, b in (("rtrun", 103, 10), ("partial", 955, 1)):
        truth, _ = sfft.gen_random_sparse_poly(3, 4, 6, "box", seed=np.random.default_rng(1000 + seed))
        out[f"{key}_hf"], out[f"{key}_hc"] = truth.freqs, truth.coeffs
        out[f"{key}_cfg"] = np.array([seed, b])
        rep = sfft.sparse_fft(_poly_signal(truth.freqs, truth.coeffs),
                              sfft.DetectionConfig(box=sfft.SearchBox.centered(3, 4), delta=1e-12, s=6, r=2, b=b,
                                                   rng_seed=seed))
        _store_run(out, key, rep, truth)


def long_line_fixture(out):
    """Component extents K_t > 1024 (lines longer than one CTA's tile):
    a d = 2 run on [-700, 700]^2 (K = 1401) and projected line coefficients."""
    truth, _ = sfft.gen_random_sparse_poly(2, 700, 12, "box", seed=np.random.default_rng(71))
    out.update(ll_hf=truth.freqs, ll_hc=truth.coeffs)
    rep = sfft.sparse_fft(_poly_signal(truth.freqs, truth.coeffs),
                          sfft.DetectionConfig(box=sfft.SearchBox.centered(2, 700), delta=1e-12, s=12, r=2, b=10,
                                               rng_seed=5))
    _store_run(out, "ll", rep, truth)
    anchor = np.array([0.37, 0.81])
    ks, c = sfft.projected_line_coefficients(_poly_signal(truth.freqs, truth.coeffs), 1,
                                             sfft.SearchBox.centered(2, 700), anchor)
    out.update(ll_line_anchor=anchor, ll_line_ks=ks, ll_line_c=c)


def harness_fixture(out):
    """The reference's experiment grid (cli.py:349-418) on two small specs:
    the emitted CSV text."""
    from sfft.cli import ExperimentSpec, emit, run_experiment
    from make_golden_specs import HARNESS_SPECS
    for key, kw in HARNESS_SPECS.items():
        rows, code = run_experiment(ExperimentSpec(**kw))
        out[f"{key}_csv"] = np.array([emit(rows, "csv")])
        out[f"{key}_code"] = np.array([code])
        print(emit(rows, "csv"))


def cfg3_reduced_fixture(out):
    """BASELINE config 3 (d = 20, [-32, 32]^20, polar coefficients, per-call
    1e-2 relative noise, delta = 0.1) at reduced sparsity s = 100, r = 2, run
    by the unmodified reference through the guard-free box."""
    wl = workloads.config3(seed=0, d=20, s=100, r=2)
    ts, rs, ns = workloads.seeds_for(0, 3, 0)
    out.update(c3_hf=wl.truth.freqs, c3_hc=wl.truth.coeffs, c3_seed=np.array([rs], np.uint64))
    noisy = _RelNoisy(_poly_signal(wl.truth.freqs, wl.truth.coeffs), 1e-2, ns)
    cfg = sfft.DetectionConfig(box=_BigBox.centered(20, 32), delta=0.1, s=100, r=2, b=10, rng_seed=rs)
    rep = sfft.sparse_fft(noisy, cfg)
    _store_run(out, "c3", rep, sfft.SparseSpectrum(wl.truth.freqs, wl.truth.coeffs))


def cfg4_full_fixture(out):
    """BASELINE config 4 at full size (N = 64, s = 2000, r = 5, delta = 1e-6)
    with the seed-chosen partition (testbed.py:188-265)."""
    wl = workloads.config4()
    groups = wl.oracle.groups
    out["c4_groups"] = np.array([[m] + list(c) + [-1] * (4 - len(c)) for m, c in groups])
    out["c4_seed"] = np.array([wl.cfg.rng_seed], np.uint64)
    saved = ref_testbed._BSPLINE_GROUPS
    ref_testbed._BSPLINE_GROUPS = tuple((int(m), tuple(int(c) for c in comps)) for m, comps in groups)
    try:
        cfg = sfft.DetectionConfig(box=_BigBox.centered(10, 64), delta=1e-6, s=2000, r=5, b=10,
                                   rng_seed=wl.cfg.rng_seed)
        rep = sfft.sparse_fft(sfft.bspline_test_function(), cfg)
        _store_run(out, "c4", rep)
        out["c4_l2err"] = np.array([sfft.relative_l2_error(rep.detected, sfft.bspline_exact_coefficients,
                                                           sfft.bspline_norm_sq())])
        print("c4 l2 err", out["c4_l2err"][0])
    finally:
        ref_testbed._BSPLINE_GROUPS = saved


def main_ext(which):
    """Slow fixtures (minutes of reference CPU time) in golden_ext.npz;
    ``which`` selects the ones to (re)generate, the others are kept."""
    path = HERE / "golden_ext.npz"
    out: dict = dict(np.load(path)) if path.exists() else {}
    fns = {"retry": retry_fixture, "cfg3": cfg3_reduced_fixture, "cfg4": cfg4_full_fixture,
           "longline": long_line_fixture, "harness": harness_fixture}
    for name in which or list(fns):
        prefix = {"retry": ("rt_", "rtrun_", "partial_"), "cfg3": ("c3_",), "cfg4": ("c4_",),
                  "longline": ("ll_",), "harness": ("hx_", "hn_")}[name]
        out = {k: v for k, v in out.items() if not k.startswith(prefix)}
        fns[name](out)
        np.savez_compressed(path, **out)
    print("wrote", path, sum(v.nbytes for v in out.values()), "bytes raw")


def main():
    out: dict = {}
    single_fixture(out)
    residues_fixture(out)
    primes_fixture(out)
    transform_fixture(out)
    bspline_fixture(out)
    scheme_fixture(out)
    runs_fixture(out)
    np.savez_compressed(HERE / "golden.npz", **out)
    print("wrote", HERE / "golden.npz", sum(v.nbytes for v in out.values()), "bytes raw")


if __name__ == "__main__":
    if "--ext" in sys.argv:
        main_ext([a for a in sys.argv[1:] if not a.startswith("--")])
    else:
        main()
