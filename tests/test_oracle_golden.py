"""Pin the CPU oracle (oracle/sfft_oracle.py) against golden vectors produced
by the unmodified reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import sfft_oracle as O


def test_residues_and_masks(golden):
    f, ms, zs = golden["res_freqs"], golden["res_ms"], golden["res_zs"]
    for i, (m, z) in enumerate(zip(ms, zs)):
        assert np.array_equal(O.residues(f, z, int(m)), golden["res_values"][i])
    for i in range(4):
        assert np.array_equal(O.alias_free_mask(f, zs[i], int(ms[i])), golden["res_masks"][i])


def test_overflow_free_residues(golden):
    # components at +-(2^31 - 1) with M = 2^31 - 1 (reference test_lattice.py:213-221)
    f, ms, zs = golden["res_freqs"], golden["res_ms"], golden["res_zs"]
    r = O.residues(f[-2:], zs[-1], int(ms[-1]))
    assert np.array_equal(r, golden["res_values"][-1][-2:])
    assert (r >= 0).all() and (r < ms[-1]).all()


def test_lattice_nodes(golden):
    got = O.lattice_nodes(golden["nodes_z"], 1009)[:64]
    assert np.array_equal(got, golden["nodes_1009"])


def test_candidate_primes_pins(golden):
    rows = np.array([[0, 0], [40, 1], [-40, 2], [3, -40]])
    assert O.candidate_primes(rows, 2 * (len(rows) - 1), 6) == golden["primes_small"].tolist()
    rng = np.random.default_rng(5)
    J = O.unique_rows(rng.integers(-32, 33, size=(5000, 10)))
    assert O.candidate_primes(J, 2 * (len(J) - 1), 19) == golden["primes_5000"].tolist()
    assert [O.max_lattices(n) for n in (1, 2, 1000, 65000, 100000, 650000)] == golden["lmax_pins"].tolist()


def test_dft_known_answers(golden):
    for K in (1, 2, 3, 5, 7, 33, 65, 97, 129, 1009, 6007):
        v = golden[f"dft_in_{K}"]
        fwd = np.fft.fft(v)
        assert np.abs(fwd - golden[f"dft_fwd_{K}"]).max() <= 1e-12 * max(1.0, np.abs(fwd).max())
        inv = np.fft.ifft(v)
        assert np.abs(inv - golden[f"dft_inv_{K}"]).max() <= 1e-12 * max(1.0, np.abs(inv).max())


def test_naive_dft_97():
    # O(K^2) oracle (reference test_transform.py:25-29, 59-66)
    rng = np.random.default_rng(0)
    v = rng.normal(size=97) + 1j * rng.normal(size=97)
    n = np.arange(97)
    naive = np.exp(-2j * np.pi * np.outer(n, n) / 97) @ v
    assert np.abs(np.fft.fft(v) - naive).max() <= 1e-12 * np.abs(naive).max()


def test_line_coefficients(golden):
    f, c = golden["line_hf"], golden["line_hc"]
    fn = lambda p: O.poly_eval(f, c, p)
    for t in range(3):
        ks, got = O.line_coefficients(fn, t, [-4, -5, -3], [4, 5, 3], golden["line_anchor"])
        assert np.array_equal(ks, golden[f"line_{t}_ks"])
        assert np.abs(got - golden[f"line_{t}_c"]).max() <= 1e-13


def test_bspline_values_and_pins(golden):
    groups = ((2, (0, 2, 7)), (4, (1, 4, 5, 9)), (6, (3, 6, 8)))
    got = O.bspline_eval(groups, golden["bsv_pts"])
    ref = golden["bsv_vals"]
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    assert np.allclose([O.bspline_constant(m) for m in (2, 4, 6)], golden["bsv_cm"], rtol=0, atol=1e-15)
    assert golden["bsv_norm_sq"][0] == pytest.approx(3.860521370158563, abs=1e-14)


def test_scheme_and_step(golden):
    cand = golden["step_cand"].astype(np.int64)
    seed = int(golden["step_seed"][0])
    sch = O.build_with_retries(cand, int(golden["step_b"][0]), np.random.SeedSequence(seed))
    assert sch.ms == golden["step_ms"].tolist()
    assert np.array_equal(np.stack(sch.zs), golden["step_zs"])
    words = np.zeros(len(cand), dtype=np.uint64)
    for l, mk in enumerate(sch.masks):
        words |= mk.astype(np.uint64) << np.uint64(l)
    assert np.array_equal(words, golden["step_masks"])
    assert sch.attempts == int(golden["step_attempts"][0])
    fn = lambda p: O.poly_eval(golden["step_hf"], golden["step_hc"], p)
    vals = [fn(O.lattice_nodes(z, m)) for m, z in zip(sch.ms, sch.zs)]
    assert np.abs(vals[0][:256] - golden["step_first_samples"]).max() <= 1e-13
    cov, coefs = O.invert_multiple(cand, sch, vals)
    assert np.array_equal(cand[cov], golden["step_cov_freqs"].astype(np.int64))
    ref = golden["step_coef"]
    assert np.linalg.norm(coefs - ref) <= 1e-12 * np.linalg.norm(ref)
    f, c = O.select(cand[cov], coefs, len(cand), 1e-12)
    assert np.array_equal(f, golden["step_sel"].astype(np.int64))


def _check_run(golden, key, rep, tol=1e-10):
    assert np.array_equal(rep.freqs, golden[f"{key}_freqs"])
    ref = golden[f"{key}_coef"]
    if len(ref):
        assert np.linalg.norm(rep.coeffs - ref) <= tol * np.linalg.norm(ref)
    cnt = golden[f"{key}_counts"]
    assert rep.candidate_counts == cnt[0].tolist()
    assert rep.prefix_counts == cnt[1].tolist()
    assert rep.component_counts == cnt[2].tolist()
    assert rep.scheme_sizes == cnt[3].tolist()
    assert rep.attempts == cnt[4].tolist()
    assert rep.oracle_calls == int(golden[f"{key}_calls"][0])


def test_engine_config0(golden):
    f, c = golden["cfg0_hf"], golden["cfg0_hc"]
    rep = O.sparse_fft(lambda p: O.poly_eval(f, c, p), [-16] * 5, [16] * 5, 1e-12, 100, r=2, b=10,
                       rng_seed=int(golden["cfg0_seed"][0]))
    _check_run(golden, "cfg0", rep)


def test_engine_caps_zero_anchor_1d(golden):
    f, c = golden["cap_hf"], golden["cap_hc"]
    rep = O.sparse_fft(lambda p: O.poly_eval(f, c, p), [-6] * 3, [6] * 3, 1e-12, 10, r=2, b=5, rng_seed=7,
                       s_local=12)
    _check_run(golden, "cap", rep)
    f, c = golden["zero_hf"], golden["zero_hc"]
    rep = O.sparse_fft(lambda p: O.poly_eval(f, c, p), [-5] * 3, [5] * 3, 1e-12, len(f), r=1, b=10,
                       zero_anchor=True)
    _check_run(golden, "zero", rep)
    f, c = golden["one_hf"], golden["one_hc"]
    rep = O.sparse_fft(lambda p: O.poly_eval(f, c, p), [-5], [5], 1e-12, 3, r=1, b=5)
    _check_run(golden, "one", rep)


def test_cbc_and_single_path(golden):
    for i in range(5):
        z, m = O.cbc(golden[f"cbc{i}_rows"])
        assert m == int(golden[f"cbc{i}_m"][0]) and np.array_equal(z, golden[f"cbc{i}_z"])
    rows = golden["cbc3_rows"]
    got = O.invert_single(rows, golden["cbc3_z"], int(golden["cbc3_m"][0]), golden["single_eval"])
    assert np.abs(got - golden["single_inv"]).max() <= 1e-13
    f, c = golden["sk_hf"], golden["sk_hc"]
    rep = O.sparse_fft(lambda p: O.poly_eval(f, c, p), [-8] * 3, [8] * 3, 1e-12, 15, r=1, b=10, rng_seed=9,
                       single=True)
    _check_run(golden, "sk", rep)


def test_engine_noisy(golden):
    f, c = golden["noisy_hf"], golden["noisy_hc"]
    rng = np.random.default_rng(123)
    sigma = float(np.sqrt(20) / np.sqrt(10 ** 3.0))

    def noisy(p):
        v = O.poly_eval(f, c, p)
        e = rng.standard_normal((len(p), 2)) @ np.array([1.0, 1.0j])
        return v + sigma / np.sqrt(2.0) * e

    rep = O.sparse_fft(noisy, [-8] * 4, [8] * 4, 0.3, 20, r=3, b=10, rng_seed=5)
    _check_run(golden, "noisy", rep)


def test_engine_bspline(golden):
    g = golden["bs_groups"]
    groups = tuple((int(row[0]), tuple(int(x) for x in row[1:] if x >= 0)) for row in g)
    rep = O.sparse_fft(lambda p: O.bspline_eval(groups, p), [-8] * 10, [8] * 10, 1e-4, 200, r=2, b=10,
                       rng_seed=3)
    # ulp-level differences may swap exact-tie cap-boundary pairs (SURVEY §7 hard part 5)
    got = set(map(tuple, rep.freqs.tolist()))
    ref = set(map(tuple, golden["bs_freqs"].tolist()))
    diff = got ^ ref
    assert len(diff) <= 4
    assert len(rep.freqs) == len(golden["bs_freqs"])


# ---------------------------------------------------------------------------
# extended reference runs (golden_ext.npz, make_golden.py --ext)

def test_retry_scheme(golden_ext):
    """A first attempt that fails, recovered by the retry (construct.py:185-206,
    test_construct.py:178-190)."""
    g = golden_ext
    sch = O.build_with_retries(g["rt_rows"], 20, np.random.SeedSequence(int(g["rt_trial"][0])))
    assert sch.attempts == int(g["rt_attempts"][0]) >= 2
    assert sch.ms == g["rt_ms"].tolist()
    assert np.array_equal(np.stack(sch.zs), g["rt_zs"])
    words = np.zeros(len(g["rt_rows"]), dtype=np.uint64)
    for l, mk in enumerate(sch.masks):
        words |= mk.astype(np.uint64) << np.uint64(l)
    assert np.array_equal(words, g["rt_masks"])


def test_engine_retry_and_partial_runs(golden_ext):
    """sparse_fft with a step that needs a second attempt (b = 10) and with a
    step whose b = 1 attempt leaves candidates uncovered (detect.py:385-392)."""
    for key in ("rtrun", "partial"):
        f, c = golden_ext[f"{key}_hf"], golden_ext[f"{key}_hc"]
        seed, b = (int(x) for x in golden_ext[f"{key}_cfg"])
        rep = O.sparse_fft(lambda p: O.poly_eval(f, c, p), [-4] * 3, [4] * 3, 1e-12, 6, r=2, b=b, rng_seed=seed)
        _check_run(golden_ext, key, rep)
    assert max(golden_ext["rtrun_counts"][4]) >= 2
    assert "covers only" in str(golden_ext["partial_warnings"][0])
    assert len(golden_ext["partial_freqs"]) < len(golden_ext["partial_hf"])


def test_engine_config3_reduced(golden_ext):
    """BASELINE config 3 at reduced sparsity (d = 20, s = 100, r = 2, delta =
    0.1) with per-call relative noise 1e-2 drawn in the reference call order."""
    from paper_1711_05152_b200 import workloads
    g = golden_ext
    f, c = g["c3_hf"], g["c3_hc"]
    _, rs, ns = workloads.seeds_for(0, 3, 0)
    assert rs == int(g["c3_seed"][0])
    rng = np.random.default_rng(ns)

    def noisy(p):
        v = O.poly_eval(f, c, p)
        e = rng.standard_normal((len(p), 2)) @ np.array([1.0, 1.0j])
        sigma = 1e-2 * np.sqrt(float(np.sum(np.abs(v) ** 2))) / np.sqrt(len(p))
        return v + sigma / np.sqrt(2.0) * e

    rep = O.sparse_fft(noisy, [-32] * 20, [32] * 20, 0.1, 100, r=2, b=10, rng_seed=rs)
    _check_run(g, "c3", rep)


def test_engine_long_lines(golden_ext):
    """Component extent K = 1401 > 1024 (reference run on [-700, 700]^2)."""
    g = golden_ext
    f, c = g["ll_hf"], g["ll_hc"]
    fn = lambda p: O.poly_eval(f, c, p)
    rep = O.sparse_fft(fn, [-700] * 2, [700] * 2, 1e-12, 12, r=2, b=10, rng_seed=5)
    _check_run(g, "ll", rep)
    ks, got = O.line_coefficients(fn, 1, [-700] * 2, [700] * 2, g["ll_line_anchor"])
    assert np.array_equal(ks, g["ll_line_ks"])
    assert np.abs(got - g["ll_line_c"]).max() <= 1e-12
