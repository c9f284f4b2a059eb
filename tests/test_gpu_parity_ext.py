"""GPU parity on the slow reference runs (tests/golden/golden_ext.npz, made by
``make_golden.py --ext`` from the unmodified reference): retries and partial
schemes, BASELINE config 3 at reduced sparsity (d = 20, per-call relative
noise) with the reference noise stream and with device noise, BASELINE
config 4 at full size.  Everything goes through the C ABI (libsfft_b200.so).

Bar: detected sets and integer accounting bit-exact; coefficients within
COEF_RTOL relative (fp64)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

COEF_RTOL = 1e-10


@pytest.fixture(scope="module")
def P():
    import paper_1711_05152_b200 as P
    from paper_1711_05152_b200 import _native
    _native.load()
    return P


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def _check(g, key, rep, exact_coef=True):
    assert np.array_equal(rep.detected.freqs, g[f"{key}_freqs"]), key
    ref = g[f"{key}_coef"]
    if len(ref) and exact_coef:
        assert _rel(rep.detected.coeffs, ref) <= COEF_RTOL, key
    cnt = g[f"{key}_counts"]
    assert rep.candidate_counts == cnt[0].tolist()
    assert rep.prefix_counts == cnt[1].tolist()
    assert rep.component_counts == cnt[2].tolist()
    assert rep.scheme_sizes == cnt[3].tolist()
    assert rep.lattice_attempts == cnt[4].tolist()
    assert rep.inversion_calls == cnt[5].tolist()
    assert rep.oracle_calls == int(g[f"{key}_calls"][0])
    want = [str(w) for w in g[f"{key}_warnings"] if str(w)]
    assert rep.warnings == want


# ---------------------------------------------------------------------------
# retries / partial schemes (construct.py:185-206; detect.py:385-392)

def test_retry_scheme_bit_exact(P, golden_ext):
    """The first attempt fails, the second covers (test_construct.py:178-190):
    attempts, primes, generating vectors and masks are the reference's."""
    g = golden_ext
    I = P.FrequencyIndexSet(g["rt_rows"])
    sch, attempts = P.build_multiple_lattice_with_retries(I, P.MLConfig(), 20,
                                                          np.random.SeedSequence(int(g["rt_trial"][0])))
    assert attempts == int(g["rt_attempts"][0]) >= 2
    assert sch.is_reconstructing
    assert [lat.m for lat in sch.lattices] == g["rt_ms"].tolist()
    assert np.array_equal(np.stack([lat.z for lat in sch.lattices]), g["rt_zs"])
    words = np.zeros(len(I), dtype=np.uint64)
    for l, mk in enumerate(sch.recon_masks):
        words |= mk.astype(np.uint64) << np.uint64(l)
    assert np.array_equal(words, g["rt_masks"])


def test_sparse_fft_step_needs_retry(P, golden_ext):
    """A sparse_fft run whose step 1 needs a second lattice attempt (b = 10)."""
    g = golden_ext
    seed, b = (int(x) for x in g["rtrun_cfg"])
    oracle = P.SparsePolynomialOracle(g["rtrun_hf"], g["rtrun_hc"])
    rep = P.sparse_fft(oracle, P.DetectionConfig(box=P.SearchBox.centered(3, 4), delta=1e-12, s=6, r=2, b=b,
                                                 rng_seed=seed))
    assert max(rep.lattice_attempts) >= 2
    _check(g, "rtrun", rep)
    assert oracle.call_count == rep.oracle_calls


def test_sparse_fft_partial_scheme_warns_and_omits(P, golden_ext):
    """b = 1 and a non-covering draw: the reference's warning text, and the
    uncovered true frequency is missing from the result (test_detect.py:310-336,
    here from a natural failure instead of a crippled builder)."""
    g = golden_ext
    seed, b = (int(x) for x in g["partial_cfg"])
    oracle = P.SparsePolynomialOracle(g["partial_hf"], g["partial_hc"])
    rep = P.sparse_fft(oracle, P.DetectionConfig(box=P.SearchBox.centered(3, 4), delta=1e-12, s=6, r=2, b=b,
                                                 rng_seed=seed))
    _check(g, "partial", rep)
    assert any("covers only" in w for w in rep.warnings)
    assert len(rep.detected) < len(g["partial_hf"])


def test_sparse_fft_crippled_scheme(P, monkeypatch):
    """test_detect.py:310-336 ported to the device seam: a scheme builder that
    drops one candidate from every lattice's reconstruction set produces the
    "covers only" warning and the candidate is omitted."""
    from paper_1711_05152_b200 import engine
    truth = P.SparseSpectrum([(1, 2), (3, 1), (-2, 0)], [1.0, 2.0, 3.0])
    dropped = (1, 2)
    real = engine.build_scheme

    def crippled(dev, cand, b, seed_seq, **kw):
        sch = real(dev, cand, b, seed_seq, **kw)
        rows = cand.to_host(dev)
        hit = np.nonzero((rows == np.array(dropped)).all(axis=1))[0] if rows.shape[1] == 2 else []
        if len(hit):
            sch.masks[int(hit[0])] = 0
            sch.uncovered = 1
        return sch

    monkeypatch.setattr(engine, "build_scheme", crippled)
    oracle = P.SparsePolynomialOracle(truth.freqs, truth.coeffs)
    rep = P.sparse_fft(oracle, P.DetectionConfig(box=P.SearchBox.centered(2, 4), delta=1e-12, s=3, b=2, rng_seed=1))
    assert any("covers only" in w for w in rep.warnings)
    assert dropped not in rep.detected
    assert (3, 1) in rep.detected


# ---------------------------------------------------------------------------
# BASELINE config 3, reduced: d = 20, [-32, 32]^20, polar coefficients,
# per-call relative noise 1e-2, delta = 0.1, s = 100, r = 2

def _cfg3(P, g, device_rng):
    from paper_1711_05152_b200 import workloads
    wl = workloads.config3(seed=0, d=20, s=100, r=2, device_rng=device_rng)
    assert np.array_equal(wl.truth.freqs, g["c3_hf"]) and np.array_equal(wl.truth.coeffs, g["c3_hc"])
    assert wl.cfg.rng_seed == int(g["c3_seed"][0])
    return wl


def test_config3_reduced_reference_noise(P, golden_ext):
    """RelativeNoisyOracle(device_rng=False): the reference's numpy noise
    realisation in the reference call order -> the reference's run."""
    g = golden_ext
    wl = _cfg3(P, g, False)
    rep = P.sparse_fft(wl.oracle, wl.cfg)
    _check(g, "c3", rep)
    assert wl.oracle.call_count == rep.oracle_calls
    err = P.relative_spectrum_l2_error(rep.detected, wl.truth)
    assert abs(err - float(g["c3_err"][0])) <= 1e-8 * max(float(g["c3_err"][0]), 1e-300) + 1e-14


def test_config3_reduced_device_noise(P, golden_ext):
    """RelativeNoisyOracle(device_rng=True): a different realisation of the
    same noise law -> the same support as the reference run, the same
    integer accounting, and an error at the noise level."""
    g = golden_ext
    wl = _cfg3(P, g, True)
    rep = P.sparse_fft(wl.oracle, wl.cfg)
    assert np.array_equal(rep.detected.freqs, g["c3_freqs"])
    assert rep.detected.support() == wl.truth.support()
    cnt = g["c3_counts"]
    assert rep.candidate_counts == cnt[0].tolist() and rep.scheme_sizes == cnt[3].tolist()
    assert rep.oracle_calls == int(g["c3_calls"][0]) == wl.oracle.call_count
    err = P.relative_spectrum_l2_error(rep.detected, wl.truth)
    ref_err = float(g["c3_err"][0])
    assert 0.5 * ref_err <= err <= 2.0 * ref_err, (err, ref_err)


def _devnoise(dev, ms, clean, units, rel, seed, base):
    """Apply sfft_finish_devnoise (no chirp) to clean samples of the listed
    units; returns the noise per slot."""
    from paper_1711_05152_b200.device import dptr, hptr
    torch = dev.torch
    L = len(ms)
    P_ = int(max(ms))
    buf = torch.zeros((len(units), P_, 2), dtype=torch.float64, device=dev.device)
    for j, u in enumerate(units):
        m = int(ms[u % L])
        buf[j, :m, 0] = torch.from_numpy(clean[u][:m].real)
        buf[j, :m, 1] = torch.from_numpy(clean[u][:m].imag)
    ua = np.ascontiguousarray(np.asarray(units, dtype=np.int32))
    rb = (max(units) // L) + 1
    nrm = dev.empty((len(units),), torch.float64)
    hm = np.ascontiguousarray(np.asarray(ms, dtype=np.int64))
    dev.call("sfft_unit_norm2", hptr(hm), L, rb, dptr(buf), P_, dptr(nrm), hptr(ua), len(ua))
    chirp = dev.zeros((int(sum(ms)), 2), torch.float64)
    dev.call("sfft_finish_devnoise", hptr(hm), L, rb, dptr(chirp), dptr(buf), P_, dptr(nrm), rel, 0.0, seed,
             base, 0, hptr(ua), len(ua))
    out = dev.download(buf)
    noisy = out[..., 0] + 1j * out[..., 1]
    return {u: noisy[j, :int(ms[u % L])] - clean[u][:int(ms[u % L])] for j, u in enumerate(units)}


def test_device_noise_law_and_unit_independence(P):
    """Device Philox noise: per call ||eta|| / ||p(X)|| = rel within the chi
    fluctuation, zero mean, unit-variance real/imag parts, uncorrelated with
    the clean signal; a unit's noise depends only on (seed, call index), not
    on which other units share the launch or their order (the sharded path
    hands each GPU a subset of the units)."""
    from paper_1711_05152_b200.device import get_device
    dev = get_device()
    rng = np.random.default_rng(5)
    ms = [20011, 30011, 40009]
    L, rb = len(ms), 2
    clean = {u: (rng.normal(size=ms[u % L]) + 1j * rng.normal(size=ms[u % L])) * (1 + u) for u in range(rb * L)}
    rel, seed, base = 1e-2, 987654321, 17
    full = _devnoise(dev, ms, clean, list(range(rb * L)), rel, seed, base)
    for u, eta in full.items():
        m = len(eta)
        ratio = np.linalg.norm(eta) / np.linalg.norm(clean[u])
        assert abs(ratio / rel - 1.0) <= 6.0 / np.sqrt(2 * m), (u, ratio)
        z = eta / (rel * np.linalg.norm(clean[u]) / np.sqrt(m) / np.sqrt(2.0))
        assert abs(z.real.mean()) <= 6 / np.sqrt(m) and abs(z.imag.mean()) <= 6 / np.sqrt(m)
        assert abs(z.real.var() - 1) <= 0.05 and abs(z.imag.var() - 1) <= 0.05
        assert abs(np.corrcoef(z.real, z.imag)[0, 1]) <= 6 / np.sqrt(m)
        assert abs(np.vdot(clean[u], eta)) / (np.linalg.norm(clean[u]) * np.linalg.norm(eta)) <= 6 / np.sqrt(m)
    # units of different calls are independent streams
    a, b = full[0][:20011], full[3][:20011]
    assert abs(np.vdot(a, b)) / (np.linalg.norm(a) * np.linalg.norm(b)) <= 6 / np.sqrt(20011)
    # subsets / permutations (what each rank of a sharded step launches) give the same noise
    for units in ([5, 1, 3], [4], [2, 0]):
        part = _devnoise(dev, ms, clean, units, rel, seed, base)
        for u in units:
            assert np.array_equal(part[u], full[u]), units
    # another call base is another realisation
    other = _devnoise(dev, ms, clean, [0], rel, seed, base + 1)
    assert not np.array_equal(other[0], full[0])


# ---------------------------------------------------------------------------
# BASELINE config 4 at full size (N = 64, s = 2000, r = 5, delta = 1e-6)

def test_config4_full_size(P, golden_ext):
    """B-spline approximation at full size against the reference run with the
    seed-chosen partition: the same number of terms and L2 error to 4 digits;
    the detected sets may differ only by cap-boundary members whose exact
    coefficients have exactly equal magnitude (+-k mirror ties, SURVEY §7
    hard part 5), each swapped member pairing with one of equal magnitude."""
    from paper_1711_05152_b200 import workloads
    g = golden_ext
    wl = workloads.config4()
    groups = tuple((int(row[0]), tuple(int(x) for x in row[1:] if x >= 0)) for row in g["c4_groups"])
    assert wl.oracle.groups == groups and wl.cfg.rng_seed == int(g["c4_seed"][0])
    c0 = wl.oracle.call_count
    rep = P.sparse_fft(wl.oracle, wl.cfg)
    assert wl.oracle.call_count - c0 == rep.oracle_calls
    assert len(rep.detected) == len(g["c4_freqs"])
    err = P.relative_l2_error(rep.detected, wl.oracle.exact_coefficients, wl.oracle.norm_sq())
    ref_err = float(g["c4_l2err"][0])
    assert abs(err - ref_err) <= 5e-5 * ref_err, (err, ref_err)
    got = set(map(tuple, rep.detected.freqs.tolist()))
    ref = set(map(tuple, g["c4_freqs"].tolist()))
    only_got = np.array(sorted(got - ref), dtype=np.int64).reshape(-1, 10)
    only_ref = np.array(sorted(ref - got), dtype=np.int64).reshape(-1, 10)
    assert len(only_got) == len(only_ref) <= 16
    if len(only_got):
        mg = np.abs(wl.oracle.exact_coefficients(only_got))
        mr = np.abs(wl.oracle.exact_coefficients(only_ref))
        for m in mg:
            assert np.min(np.abs(mr - m)) <= 1e-12 * m
    # the first nine steps' integer accounting is the reference's; the last
    # step's candidate set inherits any tie swap of step 8
    cnt = g["c4_counts"]
    assert rep.component_counts == cnt[2].tolist()
    assert rep.lattice_attempts == cnt[4].tolist()


# ---------------------------------------------------------------------------
# component extents K_t > 1024 (tiled line sampling + Bluestein line DFT)

def test_long_lines_projected_coefficients(P, golden_ext):
    g = golden_ext
    oracle = P.SparsePolynomialOracle(g["ll_hf"], g["ll_hc"])
    ks, c = P.projected_line_coefficients(oracle, 1, P.SearchBox.centered(2, 700), g["ll_line_anchor"])
    assert np.array_equal(ks, g["ll_line_ks"])
    assert np.abs(c - g["ll_line_c"]).max() <= 1e-12


def test_long_lines_sparse_fft(P, golden_ext):
    g = golden_ext
    oracle = P.SparsePolynomialOracle(g["ll_hf"], g["ll_hc"])
    rep = P.sparse_fft(oracle, P.DetectionConfig(box=P.SearchBox.centered(2, 700), delta=1e-12, s=12, r=2, b=10,
                                                 rng_seed=5))
    _check(g, "ll", rep)


def test_long_lines_binding_cap_matches_oracle(P):
    """K = 1401 lines whose survivors exceed the cap: the row selection keeps
    the reference's (|c| desc, k asc) order, as the oracle's _select."""
    from oracle import sfft_oracle as O
    rng = np.random.default_rng(3)
    freqs = np.unique(rng.integers(-700, 701, size=(40, 2)), axis=0)
    coef = rng.uniform(0.5, 2.0, len(freqs)) + 0j
    coef[:6] = 1.25  # exact ties across the cap boundary
    oracle = P.SparsePolynomialOracle(freqs, coef)
    box = P.SearchBox.centered(2, 700)
    cfg = P.DetectionConfig(box=box, delta=1e-9, s=len(freqs), s_local=9, r=2, b=10, rng_seed=4)
    comp = P.detect_component(oracle, 0, cfg, rng=np.random.default_rng(8))
    fn = lambda p: O.poly_eval(freqs, coef, p)
    rng2 = np.random.default_rng(8)
    want = []
    for _ in range(2):
        ks, cf = O.line_coefficients(fn, 0, [-700] * 2, [700] * 2, rng2.random(2))
        kept, _ = O.select(ks[:, None], cf, 9, 1e-9)
        want.append(kept[:, 0])
    assert np.array_equal(comp.freqs[:, 0], np.unique(np.concatenate(want)))


# ---------------------------------------------------------------------------
# K1b: the B-spline sampler (lattice factors shared by the units of a lattice)

@pytest.mark.parametrize("units", [None, [5, 0, 3], [4]])
def test_bspline_sampler_matches_oracle(P, units):
    """sfft_sample_bspline at lattice nodes + anchor tails (detect.py:290-297)
    against the CPU oracle's B-spline (testbed.py:198-244), raw samples
    (no chirp): every unit, or a unit subset in any order (sharded steps)."""
    from oracle import sfft_oracle as O
    from paper_1711_05152_b200.device import dptr, get_device, hptr
    dev = get_device()
    torch = dev.torch
    groups = ((2, (0, 5, 7)), (4, (1, 3, 4, 9)), (6, (2, 6, 8)))
    oracle = P.bspline_test_function(groups)
    order, start, comps, scale = oracle.host_spec()
    rng = np.random.default_rng(4)
    t1, d, rb = 6, 10, 2
    ms = np.array([10007, 7919, 4099], dtype=np.int64)
    L = len(ms)
    zs = np.ascontiguousarray(np.stack([rng.integers(0, m, t1) for m in ms]).astype(np.int32))
    anchor = np.ascontiguousarray(rng.random((rb, d - t1)))
    ulist = list(range(rb * L)) if units is None else units
    ua = None if units is None else np.ascontiguousarray(np.asarray(units, dtype=np.int32))
    Pl = 10240
    buf = dev.zeros((len(ulist), Pl, 2), torch.float64)
    chirp = dev.zeros((int(ms.sum()), 2), torch.float64)
    dev.call("sfft_sample_bspline", len(groups), hptr(order), hptr(start), hptr(comps), hptr(scale), d, t1,
             hptr(ms), hptr(zs), L, hptr(anchor), rb, dptr(chirp), dptr(buf), Pl, 0,
             hptr(ua) if ua is not None else 0, len(ua) if ua is not None else 0)
    got = dev.download(buf)
    for j, u in enumerate(ulist):
        i, l = divmod(u, L)
        m = int(ms[l])
        pts = np.empty((m, d))
        pts[:, :t1] = O.lattice_nodes(zs[l].astype(np.int64), m)
        pts[:, t1:] = anchor[i]
        ref = O.bspline_eval(groups, pts)
        v = got[j, :m, 0] + 1j * got[j, :m, 1]
        assert np.abs(v - ref).max() <= 1e-13 * np.abs(ref).max(), (u, np.abs(v - ref).max())


@pytest.mark.parametrize("n,nvals", [(100_000, 7), (3_000_000, 40)])
def test_cap_selection_many_ties(P, n, nvals):
    """The cap (detect.py:205-211: |c| descending, ties by ascending index =
    lexicographic candidate order) when far more than 2048 entries tie at the
    threshold (the chunked count / scan / mark path), for two rows at once."""
    from paper_1711_05152_b200 import _native
    from paper_1711_05152_b200.device import dptr, get_device, hptr
    dev = get_device()
    torch = dev.torch
    rng = np.random.default_rng(n)
    levels = rng.uniform(0.5, 2.0, nvals)
    mags = levels[rng.integers(0, nvals, (2, n))]
    quarter = rng.integers(0, 4, (2, n))  # c = level * i^q: exact magnitudes, many exact ties
    c = np.where(quarter % 2 == 0, mags * (1 - quarter) + 0j, 1j * mags * (2 - quarter))
    keep0 = (rng.random((2, n)) < 0.9).astype(np.uint8)
    cap = n // 3
    coef = torch.from_numpy(np.stack([c.real, c.imag], axis=-1)).to(dev.device)
    keep = torch.from_numpy(keep0.copy()).to(dev.device)
    counts = torch.from_numpy(keep0.sum(axis=1).astype(np.int32)).to(dev.device)
    rows = np.arange(2, dtype=np.int32)
    sb = int(_native.query("sfft_select_rows_scratch_bytes", 2))
    scratch = dev.empty((sb,), torch.uint8)
    dev.call("sfft_select_cap_rows", dptr(coef), dptr(keep), n, hptr(rows), 2, cap, dptr(counts), dptr(scratch))
    got = dev.download(keep).astype(bool)
    mag_dev = np.hypot(c.real, c.imag)
    for y in range(2):
        idx = np.nonzero(keep0[y])[0]
        order = np.lexsort((idx, -mag_dev[y, idx]))[:cap]
        want = np.zeros(n, dtype=bool)
        want[idx[order]] = True
        thr = mag_dev[y, idx[order[-1]]]
        assert (mag_dev[y, idx] == thr).sum() > 2048  # the overflow path ran
        assert np.array_equal(got[y], want), y
    assert dev.download(counts).tolist() == [cap, cap]


# ---------------------------------------------------------------------------
# api.reconstruct_step (the e2e entry): speculative first attempt, deferred
# extent read-back, and its fallbacks

@pytest.mark.parametrize("kind", ["config1", "wide", "int64_rows"])
def test_reconstruct_step_matches_oracle(P, kind):
    """The composed step (construction + sampling + inversion + threshold)
    against the oracle's mr1l_step: same lattices, masks, coefficients.
    'wide': components spanning more than lambda = 2(|J| - 1), so the
    speculated primes are invalid and the reference's construction runs."""
    from oracle import sfft_oracle as O
    from paper_1711_05152_b200 import workloads
    if kind == "config1":
        wl = workloads.config1(seed=4, n=5000, nnz=90)
        cand, oracle, seed = wl.cand, wl.oracle, wl.lattice_seed
    else:
        rng = np.random.default_rng(12)
        cand = np.unique(rng.integers(-3000, 3001, size=(300, 3)), axis=0)
        hf = cand[rng.choice(len(cand), 20, replace=False)]
        hc = rng.uniform(-1, 1, 20) + 1j * rng.uniform(-1, 1, 20)
        oracle = P.SparsePolynomialOracle(hf, hc)
        seed = 77
    arg = cand
    if kind == "int64_rows":  # a pinned torch tensor, as the bench passes it
        import torch
        arg = torch.from_numpy(np.ascontiguousarray(cand, dtype=np.int64)).pin_memory()
    rep = P.api.reconstruct_step(arg, oracle, b=10, seed_seq=seed, delta=1e-12)
    sch = O.build_with_retries(np.asarray(cand, np.int64), 10, np.random.SeedSequence(seed))
    assert rep.lattice_sizes == sch.ms and rep.attempts == sch.attempts
    assert np.array_equal(np.asarray(rep.generating_vectors), np.stack(sch.zs))
    vals = [O.poly_eval(oracle.freqs, oracle.coeffs, O.lattice_nodes(z, m)) for m, z in zip(sch.ms, sch.zs)]
    cov, coefs = O.invert_multiple(np.asarray(cand, np.int64), sch, vals)
    assert np.array_equal(rep.covered, cov)
    assert _rel(rep.coeffs[cov], coefs) <= COEF_RTOL


def test_reconstruct_step_rejects_out_of_range_components(P):
    rows = np.array([[0, 1], [2**31, 0]], dtype=np.int64)
    with pytest.raises(ValueError, match="2147483647"):
        P.api.reconstruct_step(rows, P.SparsePolynomialOracle(np.array([[0, 1]]), np.array([1.0 + 0j])), b=5,
                               seed_seq=1, delta=1e-12)
