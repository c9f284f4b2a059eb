"""GPU parity: the CUDA path (through libsfft_b200.so) against the golden
vectors of the unmodified reference and the CPU oracle.

Bar (BASELINE north_star): detected frequency sets and every integer
quantity (residues, masks, schemes, counts) bit-exact; complex coefficients
within 1e-10 relative (fp64)."""

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


def test_cuda_path_is_native(P):
    import torch
    from paper_1711_05152_b200.device import get_device
    assert torch.cuda.is_available()
    dev = get_device()
    assert dev.cc[0] == 10, f"expected sm_100 (B200), got {dev.cc}"
    maps = open("/proc/self/maps").read()
    assert "libsfft_b200.so" in maps


def test_residues_bit_exact(P, golden):
    f, ms, zs = golden["res_freqs"], golden["res_ms"], golden["res_zs"]
    I = P.FrequencyIndexSet(f, _presorted=True)
    for i, (m, z) in enumerate(zip(ms, zs)):
        assert np.array_equal(P.residues(I, z, int(m)), golden["res_values"][i])


def test_lattice_nodes_bit_exact(P, golden):
    got = P.lattice_nodes(P.Rank1Lattice(golden["nodes_z"], 1009))
    assert got.shape == (1009, 6)
    assert np.array_equal(got[:64], golden["nodes_1009"])


def test_alias_masks_bit_exact(P, golden):
    from paper_1711_05152_b200.api import _masks_for
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs
    dev = get_device()
    f, ms, zs = golden["res_freqs"], golden["res_ms"][:4], golden["res_zs"][:4]
    cand = DeviceFreqs.from_host(dev, f)
    sch = _masks_for(dev, cand, [int(m) for m in ms], zs)
    words = dev.download(sch.masks).view(np.uint64)
    for l in range(4):
        got = ((words >> np.uint64(l)) & np.uint64(1)).astype(bool)
        assert np.array_equal(got, golden["res_masks"][l])


def test_alias_chunks_equal_one_pass(P):
    """Masks and stats of lattices [0, l1) then [l1, L) (sfft_alias_masks_range)
    equal one pass over all L, bit for bit."""
    from paper_1711_05152_b200.device import dptr, get_device, hptr
    from paper_1711_05152_b200.mr1l import DeviceFreqs
    from paper_1711_05152_b200.primes import primes_above
    from paper_1711_05152_b200 import _native
    dev = get_device()
    torch = dev.torch
    rng = np.random.default_rng(11)
    rows = np.unique(rng.integers(-32, 33, size=(30000, 10)), axis=0)
    cand = DeviceFreqs.from_host(dev, rows)
    n = len(rows)
    ms = np.asarray(primes_above(2 * (n - 1), 22), dtype=np.int64)
    zh = np.ascontiguousarray(rng.integers(0, ms[:, None], size=(22, 10)).astype(np.int32))
    words = int(_native.query("sfft_alias_scratch_words", hptr(ms), 22))
    scratch = dev.empty((words,), torch.int32)
    out = []
    for chunks in ([(0, 22)], [(0, 7), (7, 22)], [(0, 1), (1, 2), (2, 21), (21, 22)]):
        masks = dev.empty((n,), torch.int64)
        stats = dev.empty((2,), torch.int32)
        for l0, l1 in chunks:
            dev.call("sfft_alias_masks_range", dptr(cand.data), n, 10, cand.kmax, hptr(ms), hptr(zh), l0, l1,
                     dptr(scratch), words, dptr(masks), dptr(stats))
        out.append((dev.download(masks), dev.download(stats)))
    for m, st in out[1:]:
        assert np.array_equal(m, out[0][0])
        assert np.array_equal(st, out[0][1])
    from oracle import sfft_oracle as O
    for l in (0, 7, 21):
        ref = O.alias_free_mask(rows, zh[l].astype(np.int64), int(ms[l]))
        assert np.array_equal(((out[0][0].view(np.uint64) >> np.uint64(l)) & np.uint64(1)).astype(bool), ref)


def test_scheme_with_small_first_chunk(P, golden, monkeypatch):
    """A first chunk that cannot cover forces the second alias pass: same scheme."""
    from paper_1711_05152_b200 import mr1l
    monkeypatch.setattr(mr1l, "first_chunk", lambda n, ms, target=0.05: 2)
    test_scheme_bit_exact(P, golden)


@pytest.mark.parametrize("K", [1, 2, 3, 5, 7, 33, 65, 97, 129, 1009, 6007])
def test_dft_1d_known_answers(P, golden, K):
    v = golden[f"dft_in_{K}"]
    for direction, key in (("forward", "dft_fwd"), ("inverse", "dft_inv")):
        got = P.dft_1d(v, direction)
        ref = golden[f"{key}_{K}"]
        assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), (K, direction)


def test_dft_large_primes_vs_numpy(P):
    rng = np.random.default_rng(1)
    # 1300021 -> P = 2^22 (largest 2048-point tiles); 2097169 and 4194319 ->
    # P = 2^23, 2^24 (4096-point tiles)
    for K in (130003, 199999, 1300021, 2097169, 4194319):
        v = rng.normal(size=K) + 1j * rng.normal(size=K)
        got = P.dft_1d(v)
        ref = np.fft.fft(v)
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), K
        back = P.dft_1d(got, "inverse")
        assert np.abs(back - v).max() <= 1e-12 * np.abs(v).max()


def test_dft_mixed_radix_sizes_vs_numpy(P):
    """Bluestein lengths P = f * 2^a * 2048 (f = 3, 5, 7, 9, 25; column
    passes of length 3 .. 1600): forward and inverse DFTs within 1e-12."""
    from paper_1711_05152_b200 import _native
    rng = np.random.default_rng(2)
    seen = set()
    for f in (3, 5, 7, 9, 25):
        for a in (0, 1, 3, 5, 6):
            P1 = f << a
            if P1 > 2048:
                continue
            K = (P1 * 2048 + 1) // 2
            Pc = int(_native.query("sfft_fft_size", K))
            odd = Pc // (Pc & -Pc)
            seen.add(odd)
            v = rng.normal(size=K) + 1j * rng.normal(size=K)
            got = P.dft_1d(v)
            ref = np.fft.fft(v)
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (K, Pc)
            back = P.dft_1d(got, "inverse")
            assert np.abs(back - v).max() <= 1e-12 * np.abs(v).max(), (K, Pc)
    assert {3, 5, 7, 9, 25} <= seen


def test_scheme_bit_exact(P, golden):
    cand = golden["step_cand"].astype(np.int64)
    I = P.FrequencyIndexSet(cand, _presorted=True)
    sch, attempts = P.build_multiple_lattice_with_retries(
        I, P.MLConfig(), int(golden["step_b"][0]), np.random.SeedSequence(int(golden["step_seed"][0])))
    assert [lat.m for lat in sch.lattices] == golden["step_ms"].tolist()
    assert np.array_equal(np.stack([lat.z for lat in sch.lattices]), golden["step_zs"])
    words = np.zeros(len(cand), dtype=np.uint64)
    for l, mk in enumerate(sch.recon_masks):
        words |= mk.astype(np.uint64) << np.uint64(l)
    assert np.array_equal(words, golden["step_masks"])
    assert attempts == int(golden["step_attempts"][0])


def test_build_multiple_lattice_rng_state(P):
    # the caller's generator ends where the reference leaves it (construct.py:173-181)
    rng = np.random.default_rng(3)
    J = P.FrequencyIndexSet(np.random.default_rng(4).integers(-20, 21, size=(800, 4)))
    sch = P.build_multiple_lattice(J, P.MLConfig(), rng)
    from oracle import sfft_oracle as O
    rng2 = np.random.default_rng(3)
    ref = O.build_multiple_lattice(J.freqs, rng2)
    assert [lat.m for lat in sch.lattices] == ref.ms
    assert rng.random() == rng2.random()


def test_invert_multiple_matches_golden(P, golden):
    cand = golden["step_cand"].astype(np.int64)
    ms, zs = golden["step_ms"], golden["step_zs"]
    words = golden["step_masks"]
    masks = [((words >> np.uint64(l)) & np.uint64(1)).astype(bool) for l in range(len(ms))]
    I = P.FrequencyIndexSet(cand, _presorted=True)
    lats = [P.Rank1Lattice(z, int(m)) for z, m in zip(zs, ms)]
    ml = P.MultipleRank1Lattice(lats, [P.FrequencyIndexSet(cand[mk], 10, _presorted=True) for mk in masks], I,
                                recon_masks=masks)
    oracle = P.SparsePolynomialOracle(golden["step_hf"], golden["step_hc"])
    samples = [P.LatticeSamples(lat, oracle(P.lattice_nodes(lat))) for lat in lats]
    assert np.abs(samples[0].values[:256] - golden["step_first_samples"]).max() <= 1e-12
    spec = P.invert_multiple(samples, ml)
    assert np.array_equal(spec.freqs, golden["step_cov_freqs"].astype(np.int64))
    assert _rel(spec.coeffs, golden["step_coef"]) <= COEF_RTOL


def test_mr1l_step_device_path(P, golden):
    """Fused device step (K3 + K1 + K2 + K4) on the config-1-shaped fixture."""
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, compact, run_step
    dev = get_device()
    cand = golden["step_cand"].astype(np.int64)
    oracle = P.SparsePolynomialOracle(golden["step_hf"], golden["step_hc"])
    dc = DeviceFreqs.from_host(dev, cand)
    sch = build_scheme(dev, dc, int(golden["step_b"][0]), np.random.SeedSequence(int(golden["step_seed"][0])))
    assert sch.primes[: sch.L] == golden["step_ms"].tolist()
    res = run_step(dev, oracle, dc, sch, [np.zeros(0)], 10, 1e-12, len(cand))
    coef = dev.download(res.coef[0])
    coef = coef[:, 0] + 1j * coef[:, 1]
    words = dev.download(sch.masks).view(np.uint64)
    cov = words != 0
    assert _rel(coef[cov], golden["step_coef"]) <= COEF_RTOL
    rows, _ = compact(dev, dc, res.keep[0], 1)
    assert np.array_equal(rows.to_host(dev), golden["step_sel"].astype(np.int64))


def test_mr1l_step_prepared_and_deferred_cap(P, golden):
    """run_step(prep=prepare_step(...), defer_cap=True) is bit-identical to the
    default path, including a binding cap (exact radix select, detect.py:205-211)
    whose survivors match the oracle's _select."""
    from oracle import sfft_oracle as O
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, compact, prepare_step, run_step
    dev = get_device()
    cand = golden["step_cand"].astype(np.int64)
    oracle = P.SparsePolynomialOracle(golden["step_hf"], golden["step_hc"])
    dc = DeviceFreqs.from_host(dev, cand)
    seed = int(golden["step_seed"][0])
    b = int(golden["step_b"][0])
    for cap in (len(cand), 37):
        sch = build_scheme(dev, dc, b, np.random.SeedSequence(seed))
        ref = run_step(dev, oracle, dc, sch, [np.zeros(0)], 10, 1e-12, cap)
        sch2 = build_scheme(dev, dc, b, np.random.SeedSequence(seed),
                            prepare=lambda ms, z: prepare_step(dev, oracle, dc, 1, ms, z))
        assert sch2.prep is not None and sch2.L == sch.L
        got = run_step(dev, oracle, dc, sch2, [np.zeros(0)], 10, 1e-12, cap, defer_cap=True, prep=sch2.prep)
        assert np.array_equal(got.counts, ref.counts)  # .counts finalizes (applies the cap)
        assert np.array_equal(dev.download(got.coef[0]), dev.download(ref.coef[0]))
        assert np.array_equal(dev.download(got.keep[0]), dev.download(ref.keep[0]))
        rows, _ = compact(dev, dc, got.keep[0], 1)
        coef = dev.download(ref.coef[0])
        coef = coef[:, 0] + 1j * coef[:, 1]
        cov = dev.download(sch.masks).view(np.uint64) != 0
        want, _ = O.select(cand[cov], coef[cov], cap, 1e-12)  # magnitude order when the cap binds
        want = want[np.lexsort(want.T[::-1])]                 # compaction keeps candidate (lex) order
        assert len(want) == min(cap, len(want)) and np.array_equal(rows.to_host(dev), want)


@pytest.mark.gpu
def test_prepared_operands_only_for_first_attempt(P, golden):
    """Operands and tensor-core B panels prepared beside the alias kernel
    belong to the first attempt's generating vectors: a scheme from a later
    attempt (construct.py:185-206 retries) must not consume them."""
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, prepare_step, run_step
    dev = get_device()
    cand = golden["step_cand"].astype(np.int64)
    oracle = P.SparsePolynomialOracle(golden["step_hf"], golden["step_hc"])
    dc = DeviceFreqs.from_host(dev, cand)
    seed = int(golden["step_seed"][0])
    b = int(golden["step_b"][0])
    tails = [np.zeros(0)]
    first = build_scheme(dev, dc, b, np.random.SeedSequence(seed),
                         prepare=lambda ms, z: prepare_step(dev, oracle, dc, 1, ms, z, tails=tails, d=10))
    assert first.prep is not None and first.prep.poly_ready
    other = build_scheme(dev, dc, b, np.random.SeedSequence(seed + 1))
    assert not np.array_equal(other.z, first.z)
    other.attempts = 2  # as if the first attempt had failed
    ref = run_step(dev, oracle, dc, other, tails, 10, 1e-12, len(cand))
    got = run_step(dev, oracle, dc, other, tails, 10, 1e-12, len(cand), prep=first.prep)
    assert np.array_equal(dev.download(got.coef[0]), dev.download(ref.coef[0]))
    assert np.array_equal(dev.download(got.keep[0]), dev.download(ref.keep[0]))


def test_prepared_step_when_first_chunk_does_not_cover(P, golden, monkeypatch):
    """A first alias chunk that leaves candidates uncovered: the second chunk
    runs, L exceeds the prepared lattices, and the step falls back to its own
    operands — same masks, L and results as the one-pass default."""
    from paper_1711_05152_b200 import mr1l
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, prepare_step, run_step
    dev = get_device()
    cand = golden["step_cand"].astype(np.int64)
    oracle = P.SparsePolynomialOracle(golden["step_hf"], golden["step_hc"])
    dc = DeviceFreqs.from_host(dev, cand)
    seed, b = int(golden["step_seed"][0]), int(golden["step_b"][0])
    tails = [np.zeros(0)]
    sch = build_scheme(dev, dc, b, np.random.SeedSequence(seed))
    ref = run_step(dev, oracle, dc, sch, tails, 10, 1e-12, len(cand))
    monkeypatch.setattr(mr1l, "first_chunk", lambda n, ms, target=0.05: 3)
    sch2 = build_scheme(dev, dc, b, np.random.SeedSequence(seed), lazy_streams=False,
                        prepare=lambda ms, z: prepare_step(dev, oracle, dc, 1, ms, z, tails=tails, d=10))
    assert sch2.prep is not None and sch2.prep.l_max == 3 < sch2.L == sch.L
    used = np.uint64((1 << sch.L) - 1)  # bits of lattices past L differ (evaluated by one run only), unused
    assert np.array_equal(dev.download(sch2.masks).view(np.uint64) & used, dev.download(sch.masks).view(np.uint64) & used)
    got = run_step(dev, oracle, dc, sch2, tails, 10, 1e-12, len(cand), prep=sch2.prep)
    assert np.array_equal(dev.download(got.coef[0]), dev.download(ref.coef[0]))
    assert np.array_equal(dev.download(got.keep[0]), dev.download(ref.keep[0]))


def _check_report(golden, key, rep, exact_coef=True):
    assert np.array_equal(rep.detected.freqs, golden[f"{key}_freqs"]), key
    ref = golden[f"{key}_coef"]
    if len(ref) and exact_coef:
        assert _rel(rep.detected.coeffs, ref) <= COEF_RTOL, key
    cnt = golden[f"{key}_counts"]
    assert rep.candidate_counts == cnt[0].tolist()
    assert rep.prefix_counts == cnt[1].tolist()
    assert rep.component_counts == cnt[2].tolist()
    assert rep.scheme_sizes == cnt[3].tolist()
    assert rep.lattice_attempts == cnt[4].tolist()
    assert rep.inversion_calls == cnt[5].tolist()
    assert rep.oracle_calls == int(golden[f"{key}_calls"][0])


def test_sparse_fft_config0(P, golden):
    oracle = P.SparsePolynomialOracle(golden["cfg0_hf"], golden["cfg0_hc"])
    cfg = P.DetectionConfig(box=P.SearchBox.centered(5, 16), delta=1e-12, s=100, r=2, b=10,
                            rng_seed=int(golden["cfg0_seed"][0]))
    rep = P.sparse_fft(oracle, cfg)
    _check_report(golden, "cfg0", rep)
    assert oracle.call_count == rep.oracle_calls


def test_sparse_fft_host_callback(P, golden):
    """Arbitrary Python oracle: nodes from the device, values from the callback."""
    from oracle import sfft_oracle as O
    f, c = golden["cfg0_hf"], golden["cfg0_hc"]
    oracle = P.SignalOracle(5, lambda p: O.poly_eval(f, c, p))
    cfg = P.DetectionConfig(box=P.SearchBox.centered(5, 16), delta=1e-12, s=100, r=2, b=10,
                            rng_seed=int(golden["cfg0_seed"][0]))
    rep = P.sparse_fft(oracle, cfg)
    _check_report(golden, "cfg0", rep)
    assert oracle.call_count == rep.oracle_calls


def test_sparse_fft_edge_cases(P, golden):
    cases = {
        "cap": (3, dict(box=P.SearchBox.centered(3, 6), delta=1e-12, s=10, s_local=12, r=2, b=5, rng_seed=7)),
        "zero": (3, dict(box=P.SearchBox.centered(3, 5), delta=1e-12, s=len(golden["zero_hf"]), r=1, b=10,
                         mode="deterministic_zero_anchor")),
        "perm": (3, dict(box=P.SearchBox.centered(3, 6), delta=1e-12, s=8, r=1, b=10, rng_seed=11,
                         dimension_order=(2, 0, 1))),
        "one": (1, dict(box=P.SearchBox.centered(1, 5), delta=1e-12, s=3, b=5)),
    }
    for key, (d, kw) in cases.items():
        oracle = P.SparsePolynomialOracle(golden[f"{key}_hf"], golden[f"{key}_hc"])
        rep = P.sparse_fft(oracle, P.DetectionConfig(**kw))
        _check_report(golden, key, rep)


def test_sparse_fft_noisy_same_realisation(P, golden):
    oracle = P.NoisyOracle(P.SparsePolynomialOracle(golden["noisy_hf"], golden["noisy_hc"]),
                           P.sigma_for_snr(20, 30.0), seed=123)
    cfg = P.DetectionConfig(box=P.SearchBox.centered(4, 8), delta=0.3, s=20, r=3, b=10, rng_seed=5)
    rep = P.sparse_fft(oracle, cfg)
    _check_report(golden, "noisy", rep)
    assert oracle.call_count == rep.oracle_calls


def test_sparse_fft_bspline(P, golden):
    g = golden["bs_groups"]
    groups = tuple((int(row[0]), tuple(int(x) for x in row[1:] if x >= 0)) for row in g)
    oracle = P.bspline_test_function(groups)
    cfg = P.DetectionConfig(box=P.SearchBox.centered(10, 8, check_cardinality=False), delta=1e-4, s=200, r=2,
                            b=10, rng_seed=3)
    c0 = oracle.call_count
    rep = P.sparse_fft(oracle, cfg)
    assert oracle.call_count - c0 == rep.oracle_calls  # the audit (detect.py:421) incl. batched line nodes
    got = set(map(tuple, rep.detected.freqs.tolist()))
    ref = set(map(tuple, golden["bs_freqs"].tolist()))
    # parity modulo exact-magnitude +-k ties at the cap boundary (SURVEY §7 hard part 5)
    assert len(got ^ ref) <= 4
    err = P.relative_l2_error(rep.detected, oracle.exact_coefficients, oracle.norm_sq())
    assert abs(err - float(golden["bs_l2err"][0])) <= 1e-4 * float(golden["bs_l2err"][0])


def test_single_lattice_path(P, golden):
    """Algorithm 5: CBC lattices bit-exact, eval_on_lattice / invert_single,
    and a lattice_kind='single' run (reference construct.py:212-278,
    transform.py:67-96, detect.py:269-271)."""
    for i in range(5):
        lat = P.build_single_lattice_cbc(P.FrequencyIndexSet(golden[f"cbc{i}_rows"]))
        assert lat.m == int(golden[f"cbc{i}_m"][0]) and np.array_equal(lat.z, golden[f"cbc{i}_z"])
    rows = golden["cbc3_rows"]
    lat = P.Rank1Lattice(golden["cbc3_z"], int(golden["cbc3_m"][0]))
    spec = P.SparseSpectrum(rows, golden["single_coef"])
    samples = P.eval_on_lattice(spec, lat)
    ref = golden["single_eval"]
    assert np.abs(samples.values - ref).max() <= 1e-12 * np.abs(ref).max()
    inv = P.invert_single(P.LatticeSamples(lat, ref), spec.support())
    assert np.abs(inv.coeffs - golden["single_inv"]).max() <= 1e-12
    oracle = P.SparsePolynomialOracle(golden["sk_hf"], golden["sk_hc"])
    cfg = P.DetectionConfig(box=P.SearchBox.centered(3, 8), delta=1e-12, s=15, r=1, b=10, rng_seed=9,
                            lattice_kind="single")
    _check_report(golden, "sk", P.sparse_fft(oracle, cfg))


def test_bspline_points(P, golden):
    f = P.bspline_test_function()
    got = f(golden["bsv_pts"])
    ref = golden["bsv_vals"]
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


def test_projected_line_coefficients(P, golden):
    oracle = P.SparsePolynomialOracle(golden["line_hf"], golden["line_hc"])
    box = P.SearchBox([-4, -5, -3], [4, 5, 3])
    for t in range(3):
        ks, c = P.projected_line_coefficients(oracle, t, box, golden["line_anchor"])
        assert np.array_equal(ks, golden[f"line_{t}_ks"])
        assert np.abs(c - golden[f"line_{t}_c"]).max() <= 1e-12


def test_oracle_errors(P):
    def broken(points):
        raise RuntimeError("sensor offline")

    cfg = P.DetectionConfig(box=P.SearchBox.centered(2, 3), delta=1e-12, s=5)
    with pytest.raises(RuntimeError, match="step 0, iteration 0"):
        P.sparse_fft(P.SignalOracle(2, broken), cfg)

    class Stop(P.OracleInterrupt):
        pass

    def bail(points):
        raise Stop("enough")

    with pytest.raises(Stop):
        P.sparse_fft(P.SignalOracle(2, bail), cfg)


def test_zero_signal(P):
    oracle = P.SignalOracle(3, lambda pts: np.zeros(len(pts), dtype=complex))
    rep = P.sparse_fft(oracle, P.DetectionConfig(box=P.SearchBox.centered(3, 4), delta=1e-12, s=5, b=5))
    assert len(rep.detected) == 0
    assert rep.oracle_calls == oracle.call_count


def test_config2_full_size_matches_reference_run(P):
    """BASELINE config 2 at full size on the instance the survey ran through the
    unmodified reference (seed 42 / rng_seed 43, r = 5; SURVEY §6.3 and
    BASELINE.md §3.1: 3127.5 s on the CPU).  Every per-step candidate count,
    every scheme size and the total oracle-call audit are the reference's."""
    truth, oracle = P.gen_random_sparse_poly(10, 32, 1000, "box", seed=42)
    cfg = P.DetectionConfig(box=P.SearchBox.centered(10, 32), delta=1e-12, s=1000, r=5, b=10, rng_seed=43)
    rep = P.sparse_fft(oracle, cfg)
    assert rep.candidate_counts == [65, 4225, 58370, 64935] + [65000] * 6
    assert rep.scheme_sizes == [0, 16928, 1284863, 1689355, 1040344, 1821004, 1430609, 1170423, 1170423,
                                1560730]
    assert rep.lattice_attempts == [0] + [1] * 9
    assert rep.oracle_calls == 49_683_725
    assert rep.detected.support() == truth.support()
    assert P.relative_spectrum_l2_error(rep.detected, truth) <= 1e-14


def test_config1_full_size(P):
    """BASELINE config 1 at full size: |J| = 100000, d = 10, 2000 nonzero.
    Masks bit-exact against the CPU oracle; coefficients against the truth."""
    from oracle import sfft_oracle as O
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, run_step
    wl = workloads.config1()
    dev = get_device()
    dc = DeviceFreqs.from_host(dev, wl.cand)
    sch = build_scheme(dev, dc, wl.b, np.random.SeedSequence(wl.lattice_seed))
    ref = O.build_with_retries(wl.cand, wl.b, np.random.SeedSequence(wl.lattice_seed))
    assert sch.primes[: sch.L] == ref.ms and sch.uncovered == 0
    words = dev.download(sch.masks).view(np.uint64)
    for l, mk in enumerate(ref.masks):
        assert np.array_equal(((words >> np.uint64(l)) & np.uint64(1)).astype(bool), mk)
    res = run_step(dev, wl.oracle, dc, sch, [np.zeros(0)], 10, wl.delta, len(wl.cand))
    coef = dev.download(res.coef[0])
    coef = coef[:, 0] + 1j * coef[:, 1]
    assert _rel(coef, wl.truth_coef) <= COEF_RTOL
    keep = dev.download(res.keep[0]).astype(bool)
    assert np.array_equal(keep, wl.truth_coef != 0)
