"""Host-side logic (CPU only): the reference-mirroring types, lattice-size
selection, configuration validation, planners/bounds, seeded workloads and
the RNG-stream contract the engine relies on for bit-exact schemes."""

import numpy as np
import pytest

import paper_1711_05152_b200 as P
from oracle import sfft_oracle as O
from paper_1711_05152_b200 import workloads


class TestTypes:
    def test_frequency_set_sorted_unique(self):
        I = P.FrequencyIndexSet([[2, 1], [0, 5], [2, 1], [-1, 7]])
        assert I.freqs.tolist() == [[-1, 7], [0, 5], [2, 1]]
        assert not I.freqs.flags.writeable
        assert I.expansion() == 6 and I.expansion(0) == 3
        assert (0, 5) in I and (5, 0) not in I
        assert I.positions_of(P.FrequencyIndexSet([[2, 1]])).tolist() == [2]
        with pytest.raises(ValueError):
            P.FrequencyIndexSet([])
        assert len(P.FrequencyIndexSet([], 3)) == 0
        with pytest.raises(ValueError):
            P.FrequencyIndexSet([[2**31, 0]])

    def test_union_project(self):
        a = P.FrequencyIndexSet([[1, 2, 3], [0, 0, 0]])
        b = P.FrequencyIndexSet([[1, 2, 3], [5, 5, 5]])
        assert len(a.union(b)) == 3
        assert a.project((2, 0)).freqs.tolist() == [[0, 0], [3, 1]]
        with pytest.raises(ValueError):
            a.project((0, 0))

    def test_search_box(self):
        box = P.SearchBox.centered(3, 4)
        assert box.sizes.tolist() == [9, 9, 9] and box.cardinality == 729
        assert box.contains(np.array([[4, -4, 0], [5, 0, 0]])).tolist() == [True, False]
        with pytest.raises(ValueError):
            P.SearchBox([1], [0])
        with pytest.raises(ValueError):
            P.SearchBox.centered(20, 32)  # u64 guard of the reference (lattice.py:204-208)
        big = P.SearchBox.centered(20, 32, check_cardinality=False)
        assert big.dim == 20 and big.max_abs == 32
        perm = P.SearchBox([0, -1, -2], [1, 2, 3]).permute((2, 0, 1))
        assert perm.lows.tolist() == [-2, 0, -1]

    def test_rank1_lattice_and_spectrum(self):
        lat = P.Rank1Lattice([7, -1], 5)
        assert lat.z.tolist() == [2, 4] and lat.m == 5
        with pytest.raises(ValueError):
            P.Rank1Lattice([1], 0)
        spec = P.SparseSpectrum([(1, 0), (0, 1)], [2.0, 1j])
        assert spec.freqs.tolist() == [[0, 1], [1, 0]]
        assert spec[(1, 0)] == 2.0 and spec.get((5, 5)) == 0.0
        assert spec.energy() == pytest.approx(5.0)
        with pytest.raises(ValueError):
            P.SparseSpectrum([(1, 0), (1, 0)], [1, 2])
        assert len(spec.restrict(1.5)) == 1

    def test_multiple_lattice_masks(self):
        I = P.FrequencyIndexSet([[0, 0], [1, 0], [0, 1]])
        lats = [P.Rank1Lattice([1, 1], 3), P.Rank1Lattice([1, 2], 3)]
        rs = [P.FrequencyIndexSet([[0, 0]]), P.FrequencyIndexSet([[1, 0], [0, 1]])]
        ml = P.MultipleRank1Lattice(lats, rs, I)
        assert ml.total_size == 6 and ml.is_reconstructing
        assert [m.tolist() for m in ml.recon_masks] == [[True, False, False], [False, True, True]]


class TestPrimes:
    def test_pins(self, golden):
        rows = np.array([[0, 0], [40, 1], [-40, 2], [3, -40]])
        I = P.FrequencyIndexSet(rows)
        assert P.candidate_primes(I, 2 * (len(I) - 1), 6) == golden["primes_small"].tolist()
        rng = np.random.default_rng(5)
        J = P.FrequencyIndexSet(rng.integers(-32, 33, size=(5000, 10)))
        assert P.candidate_primes(J, 2 * (len(J) - 1), 19) == golden["primes_5000"].tolist()

    def test_mlconfig(self, golden):
        cfg = P.MLConfig()
        assert [cfg.max_lattices(n) for n in (1, 2, 1000, 65000, 100000, 650000)] == golden["lmax_pins"].tolist()
        assert cfg.max_lattices(1) == 2 and cfg.max_lattices(1000) == 16
        assert cfg.size_lower_bound(10) == 18.0
        with pytest.raises(ValueError):
            P.MLConfig(c=1.0)
        with pytest.raises(ValueError):
            P.MLConfig(gamma=1.0)

    def test_primes_above_matches_oracle(self):
        from paper_1711_05152_b200.primes import primes_above
        for bound in (0, 1, 2.5, 1000, 199998, 1299998):
            assert primes_above(bound, 25) == O.primes_above(bound, 25)


class TestConfig:
    def test_detection_config_validation(self):
        box = P.SearchBox.centered(2, 4)
        cfg = P.DetectionConfig(box=box, delta=1e-3, s=5)
        assert cfg.local_sparsity == 5 and cfg.component_threshold == 1e-3
        for bad in (dict(delta=0.0), dict(s=0), dict(r=0), dict(b=0), dict(mode="x"),
                    dict(lattice_kind="triple"), dict(dimension_order=(0, 0)), dict(s_local=0),
                    dict(component_delta=0.0), dict(rng_seed=-1)):
            kw = dict(box=box, delta=1e-3, s=5)
            kw.update(bad)
            with pytest.raises(ValueError):
                P.DetectionConfig(**kw)
        with pytest.raises(TypeError):
            P.DetectionConfig(box="grid", delta=1e-3, s=5)

    def test_planners_and_bounds(self):
        assert P.plan_r(1000, 10, 0.01, "multiple") == 29829
        assert P.plan_r(1, 1, 0.999999) == 3
        assert P.plan_r(1000, 10, 0.01, "single") < P.plan_r(1000, 10, 0.01)
        assert P.plan_b(10, 0.01, 0.5) == 12
        assert P.plan_b(10, 0.01, 1e-9) == 1
        assert P.failure_bound_single_coeff([1.0, 1.0, 1.0], 0.0) == pytest.approx(2 / 3)
        assert P.union_failure_bound(0.5, 2, 10, 4) == pytest.approx(1.0)
        with pytest.raises(ValueError):
            P.failure_bound_single_coeff([0.5, 0.5], 0.5)


class TestWorkloadsAndRng:
    def test_generator_matches_reference_draws(self, golden):
        wl = workloads.config0()
        assert np.array_equal(wl.truth.freqs, golden["cfg0_hf"])
        assert np.array_equal(wl.truth.coeffs, golden["cfg0_hc"])
        assert wl.cfg.rng_seed == int(golden["cfg0_seed"][0])
        assert np.abs(wl.truth.coeffs).min() >= 1e-3

    def test_config_shapes(self):
        s1 = workloads.config1(n=5000, nnz=100)
        assert s1.cand.shape == (5000, 10) and len(np.unique(s1.cand, axis=0)) == 5000
        assert np.array_equal(s1.cand, O.lexsort_rows(s1.cand))
        assert (s1.truth_coef != 0).sum() == 100 and s1.oracle.s == 100
        w3 = workloads.config3(s=50)
        assert w3.cfg.box.dim == 20 and w3.oracle.rel == 1e-2
        assert np.all(np.abs(np.abs(w3.truth.coeffs) - 1.5) <= 0.5 + 1e-12)
        w4 = workloads.config4()
        sizes = sorted(len(c) for _, c in w4.oracle.groups)
        assert sizes == [3, 3, 4] and sorted(sum((list(c) for _, c in w4.oracle.groups), [])) == list(range(10))

    def test_predrawn_vectors_are_stream_identical(self):
        # SURVEY §7 hard part 1: an attempt's generator is discarded, so drawing
        # all L_max vectors up front yields the same first L vectors
        primes = O.primes_above(9999, 19)
        seq = [np.random.default_rng(np.random.SeedSequence(3).spawn(1)[0]) for _ in range(2)]
        pre = [seq[0].integers(0, m, size=10, dtype=np.int64) for m in primes]
        one = [seq[1].integers(0, m, size=10, dtype=np.int64) for m in primes[:7]]
        assert all(np.array_equal(a, b) for a, b in zip(pre, one))

    def test_vectorised_bounded_draw_is_stream_identical(self):
        # build_scheme draws rng.integers(0, M[:, None], (L, d)) in one call; it
        # must equal the reference's per-prime rng.integers(0, m, size=d) loop
        for ms in ([2, 3, 5, 7, 11, 13], O.primes_above(100, 20), [2**31 - 1, 2**31 - 19, 2**30 + 3]):
            ms = np.asarray(ms, dtype=np.int64)
            for seed in range(3):
                a = np.random.default_rng(seed)
                b = np.random.default_rng(seed)
                loop = np.stack([a.integers(0, m, size=7, dtype=np.int64) for m in ms])
                vec = b.integers(0, ms[:, None], size=(len(ms), 7), dtype=np.int64)
                assert np.array_equal(loop, vec)
                assert a.random() == b.random()

    def test_lazy_attempt_streams_equal_spawn(self):
        from paper_1711_05152_b200.mr1l import _attempt_streams
        for parent in (np.random.SeedSequence(7), np.random.SeedSequence(3).spawn(4)[2]):
            eager = [np.random.default_rng(c).integers(0, 1 << 40, 5) for c in
                     np.random.SeedSequence(parent.entropy, spawn_key=parent.spawn_key).spawn(10)]
            lazy = [np.random.default_rng(c).integers(0, 1 << 40, 5) for c in _attempt_streams(parent, 10, True)]
            assert all(np.array_equal(a, b) for a, b in zip(eager, lazy))

    def test_speculated_first_attempt_equals_oracle_scheme(self):
        # api.reconstruct_step draws attempt 1 while the rows are in flight
        # (speculate_scheme); with every prime above the spread it must equal
        # the oracle's Algorithm 1 primes and first generating vectors
        from paper_1711_05152_b200.mr1l import speculate_scheme
        rng = np.random.default_rng(11)
        cand = O.unique_rows(rng.integers(-8, 9, size=(3000, 6)))
        g = speculate_scheme(len(cand), 6, np.random.SeedSequence(21), 10)
        assert g.primes == O.candidate_primes(cand, 2 * (len(cand) - 1), O.max_lattices(len(cand)))
        assert g.primes[0] > 16
        child = np.random.SeedSequence(21).spawn(10)[0]
        r = np.random.default_rng(child)
        want = np.stack([r.integers(0, m, size=6, dtype=np.int64) for m in g.primes])
        assert np.array_equal(g.z, want)

    def test_first_alias_chunk(self):
        # the first chunk of primes whose alias masks are evaluated before the
        # coverage check: a prefix, monotone in n, all primes when nearly all
        # would be needed; the early exit it predicts matches the oracle's
        # typical L on a config-1-shaped set
        from paper_1711_05152_b200.mr1l import first_chunk
        prev = 0
        for n in (2, 50, 1000, 20000, 100000, 650000):
            lm = O.max_lattices(n)
            ms = O.candidate_primes(np.zeros((1, 1), dtype=np.int64), 2 * (n - 1), lm)
            k = first_chunk(n, ms)
            assert 1 <= k <= lm and k != lm - 1
            assert k >= prev
            prev = k
        assert first_chunk(1, [3, 5, 7]) == 3
        rng = np.random.default_rng(5)
        cand = O.unique_rows(rng.integers(-32, 33, size=(20000, 10)))
        sch = O.build_with_retries(cand, 10, np.random.SeedSequence(9))
        assert len(sch.ms) <= first_chunk(len(cand), O.candidate_primes(cand, 2 * (len(cand) - 1),
                                                                           O.max_lattices(len(cand))))

    def test_spawn_is_stateful(self):
        ss = np.random.SeedSequence(1)
        a = ss.spawn(2)
        b = ss.spawn(2)
        assert [c.spawn_key for c in a] == [(0,), (1,)] and [c.spawn_key for c in b] == [(2,), (3,)]


class TestOracleDescriptors:
    def test_poly_permutation(self):
        o = P.SparsePolynomialOracle([[1, 2, 3]], [1.0])
        p = o.permuted((2, 0, 1))
        assert p.freqs.tolist() == [[3, 1, 2]]
        p.count_samples(5)
        assert o.call_count == 5  # shared counter

    def test_bspline_groups_permutation(self):
        b = P.bspline_test_function()
        order = tuple(range(9, -1, -1))
        pb = b.permuted(order)
        # slot t holds original component order[t]
        assert pb.groups[0] == (2, (9, 7, 2))
        assert pb.norm_sq() == pytest.approx(3.860521370158563, abs=1e-14)

    def test_bspline_exact(self, golden):
        got = P.bspline_exact_coefficients(golden["bsv_ks"])
        assert np.allclose(got, golden["bsv_exact"], rtol=0, atol=1e-16)

    def test_metrics(self):
        t = P.SparseSpectrum([(0,), (1,)], [1.0, 1.0])
        d = P.SparseSpectrum([(0,)], [1.0])
        assert P.relative_spectrum_l2_error(d, t) == pytest.approx(np.sqrt(0.5))
        assert P.sigma_for_snr(100, 20.0) == pytest.approx(1.0)

    def test_generic_callable_oracle(self):
        o = P.SignalOracle(2, lambda p: p[:, 0] + 1j * p[:, 1])
        v = o(np.array([[0.25, 0.5]]))
        assert v.tolist() == [0.25 + 0.5j] and o.call_count == 1
        with pytest.raises(ValueError):
            o(np.zeros((3, 3)))
