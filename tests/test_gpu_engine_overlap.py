"""The engine enqueues step t+1 (compaction gather with a guessed count,
candidate product, first alias kernel, preparation) during step t once the
prefix counts have settled (engine._start_next_step).  It must change
nothing: the same report, field by field, as the engine with every step
run after its predecessor's synchronisation — whether the guessed count
was right (the enqueued step is used) or wrong (it is discarded)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert np.array_equal(a.detected.freqs, b.detected.freqs)
    assert np.array_equal(a.detected.coeffs, b.detected.coeffs)
    for f in ("component_counts", "prefix_counts", "candidate_counts", "scheme_sizes", "lattice_attempts",
              "detection_calls", "inversion_calls", "warnings"):
        assert getattr(a, f) == getattr(b, f), f
    assert a.oracle_calls == b.oracle_calls


def _runs(monkeypatch, oracle, cfg):
    from paper_1711_05152_b200 import engine
    import paper_1711_05152_b200 as P
    used, made = [], []
    real_start = engine._start_next_step

    def spy(*a, **k):
        nxt = real_start(*a, **k)
        made.append(nxt is not None)
        return nxt
    monkeypatch.setattr(engine, "_start_next_step", spy)
    got = P.sparse_fft(oracle, cfg)
    monkeypatch.undo()
    real_build = engine.build_scheme
    monkeypatch.setattr(engine, "build_scheme", lambda *a, **k: real_build(*a, **k))  # disables the overlap
    ref = P.sparse_fft(oracle, cfg)
    monkeypatch.undo()
    return got, ref, made


def test_overlapped_steps_equal_sequential_config2_shape(monkeypatch):
    """d = 10, N = 32, s = 200, r = 3: the prefix counts settle at s, so the
    later steps run enqueued ahead."""
    import paper_1711_05152_b200 as P
    truth, oracle = P.gen_random_sparse_poly(10, 32, 200, "box", seed=5, min_magnitude=1e-3)
    cfg = P.DetectionConfig(box=P.SearchBox.centered(10, 32), delta=1e-12, s=200, r=3, b=10, rng_seed=9)
    got, ref, made = _runs(monkeypatch, oracle, cfg)
    _same(got, ref)
    assert sum(made) >= 4, made
    assert len(got.detected) == 200


def test_overlapped_steps_wrong_guess_discarded(monkeypatch):
    """Every started step with a wrong count guess (forced off by one) is
    discarded and the step runs after the synchronisation: same report."""
    import paper_1711_05152_b200 as P
    from paper_1711_05152_b200 import engine
    truth, oracle = P.gen_random_sparse_poly(10, 32, 200, "box", seed=5, min_magnitude=1e-3)
    cfg = P.DetectionConfig(box=P.SearchBox.centered(10, 32), delta=1e-12, s=200, r=3, b=10, rng_seed=9)
    real = engine._start_next_step
    calls = []

    def off_by_one(dev, oracle_, prefixes, pend, cnt, *a):
        if prefixes is not None:  # step 1: the exact prefix set, nothing to guess
            return real(dev, oracle_, prefixes, pend, cnt, *a)
        calls.append(cnt)
        return real(dev, oracle_, prefixes, pend, cnt + 1, *a)
    monkeypatch.setattr(engine, "_start_next_step", off_by_one)
    got = P.sparse_fft(oracle, cfg)
    monkeypatch.undo()
    real_build = engine.build_scheme
    monkeypatch.setattr(engine, "build_scheme", lambda *a, **k: real_build(*a, **k))
    ref = P.sparse_fft(oracle, cfg)
    monkeypatch.undo()
    assert len(calls) >= 4
    _same(got, ref)


def test_line_sampling_all_components_bit_identical():
    """sfft_line_sample_poly_all (every component's lines in one launch) gives
    the samples of d separate sfft_line_sample_poly calls, bit for bit."""
    import paper_1711_05152_b200 as P
    from paper_1711_05152_b200.device import dptr, get_device, hptr
    dev = get_device()
    torch = dev.torch
    truth, oracle = P.gen_random_sparse_poly(6, 20, 300, "box", seed=3, min_magnitude=1e-3)
    hf, cf = oracle.device_terms(dev)
    d, r, K = 6, 3, 41
    anchors = np.random.default_rng(2).random((d, r, d))
    ref = dev.empty((d * r, K, 2), torch.float64)
    for t in range(d):
        a = np.ascontiguousarray(anchors[t])
        dev.call("sfft_line_sample_poly", dptr(hf), dptr(cf), oracle.s, d, t, K, hptr(a), r, dptr(ref[t * r:]))
    got = dev.empty((d * r, K, 2), torch.float64)
    a_all = np.ascontiguousarray(anchors.reshape(d * r, d))
    dev.call("sfft_line_sample_poly_all", dptr(hf), dptr(cf), oracle.s, d, K, hptr(a_all), r, dptr(got))
    assert np.array_equal(dev.download(got), dev.download(ref))
    # and against the oracle itself at the line points
    pts = np.repeat(anchors.reshape(d * r, d), K, axis=0)
    for t in range(d):
        pts[t * r * K:(t + 1) * r * K, t] = np.tile(np.arange(K) / K, r)
    want = oracle(pts).reshape(d * r, K)
    g = dev.download(got)
    assert np.abs(g[..., 0] + 1j * g[..., 1] - want).max() <= 1e-10 * np.abs(want).max()


def test_line_points_bit_exact():
    """sfft_line_points builds exactly the host's line points (anchor rows,
    component t of component t's lines set to np.arange(K) / K)."""
    from paper_1711_05152_b200.device import dptr, get_device
    dev = get_device()
    d, r, K = 7, 3, 129
    anchors = np.random.default_rng(5).random((d * r, d))
    want = np.repeat(anchors, K, axis=0)
    line = np.tile(np.arange(K) / K, r)
    for t in range(d):
        want[t * r * K:(t + 1) * r * K, t] = line
    d_a = dev.upload(anchors)
    pts = dev.empty((d * r * K, d), dev.torch.float64)
    dev.call("sfft_line_points", dptr(d_a), d, r, K, dptr(pts))
    assert np.array_equal(dev.download(pts), want)
