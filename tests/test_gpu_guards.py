"""Out-of-bounds guard checks of the device path (compute-sanitizer is not
available on this GPU pool).

Every buffer the engine allocates through Device.empty / Device.zeros gets a
256-byte guard region on both sides, filled with a sentinel; the kernels
see exactly the sizes the engine asks for.  After full runs (config-0
sparse_fft, a capped run, a B-spline run, a noisy run, a config-1-shaped MR1L
step, lines longer than 1024 points, a sharded step with simulated ranks)
every guard byte must be intact: no kernel wrote outside its buffers."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GUARD = 256
SENTINEL = 0xA5


class _Guarded:
    def __init__(self, dev):
        self.dev = dev
        self.bufs = []
        self.real_empty, self.real_zeros = dev.empty, dev.zeros

    def empty(self, shape, dtype, fill=None):
        torch = self.dev.torch
        shape = tuple(int(x) for x in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        numel = int(np.prod(shape)) if shape else 1
        nbytes = numel * torch.empty((), dtype=dtype).element_size()
        raw = torch.full((nbytes + 2 * GUARD,), SENTINEL, dtype=torch.uint8, device=self.dev.device)
        inner = raw[GUARD:GUARD + nbytes]
        if fill is not None:
            inner.fill_(fill)
        self.bufs.append((raw, nbytes, shape, str(dtype)))
        return inner.view(dtype).reshape(shape)

    def zeros(self, shape, dtype):
        return self.empty(shape, dtype, fill=0)

    def __enter__(self):
        self.dev.empty, self.dev.zeros = self.empty, self.zeros
        return self

    def __exit__(self, *exc):
        self.dev.empty, self.dev.zeros = self.real_empty, self.real_zeros
        return False

    def check(self):
        self.dev.sync()
        bad = []
        for raw, nbytes, shape, dt in self.bufs:
            head = raw[:GUARD]
            tail = raw[GUARD + nbytes:]
            if bool((head != SENTINEL).any()) or bool((tail != SENTINEL).any()):
                bad.append((shape, dt))
        assert not bad, f"kernels wrote outside {len(bad)} buffers: {bad[:5]}"
        return len(self.bufs)


@pytest.fixture
def guarded():
    from paper_1711_05152_b200 import mr1l
    from paper_1711_05152_b200.device import get_device
    dev = get_device()
    mr1l.clear_caches(dev)  # tables allocated under guard too
    with _Guarded(dev) as g:
        yield g
    mr1l.clear_caches(dev)


def test_guards_sparse_fft_runs(guarded):
    import paper_1711_05152_b200 as P
    from paper_1711_05152_b200 import workloads
    w0 = workloads.config0()
    rep = P.sparse_fft(w0.oracle, w0.cfg)
    assert rep.detected.support() == w0.truth.support()
    truth, oracle = P.gen_random_sparse_poly(3, 6, 25, "box", seed=np.random.default_rng(42))
    P.sparse_fft(oracle, P.DetectionConfig(box=P.SearchBox.centered(3, 6), delta=1e-12, s=10, s_local=12, r=2,
                                           b=5, rng_seed=7))
    P.sparse_fft(P.bspline_test_function(), P.DetectionConfig(box=P.SearchBox.centered(10, 8,
                                                                                        check_cardinality=False),
                                                                delta=1e-4, s=200, r=2, b=10, rng_seed=3))
    truth, poly = P.gen_random_sparse_poly(4, 8, 20, "unit_modulus", seed=np.random.default_rng(9))
    for dev_rng in (False, True):
        P.sparse_fft(P.RelativeNoisyOracle(poly, 1e-2, seed=1, device_rng=dev_rng),
                     P.DetectionConfig(box=P.SearchBox.centered(4, 8), delta=0.3, s=20, r=3, b=10, rng_seed=5))
    truth, oracle = P.gen_random_sparse_poly(2, 700, 12, "box", seed=np.random.default_rng(71))
    P.sparse_fft(oracle, P.DetectionConfig(box=P.SearchBox.centered(2, 700), delta=1e-12, s=12, r=2, b=10,
                                           rng_seed=5))
    assert guarded.check() > 100


def test_guards_mr1l_step_and_sharded(guarded):
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, prepare_step, run_step
    from paper_1711_05152_b200.parallel import Shard, run_step_sharded
    dev = guarded.dev
    wl = workloads.config1(seed=2, n=12000, nnz=200)
    cand = DeviceFreqs.from_host(dev, wl.cand)
    tails = [np.zeros(0)]
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), lazy_streams=True,
                       prepare=lambda ms, z: prepare_step(dev, wl.oracle, cand, 1, ms, z, tails=tails, d=10))
    ref = run_step(dev, wl.oracle, cand, sch, tails, 10, 1e-12, 50, prep=sch.prep, defer_cap=True)
    ref.finalize()
    got = run_step_sharded(dev, wl.oracle, cand, sch, tails, 10, 1e-12, 50, Shard(), simulate_world=3)
    assert np.array_equal(dev.download(ref.keep), dev.download(got.keep))
    assert guarded.check() > 20
