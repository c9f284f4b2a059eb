"""Sharded MR1L step (parallel.py) on one GPU with simulated ranks: the units
of a step dealt over W ranks, rows gathered per rank and combined in lattice
order must equal the single-GPU step bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_step_bit_identical(world):
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, run_step
    from paper_1711_05152_b200.parallel import Shard, run_step_sharded
    dev = get_device()
    wl = workloads.config1(seed=5, n=20000, nnz=300)
    cand = DeviceFreqs.from_host(dev, wl.cand)
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed))
    # 3 anchored iterations on a 10-D oracle seen from a 7-D candidate set
    cand7 = DeviceFreqs.from_host(dev, np.unique(wl.cand[:, :7], axis=0))
    sch7 = build_scheme(dev, cand7, wl.b, np.random.SeedSequence(11))
    rng = np.random.default_rng(0)
    tails = [rng.random(3) for _ in range(3)]
    for c, s, tl in ((cand, sch, [np.zeros(0)]), (cand7, sch7, tails)):
        ref = run_step(dev, wl.oracle, c, s, tl, 10, 1e-12, c.n)
        got = run_step_sharded(dev, wl.oracle, c, s, tl, 10, 1e-12, c.n, Shard(), simulate_world=world)
        assert np.array_equal(dev.download(ref.coef), dev.download(got.coef))
        assert np.array_equal(dev.download(ref.keep), dev.download(got.keep))
        assert np.array_equal(ref.counts, got.counts)
