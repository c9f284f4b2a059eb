"""A config-1 step's device buffers go when the last reference to them does
(no reference cycle through the step's preparation): device memory stays
flat over repeated steps with the cyclic garbage collector off.  (A cycle
here once let every step's ~0.8 GB of buffers pile up until a collection,
and the allocator's fresh segments cost up to milliseconds per step.)"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _step(wl, dev, cand):
    from paper_1711_05152_b200.mr1l import build_scheme, prepare_step, run_step
    tails = [np.zeros(0)]
    prepare = lambda ms, z: prepare_step(dev, wl.oracle, cand, 1, ms, z, tails=tails, d=10)  # noqa: E731
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64,
                       lazy_streams=True, prepare=prepare)
    res = run_step(dev, wl.oracle, cand, sch, tails, 10, wl.delta, len(wl.cand), prep=sch.prep).finalize()
    return sch, res


def test_step_buffers_freed_without_gc():
    import gc
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs
    dev = get_device()
    wl = workloads.config1()
    cand = DeviceFreqs.from_host(dev, wl.cand)
    _step(wl, dev, cand)
    dev.sync()
    gc.collect()
    gc.disable()
    try:
        base = dev.torch.cuda.memory_allocated(dev.device)
        for _ in range(6):
            _step(wl, dev, cand)
        dev.sync()
        grown = dev.torch.cuda.memory_allocated(dev.device) - base
    finally:
        gc.enable()
    assert grown < 64 << 20, grown


def test_api_and_engine_buffers_freed_without_gc():
    """The same for the public entry points: api.reconstruct_step (host rows
    in, host results out) and a small sparse_fft run."""
    import gc
    import paper_1711_05152_b200 as P
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.api import reconstruct_step
    from paper_1711_05152_b200.device import get_device
    dev = get_device()
    wl = workloads.config1()
    truth, oracle = P.gen_random_sparse_poly(6, 16, 60, "box", seed=3, min_magnitude=1e-3)
    cfg = P.DetectionConfig(box=P.SearchBox.centered(6, 16), delta=1e-12, s=60, r=2, b=10, rng_seed=4)

    def once():
        reconstruct_step(wl.cand, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
        P.sparse_fft(oracle, cfg)
    once()
    dev.sync()
    gc.collect()
    gc.disable()
    try:
        base = dev.torch.cuda.memory_allocated(dev.device)
        for _ in range(4):
            once()
        dev.sync()
        grown = dev.torch.cuda.memory_allocated(dev.device) - base
    finally:
        gc.enable()
    assert grown < 64 << 20, grown
