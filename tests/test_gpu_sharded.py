"""Sharded MR1L step (parallel.py) on one GPU.

1. Simulated ranks in one process: the units of a step dealt over W ranks,
   exchanged as slices (default) or dense rows, must equal the single-GPU
   step bit for bit.
2. A real process group: 2 processes on cuda:0 with gloo collectives (the
   NCCL path needs one GPU per rank; the kernels and the host bookkeeping are
   the same), run_step_sharded and sparse_fft against one rank, bit for bit."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("exchange", ["slices", "rows"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_step_bit_identical(world, exchange):
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
    for c, s, tl, cap in ((cand, sch, [np.zeros(0)], cand.n), (cand7, sch7, tails, cand7.n), (cand7, sch7, tails, 57)):
        ref = run_step(dev, wl.oracle, c, s, tl, 10, 1e-12, cap)
        got = run_step_sharded(dev, wl.oracle, c, s, tl, 10, 1e-12, cap, Shard(), simulate_world=world,
                               exchange=exchange)
        assert np.array_equal(dev.download(ref.coef), dev.download(got.coef))
        assert np.array_equal(dev.download(ref.keep), dev.download(got.keep))
        assert np.array_equal(ref.counts, got.counts)


def test_sharded_step_with_preparation():
    """The step preparation made beside the alias kernel (tables, prepared
    sampling operands and B panels, buffers) is used by the sharded step too."""
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, prepare_step, run_step
    from paper_1711_05152_b200.parallel import Shard, run_step_sharded
    dev = get_device()
    wl = workloads.config1(seed=6, n=30000, nnz=400)
    cand = DeviceFreqs.from_host(dev, wl.cand)
    tails = [np.zeros(0)]
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), lazy_streams=True,
                       prepare=lambda ms, z: prepare_step(dev, wl.oracle, cand, 1, ms, z, tails=tails, d=10))
    assert sch.prep is not None and sch.prep.poly_ready
    ref = run_step(dev, wl.oracle, cand, sch, tails, 10, 1e-12, cand.n)
    for world in (2, 4):
        got = run_step_sharded(dev, wl.oracle, cand, sch, tails, 10, 1e-12, cand.n, Shard(), simulate_world=world,
                               prep=sch.prep)
        assert np.array_equal(dev.download(ref.coef), dev.download(got.coef))
        assert np.array_equal(dev.download(ref.keep), dev.download(got.keep))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _noisy_runs(P):
    """Noisy oracles through a sharded step: every rank consumes the whole
    numpy noise stream / the whole call-index range (parallel._align_noise)."""
    truth, poly = P.gen_random_sparse_poly(4, 8, 20, "unit_modulus", seed=np.random.default_rng(9))
    cfg = P.DetectionConfig(box=P.SearchBox.centered(4, 8), delta=0.3, s=20, r=3, b=10, rng_seed=5)
    return [(P.NoisyOracle(poly, P.sigma_for_snr(20, 30.0), seed=123), cfg),
            (P.RelativeNoisyOracle(poly, 1e-2, seed=7, device_rng=True), cfg)]


def _mp_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1711_05152_b200 as P
        from paper_1711_05152_b200 import workloads
        from paper_1711_05152_b200.device import get_device
        from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme
        from paper_1711_05152_b200.parallel import Shard, run_step_sharded
        dev = get_device()
        wl = workloads.config1(seed=5, n=20000, nnz=300)
        cand = DeviceFreqs.from_host(dev, wl.cand)
        sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed))
        res = run_step_sharded(dev, wl.oracle, cand, sch, [np.zeros(0)], 10, 1e-12, cand.n, Shard())
        coef, keep = dev.download(res.coef), dev.download(res.keep)
        w0 = workloads.config0()
        rep = P.sparse_fft(w0.oracle, w0.cfg)  # sharded over the process group
        noisy = [P.sparse_fft(o, c).detected for o, c in _noisy_runs(P)]
        q.put((rank, coef, keep, rep.detected.freqs, rep.detected.coeffs, rep.oracle_calls,
               rep.candidate_counts, rep.scheme_sizes, [(x.freqs, x.coeffs) for x in noisy]))
    except Exception as exc:  # surface the worker's error in the test
        q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_process_group_on_one_gpu_bit_identical():
    import multiprocessing as mp
    import paper_1711_05152_b200 as P
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, run_step
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=500) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for g in got:
        assert len(g) > 2, g
    dev = get_device()
    wl = workloads.config1(seed=5, n=20000, nnz=300)
    cand = DeviceFreqs.from_host(dev, wl.cand)
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed))
    ref = run_step(dev, wl.oracle, cand, sch, [np.zeros(0)], 10, 1e-12, cand.n)
    w0 = workloads.config0()
    rep = P.sparse_fft(w0.oracle, w0.cfg)
    noisy = [P.sparse_fft(o, c).detected for o, c in _noisy_runs(P)]
    for rank, coef, keep, f, c, calls, cc, ss, nz in got:
        assert np.array_equal(coef, dev.download(ref.coef)), rank
        assert np.array_equal(keep, dev.download(ref.keep)), rank
        assert np.array_equal(f, rep.detected.freqs) and np.array_equal(c, rep.detected.coeffs), rank
        assert calls == rep.oracle_calls and cc == rep.candidate_counts and ss == rep.scheme_sizes
        for (nf, nc), one in zip(nz, noisy):
            assert np.array_equal(nf, one.freqs) and np.array_equal(nc, one.coeffs), rank
    for p in procs:
        assert p.exitcode == 0
