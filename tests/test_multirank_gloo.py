"""The N > 1 path of parallel.py on CPU: world_size 2 over gloo.

Each rank computes the per-unit rows of its own (iteration, lattice) units
with the CPU oracle (standing in for the device kernels, which need a GPU),
exchanges them with parallel.exchange_rows and combines them through
parallel.row_map in lattice order; the result must equal the single-process
inversion of the same step (reference transform.py:99-127 semantics)."""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _step_data():
    from oracle import sfft_oracle as O
    from paper_1711_05152_b200 import workloads
    wl = workloads.config1(seed=9, n=3000, nnz=40)
    sch = O.build_with_retries(wl.cand, wl.b, np.random.SeedSequence(wl.lattice_seed))
    vals = [O.poly_eval(wl.oracle.freqs, wl.oracle.coeffs, O.lattice_nodes(z, m)) for m, z in zip(sch.ms, sch.zs)]
    return O, wl, sch, vals


def _unit_row(O, cand, sch, vals, l):
    """Dense row of unit l: X_l[res] * (1/M_l) where alias-free, else 0."""
    m, z, mk = sch.ms[l], sch.zs[l], sch.masks[l]
    spec = np.fft.fft(vals[l])
    row = np.zeros(len(cand), dtype=np.complex128)
    res = O.residues(cand[mk], z, m)
    row[mk] = spec[res] * (1.0 / m)
    return row


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_05152_b200.parallel import exchange_rows, owned_units, row_map
        O, wl, sch, vals = _step_data()
        L = len(sch.ms)
        n = len(wl.cand)
        per = -(-L // world)
        rows = torch.zeros((per, n, 2), dtype=torch.float64)
        for j, u in enumerate(owned_units(L, world, rank)):
            r = _unit_row(O, wl.cand, sch, vals, u)
            rows[j, :, 0] = torch.from_numpy(r.real.copy())
            rows[j, :, 1] = torch.from_numpy(r.imag.copy())
        allrows = exchange_rows(rows, world).numpy()
        rmap = row_map(L, world)
        sums = np.zeros(n, dtype=np.complex128)
        cnt = np.zeros(n, dtype=np.int64)
        for l in range(L):  # lattice order, as transform.py:118-124
            mk = sch.masks[l]
            t = allrows[rmap[l], :, 0] + 1j * allrows[rmap[l], :, 1]
            sums[mk] += t[mk]
            cnt[mk] += 1
        cov = cnt > 0
        q.put((rank, cov, sums[cov] / cnt[cov]))
    finally:
        dist.destroy_process_group()


def test_row_map_and_ownership():
    from paper_1711_05152_b200.parallel import owned_units, row_map
    for U in (1, 5, 13, 65):
        for W in (1, 2, 3, 8):
            per = -(-U // W)
            rm = row_map(U, W)
            seen = set()
            for g in range(W):
                for j, u in enumerate(owned_units(U, W, g)):
                    assert rm[u] == g * per + j
                    seen.add(u)
            assert seen == set(range(U))


@pytest.mark.timeout(300)
def test_two_rank_gloo_exchange_matches_single_process():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O, wl, sch, vals = _step_data()
    cov_ref, coef_ref = O.invert_multiple(wl.cand, sch, vals)
    for rank, cov, coef in got:
        assert np.array_equal(cov, cov_ref)
        assert np.array_equal(coef, coef_ref), rank  # same per-lattice terms, same order
