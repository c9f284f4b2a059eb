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


# ---------------------------------------------------------------------------
# sliced exchange (parallel.exchange_plan + all_to_all_single), the host side
# of sfft_pack_units / sfft_combine_slice emulated in numpy

def _slice_bounds(n, W):
    from paper_1711_05152_b200.parallel import slice_geometry
    ntiles, ts, S = slice_geometry(n, W)
    return [(min(n, q * S), min(n, (q + 1) * S)) for q in range(W)]


def _slice_counts(masks, n, W):
    b = _slice_bounds(n, W)
    return np.array([[int(mk[a:e].sum()) for mk in masks] for a, e in b], dtype=np.int64)


def _pack(O, cand, sch, vals, W, g, soff, mine):
    """sfft_pack_units in numpy: slot j's entries of slice q at soff[q * nown + j]."""
    L = len(sch.ms)
    total = int(_slice_counts(sch.masks, len(cand), W)[:, [u % L for u in mine]].sum()) if mine else 0
    send = np.zeros(max(total, 1), dtype=np.complex128)
    for q, (a, e) in enumerate(_slice_bounds(len(cand), W)):
        for j, u in enumerate(mine):
            l = u % L
            row = _unit_row(O, cand, sch, vals, l)
            sel = np.nonzero(sch.masks[l][a:e])[0] + a
            p0 = int(soff[q * len(mine) + j])
            send[p0:p0 + len(sel)] = row[sel]
    return send


def _combine(sch, n, W, q, recv, roff):
    """sfft_combine_slice in numpy (lattice order)."""
    L = len(sch.ms)
    a, e = _slice_bounds(n, W)[q]
    sums = np.zeros(e - a, dtype=np.complex128)
    cnt = np.zeros(e - a, dtype=np.int64)
    for l in range(L):
        mk = sch.masks[l][a:e]
        idx = np.nonzero(mk)[0]
        sums[idx] += recv[int(roff[l]): int(roff[l]) + len(idx)]
        cnt[idx] += 1
    return sums, cnt


@pytest.mark.parametrize("W", [2, 3, 8])
def test_exchange_plan_all_ranks_simulated(W):
    from paper_1711_05152_b200.parallel import exchange_plan
    O, wl, sch, vals = _step_data()
    L, n = len(sch.ms), len(wl.cand)
    sc = _slice_counts(sch.masks, n, W)
    plans = [exchange_plan(sc, L, L, W, g) for g in range(W)]
    sends = [_pack(O, wl.cand, sch, vals, W, g, p[1], p[0]) for g, p in enumerate(plans)]
    cov_ref, coef_ref = O.invert_multiple(wl.cand, sch, vals)
    sums_all, cnt_all = [], []
    for q in range(W):
        parts = []
        for h in range(W):
            ins = plans[h][2]
            off = int(ins[:q].sum())
            parts.append(sends[h][off:off + int(ins[q])])
        recv = np.concatenate(parts)
        assert len(recv) == int(plans[q][3].sum())
        s_, c_ = _combine(sch, n, W, q, recv, plans[q][4])
        sums_all.append(s_)
        cnt_all.append(c_)
    sums, cnt = np.concatenate(sums_all), np.concatenate(cnt_all)
    assert np.array_equal(cnt > 0, cov_ref)
    assert np.array_equal(sums[cov_ref] / cnt[cov_ref], coef_ref)


def _worker_slices(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_05152_b200.parallel import _a2a, exchange_plan
        O, wl, sch, vals = _step_data()
        L, n = len(sch.ms), len(wl.cand)
        sc = _slice_counts(sch.masks, n, world)
        mine, soff, ins, outs, roff = exchange_plan(sc, L, L, world, rank)
        send = _pack(O, wl.cand, sch, vals, world, rank, soff, mine)
        st = torch.from_numpy(np.stack([send.real, send.imag], axis=1).copy())
        rt = torch.empty((max(int(outs.sum()), 1), 2), dtype=torch.float64)
        _a2a(None, rt, st, outs, ins, None)
        recv = rt.numpy()[:, 0] + 1j * rt.numpy()[:, 1]
        sums, cnt = _combine(sch, n, world, rank, recv, roff)
        q.put((rank, sums, cnt))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_sliced_exchange_matches_single_process():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_slices, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([q.get(timeout=240) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O, wl, sch, vals = _step_data()
    cov_ref, coef_ref = O.invert_multiple(wl.cand, sch, vals)
    sums = np.concatenate([g[1] for g in got])
    cnt = np.concatenate([g[2] for g in got])
    assert np.array_equal(cnt > 0, cov_ref)
    assert np.array_equal(sums[cov_ref] / cnt[cov_ref], coef_ref)  # bit-identical: same terms, same order
