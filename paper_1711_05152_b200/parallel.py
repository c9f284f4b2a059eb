"""Sharding one MR1L step across the GPUs of a node.

Every rank replays the reference's RNG streams, so candidate sets, primes,
generating vectors and anchors are identical on all ranks without any
communication; the alias masks are recomputed on every rank (they are cheap
and integer-exact).  The (iteration, lattice) units of a step are dealt out
round-robin — unit u = i * L + l goes to rank u mod G — and each rank samples
and transforms its own units.  The merge is a sliced exchange (shard.cu):
candidates are cut into G slices; every rank packs its units' alias-free bins
per slice, one all-to-all (NCCL over NVLink; gloo via host staging in the
CPU tests) brings each rank the packs of its slice, which it combines in
lattice order with the single-GPU rounding sequence; the keep flags (and the
coefficients where needed) are all-gathered.  Results are bit-identical for
any GPU count.  Per rank and iteration the exchange moves about
0.61 * 16 B * |J| * L / G instead of the 16 B * |J| * L of dense rows.
"""

from __future__ import annotations

import math

import numpy as np

from .device import Device, dptr, hptr
from .mr1l import (RBMAX, UMAX, DeviceFreqs, DeviceScheme, StepPrep, StepResult, _sample_units, apply_cap_rows,
                   lattice_tables)
from .oracles import NoisyOracle
from . import _native

__all__ = ["Shard", "owned_units", "row_map", "exchange_rows", "run_step_sharded", "slice_geometry",
           "exchange_plan"]


class Shard:
    """Rank / world of a torch.distributed process group (1 / 0 when absent)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
        else:
            self.world, self.rank = 1, 0

    @property
    def active(self) -> bool:
        return self.world > 1


def owned_units(nunits: int, world: int, rank: int) -> list[int]:
    """Round-robin ownership of the step's units (u mod world == rank)."""
    return list(range(rank, nunits, world))


def row_map(nunits: int, world: int) -> np.ndarray:
    """Row of unit u in the all-gathered buffer [world][per][n]."""
    per = math.ceil(nunits / world)
    u = np.arange(nunits)
    return np.ascontiguousarray(((u % world) * per + u // world).astype(np.int32))


def exchange_rows(local, world: int, group=None):
    """All-gather equally shaped per-rank row blocks -> [world * per, ...]."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    # concatenated output layout [world * per, ...]: accepted by every backend's
    # all_gather_into_tensor (NCCL also takes a stacked one, gloo does not)
    out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    if hasattr(dist, "all_gather_into_tensor") and local.is_cuda:
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    else:
        parts = list(out.reshape((world,) + tuple(local.shape)).unbind(0))
        dist.all_gather(parts, local.contiguous(), group=group)
        out = torch.cat(parts)
    return out


def _align_noise(oracle, U: int, ms, L: int):
    """A rank without units in a chunk still consumes the chunk's noise
    stream / call counter, so every rank's copy stays aligned."""
    if isinstance(oracle, NoisyOracle):
        if oracle.device_rng:
            oracle.reserve_calls(U)
        else:
            for u in range(U):
                oracle.draw(int(ms[u % L]))


def _local_rows(dev, oracle, cand, sch, tabs, tails_chunk, d, step, i0, world, rank):
    """Dense rows [per, n] of this rank's units of one iteration chunk (the
    all-gather exchange of ``exchange="rows"``)."""
    torch = dev.torch
    n, t1, L, P = cand.n, cand.ncomp, sch.L, tabs.P
    rb = len(tails_chunk)
    U = rb * L
    mine = owned_units(U, world, rank)
    per = math.ceil(U / world)
    rows = dev.zeros((per, n, 2), torch.float64)
    nodes = 0
    if mine:
        buf = dev.empty((len(mine), P, 2), torch.float64)
        nodes = _sample_units(dev, oracle, tabs, t1, d, tails_chunk, buf, step, i0, units=mine)
        uarr = np.ascontiguousarray(np.asarray(mine, dtype=np.int32))
        dev.call("sfft_bluestein", hptr(tabs.ms), L, rb, tabs.P, dptr(tabs.ftab), dptr(tabs.bhat),
                 dptr(tabs.chirp), dptr(buf), hptr(uarr), len(mine), ctx=f"Bluestein FFT, step {step}")
        dev.call("sfft_gather_units", dptr(cand.data), n, t1, cand.kmax, hptr(tabs.ms), hptr(tabs.zs), L,
                 dptr(sch.masks), dptr(buf), P, rb, hptr(uarr), len(mine), dptr(rows),
                 ctx=f"unit gather, step {step}")
    else:
        _align_noise(oracle, U, tabs.ms, L)
    return rows, nodes


# ---------------------------------------------------------------------------
# sliced exchange (default)

TILE = 256


def slice_geometry(n: int, world: int) -> tuple[int, int, int]:
    """(tiles, tiles per slice, candidates per slice) of an n-candidate set
    cut into ``world`` slices of whole 256-candidate tiles."""
    ntiles = (n + TILE - 1) // TILE
    ts = max(1, (ntiles + world - 1) // world)
    return ntiles, ts, ts * TILE


def exchange_plan(sc: np.ndarray, L: int, U: int, world: int, rank: int):
    """Host bookkeeping of one chunk's all-to-all from the slice counts
    sc[q, l] (alias-free candidates of slice q on lattice l).

    Returns (own units, soff [world * nown] int64 send offsets (slice-major:
    slice q of own slot j), in_splits, out_splits (complex elements per
    destination / source rank), roff [U] int64: where unit u's entries of
    this rank's slice start in the receive buffer)."""
    sc = np.asarray(sc, dtype=np.int64).reshape(world, L)
    mine = owned_units(U, world, rank)
    seg = np.array([[sc[q, u % L] for u in mine] for q in range(world)], dtype=np.int64).reshape(world, len(mine))
    in_splits = seg.sum(axis=1)
    soff = (np.concatenate([[0], np.cumsum(in_splits)[:-1]])[:, None]
            + np.concatenate([np.zeros((world, 1), np.int64), np.cumsum(seg, axis=1)[:, :-1]], axis=1))
    roff = np.zeros(U, dtype=np.int64)
    out_splits = np.zeros(world, dtype=np.int64)
    base = 0
    for g in range(world):
        for u in owned_units(U, world, g):
            roff[u] = base + out_splits[g]
            out_splits[g] += sc[rank, u % L]
        base += out_splits[g]
    return mine, np.ascontiguousarray(soff.reshape(-1)), in_splits, out_splits, roff


def _a2a(dev, recv, send, out_splits, in_splits, group):
    """all_to_all_single of float64 buffers (splits in complex elements):
    NCCL on the device; other backends (gloo) through host staging."""
    import torch.distributed as dist
    ins = [int(x) * 2 for x in in_splits]
    outs = [int(x) * 2 for x in out_splits]
    sv, rv = send.reshape(-1)[: sum(ins)], recv.reshape(-1)[: sum(outs)]
    if dist.get_backend(group) == "nccl":
        dist.all_to_all_single(rv, sv, outs, ins, group=group)
        return
    if dev is not None:
        dev.sync()
    rh = rv.new_empty(rv.shape, device="cpu")
    dist.all_to_all_single(rh, sv.cpu(), outs, ins, group=group)
    rv.copy_(rh)


def _all_gather_flat(dev, out, local, group):
    """all_gather_into_tensor (concatenated layout); host-staged for gloo."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
        return
    import torch
    dev.sync()
    parts = list(out.new_empty(out.shape, device="cpu").chunk(dist.get_world_size(group)))
    dist.all_gather(parts, local.contiguous().cpu(), group=group)
    out.copy_(torch.cat(parts))


def _all_reduce_sum(dev, t, group):
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, group=group)
        return
    dev.sync()
    h = t.cpu()
    dist.all_reduce(h, group=group)
    t.copy_(h)


def run_step_sharded(dev: Device, oracle, cand: DeviceFreqs, sch: DeviceScheme, tails: list,
                     d: int, delta: float, cap: int, shard: Shard, step: int = 0,
                     simulate_world: int | None = None, prep: StepPrep | None = None,
                     need_coef: bool = True, exchange: str = "slices") -> StepResult:
    """run_step with the units of every iteration chunk spread over the ranks.

    ``exchange="slices"`` (default): packed alias-free bins, one all-to-all
    per chunk, each rank combines its candidate slice, the keep flags (and the
    coefficients when ``need_coef`` or a cap binds) are all-gathered.
    ``exchange="rows"``: the dense-row all-gather of round 1 (kept as the
    reference point of the tests).  ``prep``: the step preparation made
    beside the alias kernel (tables, sampling operands, buffers).
    ``simulate_world`` (single process, tests): run every simulated rank in
    turn and combine their buffers as the collectives would."""
    if exchange == "rows":
        return _run_step_rows(dev, oracle, cand, sch, tails, d, delta, cap, shard, step, simulate_world)
    torch = dev.torch
    n = cand.n
    L = sch.L
    r = len(tails)
    W = simulate_world or shard.world
    ranks = list(range(W)) if simulate_world else [shard.rank]
    if simulate_world and isinstance(oracle, NoisyOracle):
        raise ValueError("simulate_world needs a noiseless oracle (each simulated rank would draw the noise)")
    if prep is not None and (prep.r != r or prep.n != n or prep.l_max < L):
        prep = None
    tabs = None
    if prep is not None and prep.tabs is not None:
        tabs = prep.tabs.prefix(L)
        if tabs is not None:
            tabs.zs = sch.z_used
    if tabs is None:
        tabs = lattice_tables(dev, sch.m_used, sch.z_used, ctx=f"lattice tables, step {step}")
    keep = dev.empty((r, n), torch.uint8)
    coef = dev.empty((r, n, 2), torch.float64)
    counts = dev.zeros((r,), torch.int32)
    rb_max = max(1, min(RBMAX, UMAX // L))
    ntiles, ts, S = slice_geometry(n, W)
    # per step: tile popcounts of the masks, their scan, the slice totals
    tc = dev.empty((max(int(_native.query("sfft_mask_tiles_len", n, L)), 1),), torch.int32)
    toff = dev.empty(((ntiles + 1) * L,), torch.int32)
    scd = dev.empty((W * L,), torch.int32)
    dev.call("sfft_mask_tiles", dptr(sch.masks), n, L, dptr(tc), dptr(toff), ts, W, dptr(scd),
             ctx=f"mask tiles, step {step}")
    # read back while the units are sampled and transformed: only the packing
    # needs the slice counts (the all-to-all's split sizes)
    sc_wait = dev.download_async(scd)
    sc_cache = []

    def slice_counts():
        if not sc_cache:
            sc_cache.append(sc_wait().astype(np.int64).reshape(W, L))
        return sc_cache[0]
    nodes = 0
    slices = []  # per chunk: (i0, rb, coef_s [W, rb, S, 2] or None)
    t1 = cand.ncomp
    for i0 in range(0, r, rb_max):
        rb = min(rb_max, r - i0)
        U = rb * L
        chunk = tails[i0:i0 + rb]
        prepared = (prep is not None and prep.poly_ready and sch.attempts == 1 and i0 == 0 and rb == r)
        sends, plans = [], []
        for g in ranks:
            mine = owned_units(U, W, g)
            if mine:
                if prep is not None and prep.buf is not None and prep.buf.shape[1] == tabs.P \
                        and prep.buf.shape[0] >= len(mine):
                    buf = prep.buf[: len(mine)]
                else:
                    buf = dev.empty((len(mine), tabs.P, 2), torch.float64)
                nodes += _sample_units(dev, oracle, tabs, t1, d, chunk, buf, step, i0, units=mine,
                                       scratch=prep.poly if prep is not None else None, prepared=prepared,
                                       panels_ready=prepared and prep.panels_ready)
                uarr = np.ascontiguousarray(np.asarray(mine, dtype=np.int32))
                dev.call("sfft_bluestein", hptr(tabs.ms), L, rb, tabs.P, dptr(tabs.ftab), dptr(tabs.bhat),
                         dptr(tabs.chirp), dptr(buf), hptr(uarr), len(mine), ctx=f"Bluestein FFT, step {step}")
            _, soff, ins, outs, roff = exchange_plan(slice_counts(), L, U, W, g)
            plans.append((mine, ins, outs, roff))
            send = dev.empty((max(int(ins.sum()), 1), 2), torch.float64)
            if mine:
                d_soff = dev.upload(soff, asynchronous=True)
                dev.call("sfft_pack_units", dptr(cand.data), n, t1, cand.kmax, hptr(tabs.ms), hptr(tabs.zs), L,
                         dptr(sch.masks), dptr(buf), tabs.P, rb, hptr(uarr), len(mine), dptr(toff), ts,
                         dptr(d_soff), dptr(send), ctx=f"pack, step {step}")
            else:
                _align_noise(oracle, U, tabs.ms, L)
            sends.append(send)
        keep_s_all, coef_s_all, cnt_all = [], [], []
        for gi, g in enumerate(ranks):
            mine, ins, outs, roff = plans[gi]
            if simulate_world:
                # what rank g receives: from every rank h, h's pack for slice g
                parts = []
                for h in range(W):
                    _, ins_h, _, _ = plans[h]
                    off = int(ins_h[:g].sum())
                    parts.append(sends[h][off: off + int(ins_h[g])])
                recv = torch.cat(parts) if parts else dev.empty((1, 2), torch.float64)
            else:
                recv = dev.empty((max(int(outs.sum()), 1), 2), torch.float64)
                with torch.cuda.stream(dev.stream):
                    _a2a(dev, recv, sends[gi], outs, ins, shard.group)
            d_roff = dev.upload(np.ascontiguousarray(roff), asynchronous=True)
            keep_s = dev.empty((rb, S), torch.uint8)
            coef_s = dev.empty((rb, S, 2), torch.float64)
            cnt = dev.empty((rb,), torch.int32)
            dev.call("sfft_combine_slice", n, L, dptr(sch.masks), dptr(toff), ts, g, dptr(recv), dptr(d_roff), rb,
                     float(delta), dptr(coef_s), dptr(keep_s), dptr(cnt), ctx=f"combine slice, step {step}")
            keep_s_all.append(keep_s)
            coef_s_all.append(coef_s)
            cnt_all.append(cnt)
        # keep flags of all slices, survivor counts
        with torch.cuda.stream(dev.stream):
            if simulate_world:
                kg = torch.cat([k.reshape(-1) for k in keep_s_all])
                ctot = torch.stack(cnt_all).sum(0).to(torch.int32)
            else:
                kg = torch.empty((W * rb * S,), dtype=torch.uint8, device=dev.device)
                _all_gather_flat(dev, kg, keep_s_all[0].reshape(-1), shard.group)
                ctot = cnt_all[0]
                _all_reduce_sum(dev, ctot, shard.group)
            counts[i0:i0 + rb].copy_(ctot)
        dev.call("sfft_unshard_rows", dptr(kg), 1, W, rb, S, n, i0, dptr(keep), ctx=f"unshard, step {step}")
        slices.append((i0, rb, coef_s_all))
    lazy = cap >= n and need_coef  # no cap can bind and every coefficient is gathered: no read-back here
    counts_h = None if lazy else dev.download_small(counts).astype(np.int64)
    over = np.zeros(r, dtype=bool) if lazy else counts_h > cap
    for i0, rb, coef_s_all in slices:
        if need_coef or over[i0:i0 + rb].any():
            with torch.cuda.stream(dev.stream):
                if simulate_world:
                    cg = torch.cat([c.reshape(-1) for c in coef_s_all])
                else:
                    cg = torch.empty((W * rb * S * 2,), dtype=torch.float64, device=dev.device)
                    _all_gather_flat(dev, cg, coef_s_all[0].reshape(-1), shard.group)
            dev.call("sfft_unshard_rows", dptr(cg), 16, W, rb, S, n, i0, dptr(coef), ctx=f"unshard, step {step}")
    if lazy:
        return StepResult(keep, coef, None, nodes, _lazy=lambda: dev.download_small(counts).astype(np.int64))
    counts_h = apply_cap_rows(dev, coef, keep, n, counts_h, cap, step)
    return StepResult(keep, coef, counts_h, nodes)


def _run_step_rows(dev: Device, oracle, cand: DeviceFreqs, sch: DeviceScheme, tails: list,
                   d: int, delta: float, cap: int, shard: Shard, step: int = 0,
                   simulate_world: int | None = None) -> StepResult:
    """Dense per-unit rows, one all-gather per chunk (round 1's exchange)."""
    torch = dev.torch
    n = cand.n
    L = sch.L
    tabs = lattice_tables(dev, sch.m_used, sch.z_used, ctx=f"lattice tables, step {step}")
    r = len(tails)
    keep = dev.empty((r, n), torch.uint8)
    coef = dev.empty((r, n, 2), torch.float64)
    counts = dev.zeros((r,), torch.int32)
    rb_max = max(1, min(RBMAX, UMAX // L))
    W = simulate_world or shard.world
    nodes = 0
    for i0 in range(0, r, rb_max):
        rb = min(rb_max, r - i0)
        U = rb * L
        chunk = tails[i0:i0 + rb]
        if simulate_world:
            blocks = []
            for g in range(W):
                rows, k = _local_rows(dev, oracle, cand, sch, tabs, chunk, d, step, i0, W, g)
                blocks.append(rows)
                nodes += k
            allrows = torch.cat(blocks, 0)
        else:
            rows, nodes_k = _local_rows(dev, oracle, cand, sch, tabs, chunk, d, step, i0, W, shard.rank)
            nodes += nodes_k
            with torch.cuda.stream(dev.stream):
                allrows = exchange_rows(rows, W, shard.group)
        rmap = row_map(U, W)
        dev.call("sfft_combine_units", n, L, dptr(sch.masks), dptr(allrows), hptr(rmap), rb, rb, 0,
                 float(delta), dptr(coef[i0]), dptr(keep[i0]), dptr(counts[i0:]),
                 ctx=f"combine, step {step}")
    counts_h = apply_cap_rows(dev, coef, keep, n, dev.download_small(counts), cap, step)
    return StepResult(keep, coef, counts_h, nodes)
