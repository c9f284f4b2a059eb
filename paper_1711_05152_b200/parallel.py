"""Sharding one MR1L step across the GPUs of a node.

Every rank replays the reference's RNG streams, so candidate sets, primes,
generating vectors and anchors are identical on all ranks without any
communication; the alias masks are recomputed on every rank (they are cheap
and integer-exact).  The (iteration, lattice) units of a step are dealt out
round-robin — unit u = i * L + l goes to rank u mod G — and each rank samples,
transforms and gathers the alias-free bins of its own units into dense rows.
One all-gather (NCCL over NVLink on GPUs, gloo on CPU in the tests) gives
every rank all rows, which are combined in lattice order with the single-GPU
rounding sequence: results are bit-identical for any GPU count.
"""

from __future__ import annotations

import math

import numpy as np

from .device import Device, dptr, hptr
from .mr1l import (RBMAX, UMAX, DeviceFreqs, DeviceScheme, StepResult, _sample_units, apply_cap_rows,
                   lattice_tables)
from .oracles import NoisyOracle
from . import _native

__all__ = ["Shard", "owned_units", "row_map", "exchange_rows", "run_step_sharded"]


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


def _local_rows(dev, oracle, cand, sch, tabs, tails_chunk, d, step, i0, world, rank):
    """Rows [per, n] of this rank's units of one iteration chunk."""
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
    elif isinstance(oracle, NoisyOracle):
        # keep this rank's copy of the noise stream / call counter aligned
        if oracle.device_rng:
            oracle.reserve_calls(U)
        else:
            for u in range(U):
                oracle.draw(int(tabs.ms[u % L]))
    return rows, nodes


def run_step_sharded(dev: Device, oracle, cand: DeviceFreqs, sch: DeviceScheme, tails: list,
                     d: int, delta: float, cap: int, shard: Shard, step: int = 0,
                     simulate_world: int | None = None) -> StepResult:
    """run_step with the units of every iteration chunk spread over the ranks.

    ``simulate_world`` (single process, tests): compute the rows of every
    simulated rank in turn and concatenate them as the all-gather would."""
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
