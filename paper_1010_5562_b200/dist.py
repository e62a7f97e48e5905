"""Multi-GPU partitioning of the FCFS hot path (BASELINE.json north_star (6)).

One process per GPU (torchrun), torch.distributed for the plumbing (NCCL over NVLink on B200).
By linearity (Prop. 2) and separability (Lemma 1):

* clips   — independent problems; each rank runs its own clip range (no collective).
* rows    — one clip, disjoint signed frequency-row ranges m in [m_lo, m_hi] (fcfs_shard ROWS);
            ranks all_gather their rows into the full window.
* vblock  — one clip, contiguous blocks of the canonical corner list (fcfs_shard VERTEX_BLOCK);
            every rank computes the whole window from its block, the partial windows are summed
            with a reduce_scatter (each rank keeps 1/P of the rows) and optionally all_gathered.

The compute step is injectable (``compute=``) so the partition / collective logic is testable on CPU
with the gloo backend; the default is the CUDA library (``fcfs.coeffs`` with an ``fcfs_shard``).
This module holds no FCFS arithmetic.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def clip_range(B: int, rank: int, world: int):
    """Contiguous, balanced clip range [b0, b1) of `rank`."""
    b0 = B * rank // world
    b1 = B * (rank + 1) // world
    return b0, b1


def row_range(M: int, rank: int, world: int):
    """Balanced contiguous signed row range [m_lo, m_hi] of [-M, M] for `rank` (may be empty: m_lo > m_hi)."""
    rows = 2 * M + 1
    r0 = rows * rank // world
    r1 = rows * (rank + 1) // world
    return -M + r0, -M + r1 - 1


def vertex_range(K: int, rank: int, world: int):
    k0 = K * rank // world
    k1 = K * (rank + 1) // world
    return k0, k1


def _cuda_rows(x, y, w, area, T, M, N, prec, m_lo, m_hi):
    from . import fcfs
    sh = fcfs.Shard(fcfs.SHARD_ROWS, m_lo, m_hi, 0, 0)
    return fcfs.coeffs(x, y, w, area, T, M, N, prec=prec, shard=sh)


def _cuda_vblock(x, y, w, T, M, N, prec, k0, k1):
    from . import fcfs
    sh = fcfs.Shard(fcfs.SHARD_VERTEX_BLOCK, 0, 0, k0, k1)
    return fcfs.coeffs(x, y, w, 0, T, M, N, prec=prec, shard=sh)


def _real(t):
    return torch.view_as_real(t) if t.is_complex() else t


def _reduce_scatter(out, inp, group):
    """sum-reduce `inp` ([world * n] elements) and keep this rank's n-slice in `out`."""
    try:
        dist.reduce_scatter_tensor(_real(out), _real(inp), op=dist.ReduceOp.SUM, group=group)
    except (RuntimeError, NotImplementedError, ValueError):
        # backends without reduce_scatter (gloo on CPU): all_reduce, then slice
        buf = inp.clone()
        dist.all_reduce(_real(buf), op=dist.ReduceOp.SUM, group=group)
        r = dist.get_rank(group)
        out.copy_(buf[r * out.numel():(r + 1) * out.numel()])


def coeffs_rows_sharded(x, y, w, area, T, M, N, prec="fp64", group=None, compute=None):
    """Full dense window of one clip, rows sharded over the ranks of `group`, all_gathered."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    compute = compute or _cuda_rows
    width = 2 * N + 1
    per = -(-(2 * M + 1) // world)                 # padded rows per rank
    m_lo, m_hi = row_range(M, rank, world)
    local = None
    if m_hi >= m_lo:
        local = compute(x, y, w, area, T, M, N, prec, m_lo, m_hi).reshape(-1, width)
    dtype = local.dtype if local is not None else (torch.complex128 if prec == "fp64" else torch.complex64)
    dev = x.device
    pad = torch.zeros(per, width, dtype=dtype, device=dev)
    if local is not None:
        pad[:local.shape[0]] = local
    gathered = torch.empty(world * per, width, dtype=dtype, device=dev)
    dist.all_gather_into_tensor(_real(gathered), _real(pad), group=group)
    parts = []
    for r in range(world):
        a, b = row_range(M, r, world)
        if b >= a:
            parts.append(gathered[r * per:r * per + (b - a + 1)])
    return torch.cat(parts).reshape(-1)


def coeffs_vertex_sharded(x, y, w, T, M, N, prec="fp64", group=None, compute=None, gather=True):
    """Window of one clip from corner blocks: partial windows summed by reduce_scatter.

    Returns the full window (gather=True) or this rank's contiguous 1/P slice of it.
    The DC of each block is its own exact sum w x y / T^2, so the sum is the unsharded DC.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    compute = compute or _cuda_vblock
    K = x.shape[0]
    k0, k1 = vertex_range(K, rank, world)
    part = compute(x, y, w, T, M, N, prec, k0, k1).reshape(-1)
    n = part.numel()
    per = -(-n // world)
    buf = torch.zeros(world * per, dtype=part.dtype, device=part.device)
    buf[:n] = part
    mine = torch.empty(per, dtype=part.dtype, device=part.device)
    _reduce_scatter(mine, buf, group)
    if not gather:
        return mine
    full = torch.empty(world * per, dtype=part.dtype, device=part.device)
    dist.all_gather_into_tensor(_real(full), _real(mine), group=group)
    return full[:n]
