"""Multi-GPU partitioning of the FCFS hot path (BASELINE.json north_star (6)).

One process per GPU (torchrun), torch.distributed for the plumbing (NCCL over NVLink on B200).
By linearity (Prop. 2) and separability (Lemma 1):

* clips   — independent problems; each rank runs its own clip range (no collective).
* bands   — a1 of one clip sharded by lattice rows: rank r extracts only the canonical corners with
            y in its band [y_r, y_{r+1}) (fcfs_vertices_from_rects_band); the bands, all_gathered in
            rank order, ARE the canonical (y, x)-sorted list, and the band areas sum to the clip's.
* rows    — one clip, disjoint signed frequency-row ranges m in [m_lo, m_hi] (fcfs_shard ROWS);
            ranks all_gather their rows into the full window.
* peers   — the rows shard with its all_gather fused into the epilogue: every rank's kernel stores its
            rows straight into every rank's full-window buffer (fcfs_coeffs_rows_to_peers; peer buffers
            mapped by CUDA IPC over NVLink), then one collective orders the ranks before the window is read.
* vblock  — one clip, contiguous blocks of the canonical corner list (fcfs_shard VERTEX_BLOCK, on the
            row-bucket GEMM route: the lattice-FFT route would repeat its per-row FFTs on every rank);
            every rank computes the whole window from its block, the partial windows are summed with a
            reduce_scatter (each rank keeps 1/P of the rows) and optionally all_gathered.

Compute steps are injectable (``compute=`` / ``extract=``) so the partition / collective logic is
testable on CPU with the gloo backend; the defaults are the CUDA library with one pre-allocated plan
per rank (workspaces are sized once, not per call).  This module holds no FCFS arithmetic.
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


def band_range(T: int, rank: int, world: int):
    """Lattice-row band [y_lo, y_hi) of `rank`: the T + 1 rows y = 0..T in equal contiguous parts."""
    rows = T + 1
    return rows * rank // world, rows * (rank + 1) // world


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


# ------------------------------------------------------------------------------------------------
# a1: y-band sharded extraction + all_gather of the corner lists
# ------------------------------------------------------------------------------------------------

def gather_corners(x, y, w, K: int, area, group=None):
    """All ranks' band corner lists concatenated in rank order, and the summed area.

    x, y, w: int32 tensors holding this rank's K corners (y-sorted, rows of its band); area: int64
    tensor [1] (the band's share).  Returns (x, y, w, K_total, area_total) on every rank, with
    area_total a host int (one small host read of the per-rank counts sizes the gather)."""
    world = dist.get_world_size(group)
    dev = x.device
    meta = torch.stack([torch.tensor(K, dtype=torch.int64, device=dev), area.reshape(-1)[0].to(torch.int64)])
    metas = torch.empty(world * 2, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(metas, meta, group=group)
    m = metas.view(world, 2).cpu()
    Ks = [int(v) for v in m[:, 0]]
    area_t = int(m[:, 1].sum())
    kmax = max(max(Ks), 1)
    pack = torch.zeros(3, kmax, dtype=torch.int32, device=dev)
    pack[0, :K] = x[:K]
    pack[1, :K] = y[:K]
    pack[2, :K] = w[:K]
    allp = torch.empty(world * 3 * kmax, dtype=torch.int32, device=dev)
    dist.all_gather_into_tensor(allp, pack.reshape(-1), group=group)
    allp = allp.view(world, 3, kmax)
    out = [torch.cat([allp[r, i, :Ks[r]] for r in range(world)]) for i in range(3)]   # three allocations
    return out[0], out[1], out[2], sum(Ks), area_t


class BandExtract:
    """This rank's band of one clip's canonical corners (fcfs_vertices_from_rects_band), one plan."""

    def __init__(self, R, T, rank, world, G=None, max_group=1, grouped=False, device="cuda", extract=None):
        self.T = int(T)
        self.band = band_range(T, rank, world)
        self.extract = extract
        if extract is None:
            from . import fcfs
            self.plan = fcfs.VerticesPlan(R, T, G, 1, max_group, grouped, device=device)

    def run(self, rects, group_ptr=None):
        """(x, y, w, K, area[1]) of this rank's band."""
        if self.extract is not None:
            return self.extract(rects, group_ptr, self.T, *self.band)
        p = self.plan
        K = p.run_band(rects, self.band[0], self.band[1], group_ptr)
        return p.x, p.y, p.w, K, p.area


def extract_band_sharded(rects, T, group_ptr=None, group=None, extractor=None, **kw):
    """a1 of one clip over the ranks of `group`: each rank extracts its band, all_gather assembles the
    canonical list.  Returns (x, y, w, K, area)."""
    if extractor is None:
        extractor = BandExtract(rects.shape[0], T, dist.get_rank(group), dist.get_world_size(group), **kw)
    x, y, w, K, area = extractor.run(rects, group_ptr)
    return gather_corners(x, y, w, K, area, group)


# ------------------------------------------------------------------------------------------------
# a2-a5: rows and vertex-block shards with one plan per rank
# ------------------------------------------------------------------------------------------------

class RowsSharded:
    """Full dense window of one clip, this rank's signed rows (fcfs_shard ROWS), all_gathered.
    One CoeffsPlan per corner count (the workload's K is fixed across steps: built once)."""

    def __init__(self, T, M, N, prec, rank, world, device="cuda", route=None, compute=None):
        self.T, self.M, self.N, self.prec, self.route = int(T), int(M), int(N), prec, route
        self.world, self.compute, self.device = world, compute, device
        self.m_lo, self.m_hi = row_range(M, rank, world)
        self.width = 2 * N + 1
        self.per = -(-(2 * M + 1) // world)            # padded rows per rank
        self.plans = {}
        self.dtype = torch.complex128 if prec == "fp64" else torch.complex64
        self.pad = torch.zeros(self.per, self.width, dtype=self.dtype, device=device)
        self.gathered = torch.empty(world * self.per, self.width, dtype=self.dtype, device=device)

    def _local(self, x, y, w, K, area):
        if self.m_hi < self.m_lo:
            return None
        if self.compute is not None:
            return self.compute(x[:K], y[:K], w[:K], area, self.T, self.M, self.N, self.prec, self.m_lo, self.m_hi)
        plan = self.plans.get(K)
        if plan is None:
            from . import fcfs
            sh = fcfs.Shard(fcfs.SHARD_ROWS, self.m_lo, self.m_hi, 0, 0)
            plan = fcfs.CoeffsPlan(K, self.T, self.M, self.N, prec=self.prec, shard=sh, device=self.device,
                                   route=self.route)
            self.plans = {K: plan}
        return plan.run(x[:K], y[:K], w[:K], area)

    def run(self, x, y, w, K, area, group=None):
        local = self._local(x, y, w, K, area)
        if local is not None:
            local = local.reshape(-1, self.width)
            self.pad[:local.shape[0]] = local
        dist.all_gather_into_tensor(_real(self.gathered), _real(self.pad), group=group)
        parts = []
        for r in range(self.world):
            a, b = row_range(self.M, r, self.world)
            if b >= a:
                parts.append(self.gathered[r * self.per:r * self.per + (b - a + 1)])
        return torch.cat(parts).reshape(-1)


def peer_buffers(full, group=None):
    """Device pointers of every rank's `full` buffer in this process (rank order): this rank's own pointer
    and the other ranks' buffers opened from their CUDA IPC handles (torch's storage sharing; same node,
    P2P over NVLink).  Returns (pointers, keep-alive storages)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        return [full.data_ptr()], []
    handle = full.untyped_storage()._share_cuda_()
    handles = [None] * world
    dist.all_gather_object(handles, handle, group=group)
    ptrs, keep = [], []
    for r in range(world):
        if r == rank:
            ptrs.append(full.data_ptr())
            continue
        st = torch.UntypedStorage._new_shared_cuda(*handles[r])
        keep.append(st)
        ptrs.append(st.data_ptr())
    return ptrs, keep


class RowsPeers:
    """Full dense window of one clip with the rows' all_gather fused into the epilogue: this rank computes
    its signed rows (fcfs_shard ROWS) and its epilogue stores every output at its full-window position into
    every rank's buffer (fcfs_coeffs_rows_to_peers over NVLink), then one small all_reduce orders the ranks
    (each rank's stores precede its collective; the collective completes after all ranks joined).  No
    all_gather of the rows, no per-rank slice buffers.  ``run_local`` (tests) replaces the CUDA call."""

    def __init__(self, T, M, N, prec, rank, world, device="cuda", route=None, group=None, run_local=None):
        self.T, self.M, self.N, self.prec, self.route = int(T), int(M), int(N), prec, route
        self.world, self.device, self.run_local = world, device, run_local
        self.m_lo, self.m_hi = row_range(M, rank, world)
        self.dtype = torch.complex128 if prec == "fp64" else torch.complex64
        self.full = torch.zeros((2 * M + 1) * (2 * N + 1), dtype=self.dtype, device=device)
        self.ptrs, self._keep = peer_buffers(self.full, group) if run_local is None else ([], [])
        self.flag = torch.zeros(1, dtype=torch.float32, device=device)
        self.plans = {}

    def run(self, x, y, w, K, area, group=None):
        if self.m_hi >= self.m_lo:
            if self.run_local is not None:
                self.run_local(self, x[:K], y[:K], w[:K], area)
            else:
                plan = self.plans.get(K)
                if plan is None:
                    from . import fcfs
                    sh = fcfs.Shard(fcfs.SHARD_ROWS, self.m_lo, self.m_hi, 0, 0)
                    plan = fcfs.CoeffsPlan(K, self.T, self.M, self.N, prec=self.prec, shard=sh, device=self.device,
                                           route=self.route)
                    self.plans = {K: plan}
                plan.run_to_peers(x[:K], y[:K], w[:K], area, self.ptrs)
        if dist.get_backend(group) == "nccl":
            dist.all_reduce(self.flag, group=group)   # stream-ordered: every rank's peer stores precede it
        else:                                         # gloo (tests): host barrier after the device work
            torch.cuda.synchronize()
            dist.barrier(group=group)
        return self.full


class VertexSharded:
    """Window of one clip from corner blocks (fcfs_shard VERTEX_BLOCK on the GEMM route): partial
    windows summed by reduce_scatter; returns the full window (gather=True) or this rank's slice.
    The DC of each block is its own exact sum w x y / T^2, so the sum is the unsharded DC."""

    def __init__(self, T, M, N, prec, rank, world, device="cuda", compute=None):
        self.T, self.M, self.N, self.prec = int(T), int(M), int(N), prec
        self.rank, self.world, self.compute, self.device = rank, world, compute, device
        self.plans = {}

    def _part(self, x, y, w, K):
        k0, k1 = vertex_range(K, self.rank, self.world)
        if self.compute is not None:
            return self.compute(x, y, w, self.T, self.M, self.N, self.prec, k0, k1)
        plan = self.plans.get(K)
        if plan is None:
            from . import fcfs
            sh = fcfs.Shard(fcfs.SHARD_VERTEX_BLOCK, 0, 0, k0, k1)
            plan = fcfs.CoeffsPlan(K, self.T, self.M, self.N, prec=self.prec, shard=sh, device=self.device,
                                   route="gemm")
            self.plans = {K: plan}
        return plan.run(x[:K], y[:K], w[:K], 0)

    def run(self, x, y, w, K, group=None, gather=True):
        part = self._part(x, y, w, K).reshape(-1)
        n = part.numel()
        per = -(-n // self.world)
        buf = torch.zeros(self.world * per, dtype=part.dtype, device=part.device)
        buf[:n] = part
        mine = torch.empty(per, dtype=part.dtype, device=part.device)
        _reduce_scatter(mine, buf, group)
        if not gather:
            return mine
        full = torch.empty(self.world * per, dtype=part.dtype, device=part.device)
        dist.all_gather_into_tensor(_real(full), _real(mine), group=group)
        return full[:n]


def coeffs_rows_sharded(x, y, w, area, T, M, N, prec="fp64", group=None, compute=None):
    """Full dense window of one clip, rows sharded over the ranks of `group`, all_gathered (one-shot)."""
    rs = RowsSharded(T, M, N, prec, dist.get_rank(group), dist.get_world_size(group), device=x.device,
                     compute=compute)
    return rs.run(x, y, w, x.shape[0], area, group)


def coeffs_vertex_sharded(x, y, w, T, M, N, prec="fp64", group=None, compute=None, gather=True):
    """Window of one clip from corner blocks (one-shot VertexSharded)."""
    vs = VertexSharded(T, M, N, prec, dist.get_rank(group), dist.get_world_size(group), device=x.device,
                       compute=compute)
    return vs.run(x, y, w, x.shape[0], group, gather)
