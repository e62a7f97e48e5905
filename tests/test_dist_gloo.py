"""World-size-2 gloo tests (CPU) of the multi-GPU partition / collective logic (dist.py).

The compute step is injected: on CPU it is the oracle restricted to the shard (rows or a corner
block), so the test checks that partitioning + all_gather / reduce_scatter reassemble exactly the
unsharded window; the CUDA compute of each shard is covered by the single-GPU shard parity tests."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1010_5562_b200 import dist as fdist
from paper_1010_5562_b200 import inputs


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_rows(x, y, w, area, T, M, N, prec, m_lo, m_hi):
    ms, ns = oracle.window(M, N)
    sel = (ms >= m_lo) & (ms <= m_hi)
    F, _ = oracle.coeffs(x.numpy(), y.numpy(), w.numpy(), int(area), T, ms[sel], ns[sel])
    return torch.from_numpy(F)


def _oracle_vblock(x, y, w, T, M, N, prec, k0, k1):
    ms, ns = oracle.window(M, N)
    xs, ys, ws = x.numpy()[k0:k1], y.numpy()[k0:k1], w.numpy()[k0:k1]
    area = int((ws.astype(np.int64) * xs * ys).sum())
    F, _ = oracle.coeffs(xs, ys, ws, area, T, ms, ns)
    return torch.from_numpy(F)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = inputs.c2(seed=5, n_poly=120, T=1024)
        e = oracle.extract(wl.rects, wl.T, wl.group_ptr)
        x, y, w = (torch.from_numpy(e[k]) for k in ("x", "y", "w"))
        M = N = 9
        rows = fdist.coeffs_rows_sharded(x, y, w, int(e["area"][0]), wl.T, M, N, compute=_oracle_rows)
        vb = fdist.coeffs_vertex_sharded(x, y, w, wl.T, M, N, compute=_oracle_vblock)
        mine = fdist.coeffs_vertex_sharded(x, y, w, wl.T, M, N, compute=_oracle_vblock, gather=False)
        q.put((rank, rows.numpy(), vb.numpy(), mine.numpy()))
    finally:
        dist.destroy_process_group()


def _oracle_band(rects, group_ptr, T, y_lo, y_hi):
    """This rank's band on CPU: the oracle's canonical list restricted to rows y_lo <= y < y_hi (what
    fcfs_vertices_from_rects_band returns on the GPU; that kernel is checked against this rule in
    test_gpu_parity.py)."""
    e = oracle.extract(rects.numpy(), T, None if group_ptr is None else group_ptr.numpy())
    sel = (e["y"] >= y_lo) & (e["y"] < y_hi)
    x, y, w = (torch.from_numpy(np.ascontiguousarray(e[k][sel])) for k in ("x", "y", "w"))
    area = torch.tensor([int((e["w"][sel].astype(np.int64) * e["x"][sel] * e["y"][sel]).sum())], dtype=torch.int64)
    return x, y, w, int(sel.sum()), area


def _worker_bands(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = inputs.c4(seed=3, n_poly=3000, T=4096, M=8)
        rects = torch.from_numpy(wl.rects)
        ex = fdist.BandExtract(rects.shape[0], wl.T, rank, world, extract=_oracle_band)
        x, y, w, K, area = fdist.extract_band_sharded(rects, wl.T, extractor=ex)
        M = N = 6
        rs = fdist.RowsSharded(wl.T, M, N, "fp64", rank, world, device="cpu", compute=_oracle_rows)
        rows = rs.run(x, y, w, K, area)
        rows2 = rs.run(x, y, w, K, area)          # the plan / buffers are reused across steps
        vs = fdist.VertexSharded(wl.T, M, N, "fp64", rank, world, device="cpu", compute=_oracle_vblock)
        vb = vs.run(x, y, w, K)
        q.put((rank, x.numpy(), y.numpy(), w.numpy(), K, area, rows.numpy(), rows2.numpy(), vb.numpy()))
    finally:
        dist.destroy_process_group()


def _spawn(target, world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=target, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda t: t[0])


@pytest.mark.parametrize("world", [2, 4])
def test_band_sharded_extraction_gathers_the_canonical_list(world):
    """y-band shards of a1 + all_gather == the single-process canonical list, bit for bit; the band
    areas sum to the clip's; rows / vertex-block shards of the gathered list reassemble the window."""
    res = _spawn(_worker_bands, world)
    wl = inputs.c4(seed=3, n_poly=3000, T=4096, M=8)
    e = oracle.extract(wl.rects, wl.T)
    ms, ns = oracle.window(6, 6)
    Fr, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], wl.T, ms, ns)
    for rank, x, y, w, K, area, rows, rows2, vb in res:
        assert K == e["K"] and area == int(e["area"][0])
        assert np.array_equal(x, e["x"]) and np.array_equal(y, e["y"]) and np.array_equal(w, e["w"])
        assert np.array_equal(rows, Fr) and np.array_equal(rows2, Fr)
        assert np.all(np.abs(vb - Fr) <= 1e-12 * B + (B == 0) * 1e-15)
    # the bands tile the lattice rows 0..T exactly
    for P in (1, 2, 3, 4, 8):
        b = [fdist.band_range(wl.T, r, P) for r in range(P)]
        assert b[0][0] == 0 and b[-1][1] == wl.T + 1 and all(b[i][1] == b[i + 1][0] for i in range(P - 1))


def test_partition_helpers_cover_exactly():
    for world in (1, 2, 3, 4, 8):
        B = 4096
        assert sum(np.diff(fdist.clip_range(B, r, world))[0] for r in range(world)) == B
        M = 27
        rows = []
        for r in range(world):
            a, b = fdist.row_range(M, r, world)
            rows += list(range(a, b + 1))
        assert rows == list(range(-M, M + 1))
        K = 1001
        ks = [fdist.vertex_range(K, r, world) for r in range(world)]
        assert ks[0][0] == 0 and ks[-1][1] == K and all(ks[i][1] == ks[i + 1][0] for i in range(world - 1))


def test_world2_rows_and_vertex_blocks_reassemble_the_window():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    wl = inputs.c2(seed=5, n_poly=120, T=1024)
    e = oracle.extract(wl.rects, wl.T, wl.group_ptr)
    ms, ns = oracle.window(9, 9)
    Fr, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], wl.T, ms, ns)
    for rank, rows, vb, mine in res:
        assert np.array_equal(rows, Fr)                       # rows: a pure permutation, exact
        assert np.all(np.abs(vb - Fr) <= 1e-12 * B + (B == 0) * 1e-15)
        n = len(Fr)
        per = -(-n // world)
        lo = rank * per
        assert np.allclose(mine[:max(0, min(per, n - lo))], vb[lo:lo + per], rtol=0, atol=1e-15)
