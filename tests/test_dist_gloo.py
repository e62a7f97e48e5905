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
