"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, on the same
seeded inputs.  Tolerances (BASELINE.json north_star):
  extraction (x, y, w, corner_ptr, area): bit-exact
  F[0,0]: exact
  FP64:   |F_gpu - F_ref| <= 1e-12 * B[m,n]
  TF32X3: |F_gpu - F_ref| <= 1e-5  * B[m,n]
where B[m,n] = sum_k |term_k| is the oracle's per-coefficient L1 bound."""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_1010_5562_b200 import inputs

pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-12, "tf32x3": 1e-5, "f16x3": 1e-5}


@pytest.fixture(scope="module")
def fcfs():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1010_5562_b200 import fcfs as f
    f.device_check()
    return f


def _dev(a, dtype):
    return None if a is None else torch.as_tensor(np.asarray(a), dtype=dtype).cuda()


def _gpu_extract(fcfs, wl, check=True):
    """GPU extraction of a workload; with check (the default) it is first asserted bit-exact against
    oracle.extract on the same rects, so every coefficient test below runs on verified corners."""
    return _extract_checked(fcfs, wl.rects, wl.T, wl.group_ptr, wl.clip_ptr, check)


def _extract_checked(fcfs, rects, T, group_ptr=None, clip_ptr=None, check=True):
    g = fcfs.vertices_from_rects(_dev(rects, torch.int32), T, _dev(group_ptr, torch.int64),
                                 _dev(clip_ptr, torch.int64))
    if check:
        _assert_extract_equal(g, oracle.extract(rects, T, group_ptr, clip_ptr))
    return g


def _assert_extract_equal(g, e):
    assert g["K"] == e["K"]
    assert np.array_equal(g["x"].cpu().numpy(), e["x"])
    assert np.array_equal(g["y"].cpu().numpy(), e["y"])
    assert np.array_equal(g["w"].cpu().numpy(), e["w"])
    assert np.array_equal(g["corner_ptr"].cpu().numpy(), e["corner_ptr"])
    assert np.array_equal(g["area"].cpu().numpy(), e["area"])


def _assert_parity(F, Fref, B, prec, what, ms=None, ns=None):
    F = np.asarray(F, np.complex128)
    err = np.abs(F - Fref)
    tol = TOL[prec]
    bad = err > tol * B
    if ms is not None:
        dc = (ms == 0) & (ns == 0)
        if prec == "fp64":
            assert np.array_equal(F[dc], Fref[dc]), f"{what}: DC not exact"
        else:
            assert np.all(np.abs(F[dc] - Fref[dc]) <= 1e-7 * np.abs(Fref[dc]) + 1e-30), f"{what}: DC"
        bad &= ~dc
    if bad.any():
        i = int(np.argmax(np.where(B > 0, err / np.maximum(B, 1e-300), 0)))
        raise AssertionError(f"{what}: {bad.sum()} of {len(F)} outside {tol}*B; worst err/B = "
                             f"{err[i] / B[i]:.3e} at index {i}")


# ------------------------------------------------------------------ a1: extraction, bit-exact

@pytest.mark.parametrize("cfg", ["c1", "c2", "c3x64", "c3one", "c4", "c5"])
def test_extraction_bit_exact(fcfs, cfg):
    if cfg == "c3x64":
        wl = inputs.c3(clips=64)                     # per-clip SMEM sort path
    elif cfg == "c3one":
        wl = inputs.c3(clips=1)
        wl.clip_ptr = None                           # single clip, singleton groups, no clip CSR
    else:
        wl = inputs.make(cfg)
    e = oracle.extract(wl.rects, wl.T, wl.group_ptr, wl.clip_ptr)
    g = _gpu_extract(fcfs, wl)
    _assert_extract_equal(g, e)


def test_extraction_edge_cases(fcfs):
    # empty clip among non-empty ones; touching T; pinch (|w| = 2); duplicate rects summed across groups
    rects = np.array([[0, 0, 8, 8], [5, 5, 8, 8], [1, 1, 2, 2], [2, 2, 3, 3], [3, 3, 5, 5], [3, 3, 5, 5]], np.int32)
    gp = np.array([0, 2, 4, 5, 6], np.int64)       # groups: {0,1} union, {2,3} pinch, {4}, {5}
    cp = np.array([0, 1, 1, 4], np.int64)          # clip 1 is empty
    e = oracle.extract(rects, 8, gp, cp)
    g = fcfs.vertices_from_rects(_dev(rects, torch.int32), 8, _dev(gp, torch.int64), _dev(cp, torch.int64))
    _assert_extract_equal(g, e)
    assert 2 in np.abs(g["w"].cpu().numpy())
    # no rects at all
    g = fcfs.vertices_from_rects(torch.zeros((0, 4), dtype=torch.int32, device="cuda"), 16)
    assert g["K"] == 0 and g["area"].item() == 0
    # invalid rect -> E_RANGE
    with pytest.raises(fcfs.FcfsError) as ei:
        fcfs.vertices_from_rects(_dev(np.array([[2, 0, 2, 5]]), torch.int32), 8)
    assert ei.value.status == fcfs.E_RANGE
    with pytest.raises(fcfs.FcfsError) as ei:
        fcfs.vertices_from_rects(_dev(np.array([[2, 0, 9, 5]]), torch.int32), 8)
    assert ei.value.status == fcfs.E_RANGE


@pytest.mark.parametrize("per_clip", [1, 7, 300, 1344, 2000, 2600])
def test_extraction_heavy_ties_per_clip_paths(fcfs, per_clip):
    """Batched singleton-group clips on a 4-value coordinate grid: identical rects, shared and abutting
    edges, equal x inside every bucket (the paired rank loop of the per-clip bucket kernel ranks both
    corners of an edge against the bucket's edges), merged weights +-2 and cancelled corners.  1344 and
    2000 rects run the two per-clip variants, 2600 the general path; bit-exact vs oracle.extract."""
    rng = np.random.default_rng(per_clip)
    clips, T = 12, 8
    n = clips * per_clip
    xs = rng.choice([0, 2, 4, 6], size=(n, 2))
    ys = rng.choice([0, 3, 5, 7], size=(n, 2))
    x0, x1 = xs.min(1), xs.max(1)
    y0, y1 = ys.min(1), ys.max(1)
    x1 = np.where(x1 == x0, x0 + 2, x1)
    y1 = np.where(y1 == y0, y0 + 1, y1)
    rects = np.stack([x0, y0, x1, y1], 1).astype(np.int32)
    cp = np.arange(clips + 1, dtype=np.int64) * per_clip
    e = oracle.extract(rects, T, None, cp)
    g = fcfs.vertices_from_rects(_dev(rects, torch.int32), T, None, _dev(cp, torch.int64))
    _assert_extract_equal(g, e)


# ------------------------------------------------------------------ a2-a5: one clip, full window

def _clip_coeffs(fcfs, wl, prec, M=None, N=None, r2=None, layout="dense", shard=None):
    g = _gpu_extract(fcfs, wl)
    M = wl.M if M is None else M
    N = wl.N if N is None else N
    r2 = wl.r2 if r2 is None else r2
    F = fcfs.coeffs(g["x"], g["y"], g["w"], int(g["area"][0].item()), wl.T, M, N, r2, layout, prec, shard)
    torch.cuda.synchronize()
    return g, F.cpu().numpy()


def _oracle_window(g, T, M, N, r2=-1.0, layout="dense"):
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    area = int(g["area"][0].item())
    ms, ns = oracle.window(M, N, r2 if layout == "pupil" else -1.0)
    F, B = oracle.coeffs(x, y, w, area, T, ms, ns)
    if layout == "dense" and r2 >= 0:
        out = (ms.astype(np.float64) ** 2 + ns.astype(np.float64) ** 2) > r2
        F[out] = 0
        B[out] = 0
    return ms, ns, F, B


@pytest.mark.parametrize("cfg,prec", [("c1", "fp64"), ("c2", "fp64"), ("c1", "tf32x3"), ("c2", "tf32x3"),
                                      ("c1", "f16x3"), ("c2", "f16x3")])
def test_full_window_parity(fcfs, cfg, prec):
    wl = inputs.make(cfg)
    g, F = _clip_coeffs(fcfs, wl, prec)
    ms, ns, Fr, B = _oracle_window(g, wl.T, wl.M, wl.N)
    _assert_parity(F, Fr, B, prec, f"{cfg}/{prec}", ms, ns)
    # exact mirror: F[-m,-n] == conj F[m,n] bitwise
    Fm = F[::-1]
    assert np.array_equal(Fm.real, F.real) and np.array_equal(Fm.imag, -F.imag)


@pytest.mark.parametrize("prec", ["fp64", "tf32x3", "f16x3"])
def test_ragged_sizes_and_tiny_windows(fcfs, prec):
    # several tiles along both sides with ragged tails, non-power-of-two T, M != N, M = 0 / N = 0
    wl = inputs.c2(seed=7, n_poly=150, T=3000)
    for (M, N) in [(40, 23), (0, 5), (7, 0), (0, 0), (33, 31)]:
        g, F = _clip_coeffs(fcfs, wl, prec, M=M, N=N, r2=-1.0)
        ms, ns, Fr, B = _oracle_window(g, wl.T, M, N)
        _assert_parity(F, Fr, B, prec, f"M={M} N={N}", ms, ns)


@pytest.mark.parametrize("prec", ["fp64", "tf32x3", "f16x3"])
def test_pupil_layouts_single_clip(fcfs, prec):
    wl = inputs.c1(seed=1)
    r2 = 300.5
    for layout in ("pupil", "dense"):
        g, F = _clip_coeffs(fcfs, wl, prec, M=20, N=18, r2=r2, layout=layout)
        ms, ns, Fr, B = _oracle_window(g, wl.T, 20, 18, r2, layout)
        _assert_parity(F, Fr, B, prec, f"pupil/{layout}", ms, ns)


@pytest.mark.parametrize("prec", ["fp64", "tf32x3", "f16x3"])
def test_empty_corner_list(fcfs, prec):
    x = torch.zeros(0, dtype=torch.int32, device="cuda")
    F = fcfs.coeffs(x, x, x, 0, 64, 3, 3, prec=prec)
    torch.cuda.synchronize()
    assert torch.count_nonzero(F).item() == 0


# ------------------------------------------------------------------ a6 building blocks: shards on one GPU

@pytest.mark.parametrize("prec", ["fp64", "tf32x3", "f16x3"])
def test_row_shards_concatenate_to_full(fcfs, prec):
    wl = inputs.c2(seed=3, n_poly=400)
    g = _gpu_extract(fcfs, wl)
    area = int(g["area"][0].item())
    M = N = 40
    full = fcfs.coeffs(g["x"], g["y"], g["w"], area, wl.T, M, N, prec=prec).cpu().numpy()
    parts = []
    for lo, hi in [(-40, -14), (-13, -1), (0, 0), (1, 9), (10, 40)]:
        sh = fcfs.Shard(fcfs.SHARD_ROWS, lo, hi, 0, 0)
        parts.append(fcfs.coeffs(g["x"], g["y"], g["w"], area, wl.T, M, N, prec=prec, shard=sh).cpu().numpy())
    cat = np.concatenate(parts)
    ms, ns, Fr, B = _oracle_window(g, wl.T, M, N)
    _assert_parity(cat, Fr, B, prec, "row shards", ms, ns)
    _assert_parity(full, Fr, B, prec, "full", ms, ns)


@pytest.mark.parametrize("route", ["fft", "gemm"])
@pytest.mark.parametrize("prec", ["fp64", "tf32x3"])
def test_rows_to_peers_emulated_ranks(fcfs, route, prec):
    """fcfs_coeffs_rows_to_peers: P = 3 ranks emulated on one GPU, each rank's epilogue storing its rows into
    all three full-window buffers (the fused all_gather); every buffer equals the unsharded window bit for
    bit (and the oracle), including an empty rank and a rank that owns the m = 0 row."""
    wl = inputs.c2(seed=5, n_poly=300)
    g = _gpu_extract(fcfs, wl)
    area = int(g["area"][0].item())
    M = N = 24
    full = fcfs.coeffs(g["x"], g["y"], g["w"], area, wl.T, M, N, prec=prec, route=route)
    bufs = [torch.full_like(full, complex(7.0, 7.0)) for _ in range(3)]
    for lo, hi in [(-24, -1), (0, 24), (5, 4)]:             # the last rank owns no rows
        sh = fcfs.Shard(fcfs.SHARD_ROWS, lo, hi, 0, 0)
        if hi < lo:
            continue
        plan = fcfs.CoeffsPlan(g["K"], wl.T, M, N, prec=prec, shard=sh, route=route)
        plan.run_to_peers(g["x"], g["y"], g["w"], area, bufs)
    torch.cuda.synchronize()
    ms, ns, Fr, B = _oracle_window(g, wl.T, M, N)
    for i, b in enumerate(bufs):
        assert torch.equal(b, full), f"peer buffer {i} != unsharded window"
    _assert_parity(bufs[2].cpu().numpy(), Fr, B, prec, "peers", ms, ns)


def test_rows_to_peers_two_processes(fcfs):
    """Two processes on one GPU (gloo plumbing): each maps the other's full window by CUDA IPC
    (dist.peer_buffers) and its epilogue stores its rows into both (RowsPeers); both windows equal the
    unsharded window bit for bit.  (No kernel waits on another: the ordering is a host barrier.)"""
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_peers_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), "2", str(port)]) for r in range(2)]
    codes = [p.wait(timeout=300) for p in procs]
    assert codes == [0, 0]


def test_rows_to_peers_rejects_bad_arguments(fcfs):
    import ctypes
    wl = inputs.c1(seed=2)
    g = _gpu_extract(fcfs, wl)
    area = int(g["area"][0].item())
    buf = torch.zeros(fcfs.window_size(8, 8), dtype=torch.complex128, device="cuda")
    sh = fcfs.Shard(fcfs.SHARD_ROWS, -8, 8, 0, 0)
    plan = fcfs.CoeffsPlan(g["K"], wl.T, 8, 8, shard=sh)
    for peers in ([], [buf] * 9, [0]):
        with pytest.raises(fcfs.FcfsError) as ei:
            plan.run_to_peers(g["x"], g["y"], g["w"], area, peers)
        assert ei.value.status == fcfs.E_INVALID
    vb = fcfs.CoeffsPlan(g["K"], wl.T, 8, 8, shard=fcfs.Shard(fcfs.SHARD_VERTEX_BLOCK, 0, 0, 0, 4))
    with pytest.raises(fcfs.FcfsError) as ei:
        vb.run_to_peers(g["x"], g["y"], g["w"], area, [buf])
    assert ei.value.status == fcfs.E_INVALID


@pytest.mark.parametrize("prec", ["fp64", "tf32x3", "f16x3"])
def test_vertex_blocks_sum_to_full(fcfs, prec):
    wl = inputs.c2(seed=4, n_poly=600)
    g = _gpu_extract(fcfs, wl)
    K = g["K"]
    M = N = 24
    cuts = [0, K // 3, K // 2, K - 5, K]
    acc = None
    dc_abs = 0.0
    ms, ns, Fr, B = _oracle_window(g, wl.T, M, N)
    dc = (ms == 0) & (ns == 0)
    for a, b in zip(cuts[:-1], cuts[1:]):
        sh = fcfs.Shard(fcfs.SHARD_VERTEX_BLOCK, 0, 0, a, b)
        Fb = fcfs.coeffs(g["x"], g["y"], g["w"], 0, wl.T, M, N, prec=prec, shard=sh).cpu().numpy()
        Fb = Fb.astype(np.complex128)
        dc_abs += abs(Fb[dc][0])
        acc = Fb if acc is None else acc + Fb
    _assert_parity(acc[~dc], Fr[~dc], B[~dc], prec, "vertex blocks")
    if prec == "fp64":
        assert acc[dc][0] == Fr[dc][0]          # block DCs are exact integers / T^2: the sum is exact
    else:
        assert abs(acc[dc][0] - Fr[dc][0]) <= 2 ** -23 * 4 * dc_abs   # complex64 rounding of each block DC


# ------------------------------------------------------------------ batched clips (a5)

@pytest.mark.parametrize("prec", ["fp64", "tf32x3", "f16x3"])
def test_batched_pupil_clips(fcfs, prec):
    wl = inputs.c3(clips=24)
    g = _gpu_extract(fcfs, wl)
    F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], wl.T, wl.M, wl.N, wl.r2,
                            "pupil", prec).cpu().numpy()
    ms, ns = oracle.window(wl.M, wl.N, wl.r2)
    cp = g["corner_ptr"].cpu().numpy()
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    area = g["area"].cpu().numpy()
    for b in (0, 7, 23):
        sl = slice(cp[b], cp[b + 1])
        Fr, B = oracle.coeffs(x[sl], y[sl], w[sl], area[b], wl.T, ms, ns)
        _assert_parity(F[b], Fr, B, prec, f"clip {b}", ms, ns)


# ------------------------------------------------------------------ full BASELINE sizes, sampled outputs

def _sample_indices(M, N, n_rand=384, seed=0):
    """all axis + DC entries, the lowest |f| block, and seeded random (m, n)."""
    rng = np.random.default_rng(seed)
    pts = set()
    for m in range(-M, M + 1):
        pts.add((m, 0))
    for n in range(-N, N + 1):
        pts.add((0, n))
    for m in range(-4, 5):
        for n in range(-4, 5):
            pts.add((m, n))
    for _ in range(n_rand):
        pts.add((int(rng.integers(-M, M + 1)), int(rng.integers(-N, N + 1))))
    pts = sorted(pts)
    return np.array([p[0] for p in pts], np.int32), np.array([p[1] for p in pts], np.int32)


@pytest.mark.parametrize("cfg,prec", [("c4", "fp64"), ("c5", "fp64"), ("c4", "tf32x3"), ("c5", "tf32x3"),
                                      ("c4", "f16x3"), ("c5", "f16x3")])
def test_full_size_sampled(fcfs, cfg, prec):
    wl = inputs.make(cfg)
    g, F = _clip_coeffs(fcfs, wl, prec)
    ms, ns = _sample_indices(wl.M, wl.N, n_rand=128 if cfg == "c5" else 256)
    idx = (ms + wl.M) * (2 * wl.N + 1) + (ns + wl.N)
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    Fr, B = oracle.coeffs(x, y, w, int(g["area"][0].item()), wl.T, ms, ns)
    _assert_parity(F[idx], Fr, B, prec, f"{cfg} sampled", ms, ns)
    # properties that hold at any size: exact mirror
    assert np.array_equal(F[::-1].real, F.real) and np.array_equal(F[::-1].imag, -F.imag)


@pytest.mark.parametrize("prec", ["tf32x3", "f16x3"])
def test_batched_full_c3_sampled_clips(fcfs, prec):
    """BASELINE configs[2] at full size (4096 clips) in the launch configuration bench.py
    times (batched, pupil, split precision); the oracle checks a seeded sample of clips."""
    wl = inputs.c3(clips=4096)
    g = _gpu_extract(fcfs, wl)
    F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], wl.T, wl.M, wl.N, wl.r2,
                            "pupil", prec).cpu().numpy()
    ms, ns = oracle.window(wl.M, wl.N, wl.r2)
    cp = g["corner_ptr"].cpu().numpy()
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    area = g["area"].cpu().numpy()
    rng = np.random.default_rng(1)
    for b in sorted(set([0, 4095] + rng.integers(0, 4096, 6).tolist())):
        sl = slice(cp[b], cp[b + 1])
        Fr, B = oracle.coeffs(x[sl], y[sl], w[sl], area[b], wl.T, ms, ns)
        _assert_parity(F[b], Fr, B, prec, f"c3 clip {b}", ms, ns)
    assert np.all(np.isfinite(F))


# ------------------------------------------------------------------ a6: NCCL path (world size 1 on the one GPU)

def test_nccl_sharded_paths_world1(fcfs):
    import socket
    import torch.distributed as dist
    from paper_1010_5562_b200 import dist as fdist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        wl = inputs.c2(seed=9, n_poly=300)
        g = _gpu_extract(fcfs, wl)
        area = int(g["area"][0].item())
        for prec in ("fp64", "tf32x3"):
            full = fcfs.coeffs(g["x"], g["y"], g["w"], area, wl.T, 20, 20, prec=prec)
            rows = fdist.coeffs_rows_sharded(g["x"], g["y"], g["w"], area, wl.T, 20, 20, prec=prec)
            vb = fdist.coeffs_vertex_sharded(g["x"], g["y"], g["w"], wl.T, 20, 20, prec=prec)
            torch.cuda.synchronize()
            assert torch.equal(rows, full)
            ms, ns, Fr, B = _oracle_window(g, wl.T, 20, 20)
            _assert_parity(vb.cpu().numpy(), Fr, B, prec, f"vblock/{prec}", ms, ns)
        # the bench's single-clip pipeline through the real NCCL collectives: y-band a1 + all_gather of the
        # corner lists, then per-rank plans (rows, vertex blocks) reused across two steps
        w4 = inputs.c4(seed=4, n_poly=5000, T=65536, M=8)
        rects = torch.from_numpy(w4.rects).cuda()
        e = oracle.extract(w4.rects, w4.T)
        bx = fdist.BandExtract(w4.R, w4.T, 0, 1)
        rs = fdist.RowsSharded(w4.T, 16, 16, "fp64", 0, 1)
        vs = fdist.VertexSharded(w4.T, 16, 16, "fp64", 0, 1)
        rp = fdist.RowsPeers(w4.T, 16, 16, "fp64", 0, 1)
        for _ in range(2):
            x, y, w, K, area = fdist.extract_band_sharded(rects, w4.T, extractor=bx)
            assert K == e["K"] and area == int(e["area"][0])
            assert np.array_equal(x.cpu().numpy(), e["x"]) and np.array_equal(y.cpu().numpy(), e["y"])
            assert np.array_equal(w.cpu().numpy(), e["w"])
            Frow = rs.run(x, y, w, K, area)
            Fvb = vs.run(x, y, w, K)
            torch.cuda.synchronize()
            ms, ns = oracle.window(16, 16)
            Fr, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], w4.T, ms, ns)
            _assert_parity(Frow.cpu().numpy(), Fr, B, "fp64", "nccl rows", ms, ns)
            _assert_parity(Fvb.cpu().numpy(), Fr, B, "fp64", "nccl vblock", ms, ns)
            Fp = rp.run(x, y, w, K, area)                   # rows stored by the epilogue (peer = itself)
            torch.cuda.synchronize()
            assert torch.equal(Fp, Frow)
        assert len(rs.plans) == 1 and len(vs.plans) == 1 and len(rp.plans) == 1
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ row buckets (Step 4 row structure)

def _long_row_clip():
    """one clip whose rows hold thousands of corners: > kRowBucketCap corners per row and rows
    crossing the 4096-corner segment boundaries of the bucket pass."""
    T = 8192
    xs = np.arange(0, 2 * 2600, 2, dtype=np.int32)
    r = np.stack([xs, np.zeros_like(xs), xs + 1, np.full_like(xs, T)], axis=1)      # rows y = 0 and y = T
    extra = np.array([[10, 5, 20, 40], [3000, 17, 3400, 18], [100, 4000, 8192, 4001]], np.int32)
    return T, np.concatenate([r, extra]).astype(np.int32)


@pytest.mark.parametrize("prec", ["fp64", "tf32x3", "f16x3"])
def test_long_rows_and_unsorted_corners(fcfs, prec):
    T, rects = _long_row_clip()
    g = _extract_checked(fcfs, rects, T)
    area = int(g["area"][0].item())
    M = N = 12
    F = fcfs.coeffs(g["x"], g["y"], g["w"], area, T, M, N, prec=prec).cpu().numpy()
    ms, ns, Fr, B = _oracle_window(g, T, M, N)
    _assert_parity(F, Fr, B, prec, "long rows", ms, ns)
    # any corner order is valid (buckets are runs of equal consecutive y)
    perm = torch.from_numpy(np.random.default_rng(5).permutation(g["K"])).cuda()
    xp, yp, wp = (g[k][perm].contiguous() for k in ("x", "y", "w"))
    Fp = fcfs.coeffs(xp, yp, wp, area, T, M, N, prec=prec).cpu().numpy()
    _assert_parity(Fp, Fr, B, prec, "permuted corners", ms, ns)


@pytest.mark.parametrize("prec", ["fp64", "tf32x3", "f16x3"])
def test_batched_empty_and_tiny_clips(fcfs, prec):
    T, rects = _long_row_clip()
    small = np.array([[1, 1, 2, 2], [5, 5, 9, 6], [7000, 8000, 8192, 8192]], np.int32)
    allr = np.concatenate([small[:1], rects, small[1:]]).astype(np.int32)
    n = len(rects)
    cp = np.array([0, 1, 1, 1 + n, 1 + n, 3 + n], np.int64)          # clips: tiny, empty, long rows, empty, two rects
    g = _extract_checked(fcfs, allr, T, None, cp)
    M = N = 9
    F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], T, M, N, -1.0, "dense",
                            prec).cpu().numpy()
    ms, ns = oracle.window(M, N, -1.0)
    cpc = g["corner_ptr"].cpu().numpy()
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    area = g["area"].cpu().numpy()
    for b in range(5):
        sl = slice(cpc[b], cpc[b + 1])
        Fr, B = oracle.coeffs(x[sl], y[sl], w[sl], area[b], T, ms, ns)
        _assert_parity(F[b], Fr, B, prec, f"clip {b}", ms, ns)


def _edge_test_clips(rng, T):
    """corner lists for the edge form (edges.cu): canonical, permuted, an odd alternating chain on
    one row, arbitrary weights (zeros, +-2, +-3, duplicates) on few rows, one corner, empty."""
    r = inputs.random_rects(rng, 12, T, 8, 200)
    e = oracle.extract(r, T, np.array([0, len(r)], np.int64))
    canon = (e["x"], e["y"], e["w"])
    p = rng.permutation(len(e["x"]))
    perm = (e["x"][p], e["y"][p], e["w"][p])
    n = 9
    chain = (np.arange(10, 10 + 20 * n, 20, dtype=np.int32), np.full(n, 33, np.int32),
             np.array([1 if i % 2 == 0 else -1 for i in range(n)], np.int32))
    k = 700
    arb = (rng.integers(0, T + 1, k).astype(np.int32), rng.choice([0, 5, 6, T], k).astype(np.int32),
           rng.integers(-3, 4, k).astype(np.int32))
    one = (np.array([7], np.int32), np.array([9], np.int32), np.array([-2], np.int32))
    empty = (np.zeros(0, np.int32),) * 3
    # chains across the 32-corner chunks and 256-corner load groups of k_edges: alternating weights
    # on long runs of one row, with breaks (equal signs, row changes) at seeded places
    n = 1500
    ly = np.repeat(np.array([3, 4, 3, 90], np.int32), [333, 300, 600, 267])
    lw = np.where(np.arange(n) % 2 == 0, 1, -1).astype(np.int32)
    lw[rng.choice(n, 25, replace=False)] *= -1
    longc = (rng.integers(0, T + 1, n).astype(np.int32), ly, lw)
    return [canon, perm, chain, arb, one, empty, longc]


@pytest.mark.parametrize("edges", ["edge", "corner"])
def test_batched_edge_form_any_corner_list(fcfs, edges):
    """The batched split-TF32 contraction pairs corners into edges (edges.cu); the pairing is a
    term-by-term identity, so any corner list (order, weights) must give the oracle's result."""
    T, M, N = 512, 15, 13
    clips = _edge_test_clips(np.random.default_rng(11), T)
    cp = np.zeros(len(clips) + 1, np.int64)
    cp[1:] = np.cumsum([len(c[0]) for c in clips])
    x, y, w = (np.concatenate([c[i] for c in clips]).astype(np.int32) for i in range(3))
    area = np.array([int(np.sum(c[2].astype(np.int64) * c[0] * c[1])) for c in clips], np.int64)
    for prec in ("tf32x3", "f16x3"):
        F = fcfs.coeffs_batched(_dev(cp, torch.int64), _dev(x, torch.int32), _dev(y, torch.int32),
                                _dev(w, torch.int32), _dev(area, torch.int64), T, M, N, -1.0, "dense",
                                prec, form=edges).cpu().numpy()
        ms, ns = oracle.window(M, N, -1.0)
        for b in range(len(clips)):
            sl = slice(cp[b], cp[b + 1])
            Fr, B = oracle.coeffs(x[sl], y[sl], w[sl], area[b], T, ms, ns)
            _assert_parity(F[b], Fr, B, prec, f"{prec} clip {b} edges={edges}", ms, ns)


@pytest.mark.parametrize("form", ["edge", "corner"])
@pytest.mark.parametrize("layout", ["dense", "pupil"])
def test_batched_multi_tile_windows(fcfs, form, layout):
    """Windows wider than one 32-frequency tile (M = 40, N = 33: 2 x 2 tiles, the unfused batched path that
    writes P tiles and runs the stand-alone epilogue), non-power-of-two T, split-TF32 edge and corner forms
    and split-FP16, every clip against the oracle."""
    rng = np.random.default_rng(77)
    T, M, N = 3000, 40, 33
    sizes = [40, 0, 25, 60]
    cp = np.zeros(len(sizes) + 1, np.int64)
    cp[1:] = np.cumsum(sizes)
    rects = inputs.random_rects(rng, int(cp[-1]), T, 4, 700)
    g = _extract_checked(fcfs, rects, T, None, cp)
    r2 = 1300.5 if layout == "pupil" else -1.0
    ms, ns = oracle.window(M, N, r2)
    cpn = g["corner_ptr"].cpu().numpy()
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    area = g["area"].cpu().numpy()
    for prec in ("tf32x3", "f16x3"):
        F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], T, M, N, r2, layout, prec,
                                form=form).cpu().numpy()
        for b in range(len(sizes)):
            sl = slice(cpn[b], cpn[b + 1])
            Fr, B = oracle.coeffs(x[sl], y[sl], w[sl], area[b], T, ms, ns)
            _assert_parity(F[b], Fr, B, prec, f"{prec} {form} {layout} clip {b}", ms, ns)


# ------------------------------------------------------------------ lattice-row form (lattice.cu)

def _lattice_clips(rng, T, n_clips, sizes=None):
    """rect clips for the lattice-row form: random rects (summed groups: |w| up to 3 at coinciding corners),
    rects touching x = T / y = T and corners on the quarter-wave boundaries T/4, T/2, 3T/4."""
    rects, cps = [], [0]
    for b in range(n_clips):
        n = int(rng.integers(0, 50)) if sizes is None else sizes[b]
        r = inputs.random_rects(rng, n, T, 1, max(2, T // 5)) if n else np.zeros((0, 4), np.int32)
        if n >= 6:
            r[0] = [T // 4, T // 2, 3 * T // 4, T]                  # quarter-wave boundaries, y = T
            r[1] = [0, 0, T, max(1, T // 7)]                        # x = 0 .. T
            r[2] = r[3]                                             # duplicate: |w| = 2
            r[4] = [T // 2 - 1, 0, T // 2 + 1, max(1, T // 4)]
        rects.append(r.astype(np.int32))
        cps.append(cps[-1] + len(r))
    return np.concatenate(rects).astype(np.int32), np.array(cps, np.int64)


@pytest.mark.parametrize("T,M,N,layout", [(2048, 27, 27, "pupil"), (64, 31, 31, "dense"), (100, 9, 0, "dense"),
                                          (1000, 0, 13, "dense"), (2000, 10, 31, "masked"), (512, 31, 7, "pupil"),
                                          (8, 3, 3, "dense")])
def test_lattice_form_parity(fcfs, T, M, N, layout):
    """The lattice-row form against the oracle on every clip: T from 8 to 4096 (one table row per quarter
    wave up to T/4 + 1 = 1025), M, N from 0 to 31 (the kernel's limits), pupil / dense / masked-dense
    layouts, clip counts that are not a multiple of the 4-clip work item, empty clips, corners on x = T,
    y = T and the quarter-wave boundaries, weights |w| > 1."""
    rng = np.random.default_rng(T * 7 + M)
    B = 11
    rects, cp = _lattice_clips(rng, T, B)
    g = _extract_checked(fcfs, rects, T, None, cp)
    r2 = -1.0 if layout == "dense" else (0.7 * (M * M + N * N) + 1.5)
    lay = "pupil" if layout == "pupil" else "dense"
    assert fcfs.BatchedPlan(B, g["K"], 50 * 4, T, M, N, r2, lay, "tf32x3", form="lattice").form == fcfs.FORM_LATTICE
    for sorted_y in (False, True):
        F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], T, M, N, r2, lay, "tf32x3",
                                form="lattice", sorted_y=sorted_y).cpu().numpy()
        ms, ns = oracle.window(M, N, r2 if lay == "pupil" else -1.0)
        cpn = g["corner_ptr"].cpu().numpy()
        x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
        area = g["area"].cpu().numpy()
        for b in range(B):
            sl = slice(cpn[b], cpn[b + 1])
            Fr, Bd = oracle.coeffs(x[sl], y[sl], w[sl], area[b], T, ms, ns)
            if layout == "masked":
                out = (ms.astype(np.float64) ** 2 + ns.astype(np.float64) ** 2) > r2
                Fr[out] = 0
                Bd[out] = 0
            _assert_parity(F[b], Fr, Bd, "tf32x3", f"lattice T={T} clip {b} sorted_y={sorted_y}", ms, ns)
        assert np.array_equal(F.real, F[:, ::-1].real) and np.array_equal(F.imag, -F[:, ::-1].imag)


def test_lattice_form_unsorted_lists_fall_back(fcfs):
    """The lattice-row form needs y-sorted clips: an unsorted batch is detected on the device and takes the
    edge form (the result is still the oracle's)."""
    rng = np.random.default_rng(91)
    T, M, N = 2048, 27, 27
    rects, cp = _lattice_clips(rng, T, 6, sizes=[30, 40, 0, 25, 33, 8])
    g = _extract_checked(fcfs, rects, T, None, cp)
    cpn = g["corner_ptr"].cpu().numpy()
    perm = np.arange(g["K"])
    for b in range(6):
        perm[cpn[b]:cpn[b + 1]] = cpn[b] + rng.permutation(cpn[b + 1] - cpn[b])
    pt = torch.from_numpy(perm).cuda()
    xp, yp, wp = (g[k][pt].contiguous() for k in ("x", "y", "w"))
    r2 = inputs.pupil_r2(T)
    F = fcfs.coeffs_batched(g["corner_ptr"], xp, yp, wp, g["area"], T, M, N, r2, "pupil", "tf32x3",
                            form="lattice").cpu().numpy()
    ms, ns = oracle.window(M, N, r2)
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    area = g["area"].cpu().numpy()
    for b in range(6):
        sl = slice(cpn[b], cpn[b + 1])
        Fr, Bd = oracle.coeffs(x[sl], y[sl], w[sl], area[b], T, ms, ns)
        _assert_parity(F[b], Fr, Bd, "tf32x3", f"unsorted clip {b}", ms, ns)


def test_lattice_form_c3_all_clips_and_forms_agree(fcfs):
    """c3-shaped clips (BASELINE configs[2] statistics, 37 clips): the lattice-row form (AUTO picks it) checked
    clip by clip against the oracle, and against the edge form within twice the contract."""
    wl = inputs.c3(clips=37)
    g = _gpu_extract(fcfs, wl)
    kw = dict(prec="tf32x3")
    plan = fcfs.BatchedPlan(wl.B, g["K"], int(np.diff(g["corner_ptr"].cpu().numpy()).max()), wl.T, wl.M, wl.N,
                            wl.r2, "pupil", "tf32x3", sorted_y=True)
    assert plan.form == fcfs.FORM_LATTICE
    F = plan.run(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"]).cpu().numpy()
    Fe = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], wl.T, wl.M, wl.N, wl.r2, "pupil",
                             form="edge", **kw).cpu().numpy()
    ms, ns = oracle.window(wl.M, wl.N, wl.r2)
    cpn = g["corner_ptr"].cpu().numpy()
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    area = g["area"].cpu().numpy()
    for b in range(wl.B):
        sl = slice(cpn[b], cpn[b + 1])
        Fr, Bd = oracle.coeffs(x[sl], y[sl], w[sl], area[b], wl.T, ms, ns)
        _assert_parity(F[b], Fr, Bd, "tf32x3", f"c3 lattice clip {b}", ms, ns)
        assert np.all(np.abs(F[b].astype(np.complex128) - Fe[b]) <= 2e-5 * Bd + 1e-7 * np.abs(Fr)), f"forms {b}"


def _edges_reference(x, y, w, cp):
    """the pairing rule of include/fcfs.h (fcfs_edges) written out: links join consecutive corners of
    one clip with equal y and opposite weights; even chain positions emit an edge."""
    out = {"xa": [], "xb": [], "y": [], "c": [], "ecnt": []}
    for b in range(len(cp) - 1):
        n0 = len(out["xa"])
        pos = 0
        for k in range(cp[b], cp[b + 1]):
            link_in = k > cp[b] and y[k - 1] == y[k] and w[k - 1] == -w[k]
            pos = pos + 1 if link_in else 0
            if pos % 2 == 0:
                nxt = k + 1 < cp[b + 1] and y[k + 1] == y[k] and w[k + 1] == -w[k]
                out["xa"].append(x[k]); out["xb"].append(x[k + 1] if nxt else -1)
                out["y"].append(y[k]); out["c"].append(w[k])
        out["ecnt"].append(len(out["xa"]) - n0)
    return {k: np.array(v, np.int64) for k, v in out.items()}


def test_edge_pairing_bit_exact(fcfs):
    """fcfs_edges (the pre-pass of the batched split-TF32 contraction) against the rule written out:
    every clip's edge list bit-exact, on adversarial lists and on canonical c3 clips."""
    T = 512
    clips = _edge_test_clips(np.random.default_rng(11), T)
    wl = inputs.c3(clips=12)
    e3 = oracle.extract(wl.rects, wl.T, None, wl.clip_ptr)
    for b in range(12):
        sl = slice(e3["corner_ptr"][b], e3["corner_ptr"][b + 1])
        clips.append((e3["x"][sl], e3["y"][sl], e3["w"][sl]))
    cp = np.zeros(len(clips) + 1, np.int64)
    cp[1:] = np.cumsum([len(c[0]) for c in clips])
    x, y, w = (np.concatenate([c[i] for c in clips]).astype(np.int32) for i in range(3))
    g = fcfs.edges(_dev(cp, torch.int64), _dev(x, torch.int32), _dev(y, torch.int32), _dev(w, torch.int32))
    ref = _edges_reference(x.tolist(), y.tolist(), w.tolist(), cp.tolist())
    ecnt = g["ecnt"].cpu().numpy()
    assert np.array_equal(ecnt, ref["ecnt"])
    got = {k: g[k].cpu().numpy() for k in ("xa", "xb", "y", "c")}
    r0 = 0
    for b in range(len(clips)):
        n = int(ecnt[b])
        for k in ("xa", "xb", "y", "c"):
            assert np.array_equal(got[k][cp[b]:cp[b] + n], ref[k][r0:r0 + n]), f"clip {b} {k}"
        r0 += n
    # canonical lists pair up: about half as many edges as corners on c3
    assert ecnt[-12:].sum() < 0.6 * (cp[-1] - cp[-13])


def _buckets_reference(y, corner_ptr, cap, seg=4096):
    """the bucket rule of include/fcfs.h written out: runs of equal consecutive y, cut at clip
    starts, at k % seg == 0 and every `cap` corners from the run start."""
    K = len(y)
    starts = set(int(c) for c in corner_ptr[:-1]) if corner_ptr is not None else {0}
    bptr, by = [], []
    run = 0
    for k in range(K):
        rs = k == 0 or k in starts or k % seg == 0 or y[k] != y[k - 1]
        if rs:
            run = k
        if (k - run) % cap == 0:
            bptr.append(k)
            by.append(int(y[k]))
    bptr.append(K)
    b = np.asarray(bptr[:-1], np.int64)
    cb = [int(np.searchsorted(b, c, side="left")) for c in (corner_ptr if corner_ptr is not None else [0, K])]
    return np.asarray(bptr, np.int32), np.asarray(by, np.int32), np.asarray(cb, np.int64)


@pytest.mark.parametrize("cap", [1, 4, 32])
def test_row_buckets_bit_exact(fcfs, cap):
    # batched clips (tiny, empty, long rows crossing 4096-corner segments) and one permuted clip
    T, rects = _long_row_clip()
    small = np.array([[1, 1, 2, 2], [5, 5, 9, 6], [7000, 8000, 8192, 8192]], np.int32)
    allr = np.concatenate([small[:1], rects, small[1:]]).astype(np.int32)
    n = len(rects)
    cp = np.array([0, 1, 1, 1 + n, 1 + n, 3 + n], np.int64)
    g = _extract_checked(fcfs, allr, T, None, cp)
    for y, cptr in [(g["y"], g["corner_ptr"]),
                    (g["y"][torch.from_numpy(np.random.default_rng(2).permutation(g["K"])).cuda()].contiguous(), None)]:
        r = fcfs.row_buckets(y, cptr, cap)
        bp, byr, cb = _buckets_reference(y.cpu().numpy(), None if cptr is None else cptr.cpu().numpy(), cap)
        assert r["nb"] == len(byr)
        assert np.array_equal(r["bptr"].cpu().numpy(), bp)
        assert np.array_equal(r["by"].cpu().numpy(), byr)
        assert np.array_equal(r["clip_bptr"].cpu().numpy(), cb)


# ------------------------------------------------------------------ a1 from polygon vertex lists (NEXT-3)

def _gpu_polys(fcfs, ps):
    return fcfs.vertices_from_polygons(_dev(ps.vx, torch.int32), _dev(ps.vy, torch.int32),
                                       _dev(ps.poly_ptr, torch.int64), ps.T, _dev(ps.clip_ptr, torch.int64))


def _sub_polys(ps, clips):
    """The polygons of the listed clips as their own PolygonSet (for per-clip oracle checks)."""
    polys, per = [], []
    for b in clips:
        p0, p1 = int(ps.clip_ptr[b]), int(ps.clip_ptr[b + 1])
        for p in range(p0, p1):
            a, e = int(ps.poly_ptr[p]), int(ps.poly_ptr[p + 1])
            polys.append(list(zip(ps.vx[a:e].tolist(), ps.vy[a:e].tolist())))
        per.append(p1 - p0)
    return inputs._pack(polys, ps.T, per)


@pytest.mark.parametrize("case", ["small", "many_clips", "one_big_clip", "long_polygons", "long_perclip",
                                  "oversized_clip_fallback"])
def test_polygon_extraction_bit_exact(fcfs, case):
    if case == "small":
        ps = inputs.polygon_clips(0, clips=4, T=256, n_poly=20)
    elif case == "many_clips":
        ps = inputs.polygon_clips(1, clips=300, T=2048, n_poly=100, max_cols=8, size=60)
    elif case == "one_big_clip":
        ps = inputs.polygon_clips(2, clips=1, T=65536, n_poly=40000, max_cols=8, size=3000)
        ps.clip_ptr = None
    elif case == "long_polygons":                    # polygons of 100s of vertices, general path (T > 8191)
        ps = inputs.polygon_clips(3, clips=3, T=8192, n_poly=30, max_cols=200, size=20, collinear=0.5)
    elif case == "long_perclip":                     # the same on the per-clip bucket path (T <= 8191)
        ps = inputs.polygon_clips(5, clips=4, T=4096, n_poly=8, max_cols=200, size=10, collinear=0.5)
    else:                                            # a clip of > 8192 vertices: per-clip path falls back
        ps = inputs.polygon_clips(6, clips=3, T=2048, n_poly=700, max_cols=8, size=60)
        assert np.diff(ps.poly_ptr[ps.clip_ptr]).max() > 8192
    e = oracle.extract_polygons(ps.vx, ps.vy, ps.poly_ptr, ps.T, ps.clip_ptr)
    g = _gpu_polys(fcfs, ps)
    _assert_extract_equal(g, e)


def test_polygon_extraction_full_c3_as_polygons(fcfs):
    """BASELINE configs[2] rects given as 4-vertex polygons (4096 clips): identical to the rect
    extraction, and seeded clips bit-exact against the oracle's polygon extraction."""
    wl = inputs.c3(clips=4096)
    ps = inputs.rects_as_polygons(wl.rects, wl.T, wl.clip_ptr)
    g = _gpu_polys(fcfs, ps)
    gr = _gpu_extract(fcfs, wl)
    for k in ("x", "y", "w", "corner_ptr", "area"):
        assert torch.equal(g[k], gr[k]), k
    rng = np.random.default_rng(3)
    clips = sorted(set([0, 4095] + rng.integers(0, 4096, 6).tolist()))
    e = oracle.extract_polygons(*(lambda s: (s.vx, s.vy, s.poly_ptr, s.T, s.clip_ptr))(_sub_polys(ps, clips)))
    cp = g["corner_ptr"].cpu().numpy()
    for i, b in enumerate(clips):
        sl = slice(cp[b], cp[b + 1])
        el = slice(e["corner_ptr"][i], e["corner_ptr"][i + 1])
        for k in ("x", "y", "w"):
            assert np.array_equal(g[k][sl].cpu().numpy(), e[k][el]), (b, k)
        assert g["area"][b].item() == e["area"][i]


def test_polygon_edge_cases_and_errors(fcfs):
    T = 16
    one = lambda vx, vy: fcfs.vertices_from_polygons(_dev(np.array(vx), torch.int32), _dev(np.array(vy), torch.int32),
                                                     _dev(np.array([0, len(vx)]), torch.int64), T)
    # empty input; an empty polygon and an empty clip among non-empty ones
    g = fcfs.vertices_from_polygons(torch.zeros(0, dtype=torch.int32, device="cuda"),
                                    torch.zeros(0, dtype=torch.int32, device="cuda"),
                                    torch.zeros(1, dtype=torch.int64, device="cuda"), T)
    assert g["K"] == 0 and g["area"].item() == 0
    vx = np.array([0, 3, 3, 0, 10, 16, 16, 10, 0, 1, 2, 2, 2, 1, 0, 0], np.int32)
    vy = np.array([2, 2, 0, 0, 16, 16, 3, 3, 2, 2, 2, 1, 0, 0, 0, 1], np.int32)
    pp = np.array([0, 4, 4, 8, 16], np.int64)          # polygon 1 empty; polygon 3 has collinear vertices
    cp = np.array([0, 2, 2, 4], np.int64)              # clip 1 empty
    e = oracle.extract_polygons(vx, vy, pp, T, cp)
    g = fcfs.vertices_from_polygons(_dev(vx, torch.int32), _dev(vy, torch.int32), _dev(pp, torch.int64), T,
                                    _dev(cp, torch.int64))
    _assert_extract_equal(g, e)
    # counter-clockwise == clockwise
    a, b = one([0, 3, 3, 0], [2, 2, 0, 0]), one([0, 0, 3, 3], [2, 0, 0, 2])
    assert all(torch.equal(a[k], b[k]) for k in ("x", "y", "w", "area"))
    for vx, vy, st in (([0, 3, 3, 0], [2, 2, 0, 1], fcfs.E_INVALID),        # diagonal edge
                       ([0, 3, 3, 3, 0], [2, 2, 2, 0, 0], fcfs.E_INVALID),  # zero-length edge
                       ([0, T + 1, T + 1, 0], [2, 2, 0, 0], fcfs.E_RANGE)):  # outside [0, T]
        with pytest.raises(fcfs.FcfsError) as ei:
            one(vx, vy)
        assert ei.value.status == st


@pytest.mark.parametrize("prec", ["fp64", "tf32x3"])
def test_polygon_clips_coefficients(fcfs, prec):
    """Polygon input through the batched pupil path: clips against the oracle (corners and F)."""
    ps = inputs.polygon_clips(4, clips=16, T=2048, n_poly=120, max_cols=8, size=80)
    g = _gpu_polys(fcfs, ps)
    e = oracle.extract_polygons(ps.vx, ps.vy, ps.poly_ptr, ps.T, ps.clip_ptr)
    _assert_extract_equal(g, e)
    r2 = inputs.pupil_r2(ps.T)
    M = int(np.floor(np.sqrt(r2)))
    F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], ps.T, M, M, r2, "pupil",
                            prec).cpu().numpy()
    ms, ns = oracle.window(M, M, r2)
    cp = e["corner_ptr"]
    for b in (0, 5, 15):
        sl = slice(cp[b], cp[b + 1])
        Fr, B = oracle.coeffs(e["x"][sl], e["y"][sl], e["w"][sl], e["area"][b], ps.T, ms, ns)
        _assert_parity(F[b], Fr, B, prec, f"polygon clip {b}", ms, ns)


# ------------------------------------------------------------------ NEXT-2: the lattice-FFT route (FP64, one clip)

@pytest.fixture
def route(monkeypatch, fcfs):
    """route("fft" | "gemm") forces the single-clip route of every fcfs.coeffs call in the test
    (fcfs_options.route through the C-ABI)."""
    import functools
    orig = fcfs.coeffs

    def set_route(r):
        monkeypatch.setattr(fcfs, "coeffs", functools.partial(orig, route=r))
    yield set_route


@pytest.mark.parametrize("prec", ["fp64", "tf32x3", "f16x3"])
@pytest.mark.parametrize("r", ["fft", "gemm"])
@pytest.mark.parametrize("cfg,M,N", [("c1", 32, 32), ("c2", 64, 64), ("c2", 40, 23), ("c2", 7, 0), ("c2", 0, 9),
                                     ("c1", 20, 2047)])
def test_fft_route_full_window(fcfs, route, r, prec, cfg, M, N):
    """Both routes (FP64, and the FP32 route of the split precisions) against the oracle on full windows
    (T2 = 64 .. 4096, M != N, M = 0, N = 0)."""
    route(r)
    wl = inputs.make(cfg)
    if N == 2047:
        wl = inputs.c1(seed=2, T=8192)              # 2N+1 = 4095 <= T2 = 4096 (the largest FFT)
    g, F = _clip_coeffs(fcfs, wl, prec, M=M, N=N, r2=-1.0)
    ms, ns, Fr, B = _oracle_window(g, wl.T, M, N)
    _assert_parity(F, Fr, B, prec, f"{r} {cfg} M={M} N={N}", ms, ns)
    Fm = F[::-1]
    assert np.array_equal(Fm.real, F.real) and np.array_equal(Fm.imag, -F.imag)


@pytest.mark.parametrize("prec", ["fp64", "tf32x3"])
@pytest.mark.parametrize("r", ["fft", "gemm"])
def test_fft_route_shards_pupil_and_boundary(fcfs, route, r, prec):
    """ROWS shards (negative-only, across 0, positive), VERTEX_BLOCK partials, pupil layouts and corners
    on y = T / x = T (the raw y weight of the axis column, reading A7) through both routes."""
    route(r)
    rng = np.random.default_rng(11)
    T = 4096
    rects = inputs.random_rects(rng, 300, T, 20, 900)
    rects[:40, 3] = T                               # rects touching y = T
    rects[40:60, 2] = T                             # and x = T
    wl = inputs.Workload("edge", T, 50, 50, -1.0, rects, None, None, ("fp64",))
    g = _gpu_extract(fcfs, wl)
    area = int(g["area"][0].item())
    M = N = 50
    ms, ns, Fr, B = _oracle_window(g, T, M, N)
    full = fcfs.coeffs(g["x"], g["y"], g["w"], area, T, M, N, prec=prec).cpu().numpy()
    _assert_parity(full, Fr, B, prec, f"{r} full", ms, ns)
    parts = [fcfs.coeffs(g["x"], g["y"], g["w"], area, T, M, N, prec=prec,
                         shard=fcfs.Shard(fcfs.SHARD_ROWS, lo, hi, 0, 0)).cpu().numpy()
             for lo, hi in [(-50, -20), (-19, 5), (6, 6), (7, 50)]]
    _assert_parity(np.concatenate(parts), Fr, B, prec, f"{r} row shards", ms, ns)
    K = g["K"]
    acc = 0
    for a, b in [(0, K // 3), (K // 3, K - 7), (K - 7, K)]:
        sh = fcfs.Shard(fcfs.SHARD_VERTEX_BLOCK, 0, 0, a, b)
        acc = acc + fcfs.coeffs(g["x"], g["y"], g["w"], 0, T, M, N, prec=prec, shard=sh).cpu().numpy().astype(np.complex128)
    dc = (ms == 0) & (ns == 0)
    _assert_parity(acc[~dc], Fr[~dc], B[~dc], prec, f"{r} vertex blocks")
    if prec == "fp64":
        assert acc[dc][0] == Fr[dc][0]
    r2 = 1234.5
    for layout in ("pupil", "dense"):
        F = fcfs.coeffs(g["x"], g["y"], g["w"], area, T, M, N, r2, layout, prec).cpu().numpy()
        ms2, ns2, Fr2, B2 = _oracle_window(g, T, M, N, r2, layout)
        _assert_parity(F, Fr2, B2, prec, f"{r} {layout}", ms2, ns2)


@pytest.mark.parametrize("prec", ["fp64", "tf32x3"])
def test_fft_route_small_T2_many_subrows(fcfs, route, prec):
    """T2 = 64 with T1 = 1024 sub-rows (narrow window on a large tile), forced FFT route."""
    route("fft")
    wl = inputs.c4(seed=1, n_poly=20000)
    g, F = _clip_coeffs(fcfs, wl, prec, M=9, N=10, r2=-1.0)
    ms, ns, Fr, B = _oracle_window(g, wl.T, 9, 10)
    _assert_parity(F, Fr, B, prec, "T2=64", ms, ns)


# ------------------------------------------------------------------ NEXT-3: a layout chopped into tiles

def test_chop_bit_exact_and_errors(fcfs):
    rng = np.random.default_rng(5)
    T, tx, ty = 64, 5, 3
    W, H = T * tx, T * ty
    x0 = rng.integers(0, W - 1, 400); y0 = rng.integers(0, H - 1, 400)
    x1 = np.minimum(x0 + rng.integers(1, 200, 400), W); y1 = np.minimum(y0 + rng.integers(1, 150, 400), H)
    rects = np.stack([x0, y0, x1, y1], 1).astype(np.int32)
    rects[0] = (0, 0, W, H)
    rects[1] = (T - 1, T - 1, T + 1, T + 1)
    e = oracle.chop_rects(rects, T, tx, ty)
    g = fcfs.chop_rects(_dev(rects, torch.int32), T, tx, ty)
    assert g["n"] == e["n"]
    assert np.array_equal(g["rects"].cpu().numpy(), e["rects"])
    assert np.array_equal(g["tile_ptr"].cpu().numpy(), e["tile_ptr"])
    # capacity: a too-small plan reports the count, the helper retries
    plan = fcfs.ChopPlan(len(rects), T, tx, ty, cap=10)
    with pytest.raises(fcfs.FcfsError) as ei:
        plan.run(_dev(rects, torch.int32))
    assert ei.value.status == fcfs.E_CAPACITY and plan.n == e["n"]
    # empty layout; a rect outside the layout
    g = fcfs.chop_rects(torch.zeros((0, 4), dtype=torch.int32, device="cuda"), T, tx, ty)
    assert g["n"] == 0 and int(g["tile_ptr"].sum()) == 0
    with pytest.raises(fcfs.FcfsError) as ei:
        fcfs.chop_rects(_dev(np.array([[0, 0, W + 1, 5]]), torch.int32), T, tx, ty)
    assert ei.value.status == fcfs.E_RANGE


@pytest.mark.parametrize("prec", ["tf32x3", "fp64"])
def test_layout_tiles_end_to_end(fcfs, prec):
    """Layout -> chop -> batched extraction -> batched pupil coefficients; seeded tiles against the
    oracle's chop + extraction + direct sums."""
    lay = inputs.layout(seed=2, T=2048, tiles_x=6, tiles_y=5)
    ch = fcfs.chop_rects(_dev(lay.rects, torch.int32), lay.T, lay.tiles_x, lay.tiles_y)
    g = fcfs.vertices_from_rects(ch["rects"], lay.T, None, ch["tile_ptr"])
    r2 = inputs.pupil_r2(lay.T)
    M = int(np.floor(np.sqrt(r2)))
    F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], lay.T, M, M, r2, "pupil",
                            prec).cpu().numpy()
    eo = oracle.chop_rects(lay.rects, lay.T, lay.tiles_x, lay.tiles_y)
    ex = oracle.extract(eo["rects"], lay.T, None, eo["tile_ptr"])
    _assert_extract_equal(g, ex)
    ms, ns = oracle.window(M, M, r2)
    cp = ex["corner_ptr"]
    for t in (0, 7, 29):
        sl = slice(cp[t], cp[t + 1])
        Fr, B = oracle.coeffs(ex["x"][sl], ex["y"][sl], ex["w"][sl], ex["area"][t], lay.T, ms, ns)
        _assert_parity(F[t], Fr, B, prec, f"tile {t}", ms, ns)


# ------------------------------------------------------------------ NEXT-4: the continuous Haar transform

@pytest.mark.parametrize("case", ["c1_union_groups", "batched_polygons", "edges_at_T"])
def test_haar_bit_exact(fcfs, case):
    """Exact dyadic coefficients: bitwise equal to the oracle (child-cell areas of the corner form)."""
    if case == "c1_union_groups":
        wl = inputs.c1(seed=3, T=256, n_rects=40)
        g = _gpu_extract(fcfs, wl)
        H = fcfs.haar(g["x"], g["y"], g["w"], g["area"], wl.T).cpu().numpy()
        ref = oracle.haar(g["x"].cpu().numpy(), g["y"].cpu().numpy(), g["w"].cpu().numpy(), wl.T)
        assert np.array_equal(H[0], ref)
        return
    if case == "batched_polygons":
        ps = inputs.polygon_clips(7, clips=4, T=128, n_poly=12, max_cols=6, size=12)
        ps.clip_ptr[2] = ps.clip_ptr[1]             # clip 1 empty
        ps = inputs._pack([list(zip(ps.vx[a:b].tolist(), ps.vy[a:b].tolist()))
                           for a, b in zip(ps.poly_ptr[:-1], ps.poly_ptr[1:])], ps.T, np.diff(ps.clip_ptr).tolist())
        g = _gpu_polys(fcfs, ps)
        T = ps.T
    else:
        T = 64
        rects = np.array([[0, 0, 64, 64], [5, 60, 64, 64], [60, 3, 64, 9], [1, 1, 2, 2]], np.int32)
        wl = inputs.Workload("edge", T, 1, 1, -1.0, rects, np.array([0, 1, 4], np.int64), None, ("fp64",))
        g = _gpu_extract(fcfs, wl)
        g["corner_ptr"] = None
    H = fcfs.haar(g["x"], g["y"], g["w"], g["area"], T, g["corner_ptr"]).cpu().numpy()
    cp = g["corner_ptr"].cpu().numpy() if g["corner_ptr"] is not None else np.array([0, g["K"]])
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    for b in range(len(cp) - 1):
        sl = slice(cp[b], cp[b + 1])
        assert np.array_equal(H[b], oracle.haar(x[sl], y[sl], w[sl], T)), f"clip {b}"


def test_haar_plan_reuse_leaves_workspace_zero(fcfs):
    """A HaarPlan reused on different clips: every call clears the scratch it used (no per-call memset)."""
    ps = inputs.polygon_clips(8, clips=3, T=64, n_poly=10, max_cols=5, size=8)
    ps2 = inputs.polygon_clips(9, clips=3, T=64, n_poly=14, max_cols=5, size=8)
    plan = fcfs.HaarPlan(3, 64)
    for p in (ps, ps2, ps):
        g = _gpu_polys(fcfs, p)
        H = plan.run(g["x"], g["y"], g["w"], g["area"], g["corner_ptr"]).cpu().numpy()
        cp = g["corner_ptr"].cpu().numpy()
        x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
        for b in range(3):
            sl = slice(cp[b], cp[b + 1])
            assert np.array_equal(H[b], oracle.haar(x[sl], y[sl], w[sl], 64))
    assert torch.count_nonzero(plan.ws[:plan.scratch_bytes]).item() == 0


@pytest.mark.parametrize("T", [64, 256, 2048])
def test_haar_any_corner_order_scatter_path(fcfs, T):
    """Corner lists NOT sorted by y (fcfs_haar accepts any order): the device flag sends them through the
    scatter + scan path; bitwise equal to the oracle and to the band sweep on the sorted list, and the
    scatter scratch is left zero."""
    ps = inputs.polygon_clips(11, clips=3, T=T, n_poly=14, max_cols=6, size=max(4, T // 16))
    g = _gpu_polys(fcfs, ps)
    cp = g["corner_ptr"].cpu().numpy()
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    plan = fcfs.HaarPlan(3, T)
    Hs = plan.run(g["x"], g["y"], g["w"], g["area"], g["corner_ptr"]).cpu().numpy().copy()   # sorted: band sweep
    rng = np.random.default_rng(T)
    perm = np.concatenate([cp[b] + rng.permutation(cp[b + 1] - cp[b]) for b in range(3)]).astype(np.int64)
    xp, yp, wp = (torch.from_numpy(np.ascontiguousarray(a[perm])).cuda() for a in (x, y, w))
    Hu = plan.run(xp, yp, wp, g["area"], g["corner_ptr"]).cpu().numpy()
    for b in range(3):
        sl = slice(cp[b], cp[b + 1])
        ref = oracle.haar(x[sl], y[sl], w[sl], T)
        assert np.array_equal(Hs[b], ref), f"band sweep clip {b}"
        assert np.array_equal(Hu[b], ref), f"scatter path clip {b}"
    assert torch.count_nonzero(plan.ws[:plan.scratch_bytes]).item() == 0


# ------------------------------------------------------------------ maximum sizes and degenerate cases

@pytest.mark.parametrize("prec", ["fp64", "tf32x3"])
@pytest.mark.parametrize("r", ["fft", "gemm"])
def test_max_T_single_clip(fcfs, route, r, prec):
    """T = 2^20 (the ABI's limit): exact integer phases (m x) mod T near 2^40 and corners on x = T / y = T,
    through both single-clip routes."""
    route(r)
    T = 1 << 20
    rng = np.random.default_rng(21)
    x0 = rng.integers(0, T - 5000, 150); y0 = rng.integers(0, T - 5000, 150)
    rects = np.stack([x0, y0, x0 + rng.integers(1, 5000, 150), y0 + rng.integers(1, 5000, 150)], 1).astype(np.int32)
    rects[:10, 2] = T
    rects[10:20, 3] = T
    wl = inputs.Workload("maxT", T, 40, 40, -1.0, rects, None, None, ("fp64",))
    g, F = _clip_coeffs(fcfs, wl, prec)
    ms, ns, Fr, B = _oracle_window(g, T, 40, 40)
    _assert_parity(F, Fr, B, prec, f"T=2^20 {r}", ms, ns)


@pytest.mark.parametrize("prec", ["tf32x3", "fp64"])
def test_many_tiny_clips(fcfs, prec):
    """70,000 clips (more than a 65,535 grid dimension) of 1-3 rects, pupil window: every clip checked
    against the closed form of its rect sum through the oracle on a sample, and empty clips give 0."""
    rng = np.random.default_rng(22)
    T = 256
    B = 70000
    sizes = rng.integers(0, 4, B)
    cp = np.zeros(B + 1, np.int64); cp[1:] = np.cumsum(sizes)
    R = int(cp[-1])
    rects = inputs.random_rects(rng, R, T, 1, 60)
    g = fcfs.vertices_from_rects(_dev(rects, torch.int32), T, None, _dev(cp, torch.int64))
    e = oracle.extract(rects, T, None, cp)
    _assert_extract_equal(g, e)
    r2 = 30.5
    F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], T, 5, 5, r2, "pupil",
                            prec).cpu().numpy()
    ms, ns = oracle.window(5, 5, r2)
    for b in [0, 1, 65534, 65535, 65536, B - 1] + rng.integers(0, B, 20).tolist():
        a, c = e["corner_ptr"][b], e["corner_ptr"][b + 1]
        if a == c:
            assert not np.any(F[b]), f"empty clip {b}"
            continue
        Fr, Bd = oracle.coeffs(e["x"][a:c], e["y"][a:c], e["w"][a:c], e["area"][b], T, ms, ns)
        _assert_parity(F[b], Fr, Bd, prec, f"clip {b}", ms, ns)


@pytest.mark.parametrize("prec", ["fp64", "tf32x3", "f16x3"])
def test_degenerate_full_tile_and_window_beyond_T(fcfs, prec):
    """The full tile is a delta (P9: F = delta_{m0} delta_{n0}); a window wider than the tile (|m| > T/2,
    frequencies alias on the lattice but the CFS does not) still matches the oracle."""
    T = 64
    wl = inputs.Workload("full", T, 5, 5, -1.0, np.array([[0, 0, T, T]], np.int32), None, None, ("fp64",))
    g, F = _clip_coeffs(fcfs, wl, prec)
    ref = np.zeros_like(F); ref[len(F) // 2] = 1.0
    assert np.allclose(F, ref, atol=1e-12 if prec == "fp64" else 1e-6)
    rng = np.random.default_rng(23)
    wl = inputs.Workload("wide", T, 40, 40, -1.0, inputs.random_rects(rng, 10, T, 2, 30), None, None, ("fp64",))
    g, F = _clip_coeffs(fcfs, wl, prec)
    ms, ns, Fr, B = _oracle_window(g, T, 40, 40)
    _assert_parity(F, Fr, B, prec, "window beyond T", ms, ns)


def test_extraction_small_variant_overflow_reruns(fcfs):
    """Clips averaging under 1344 rects run the small per-clip kernel; one clip of 1500 rects overflows it
    and the batch reruns with the 2048-rect kernel: bit-exact either way."""
    rng = np.random.default_rng(31)
    T = 2048
    sizes = np.array([100, 1500, 80, 0, 300, 1344, 1345, 20], np.int64)
    cp = np.zeros(len(sizes) + 1, np.int64); cp[1:] = np.cumsum(sizes)
    rects = inputs.random_rects(rng, int(cp[-1]), T, 4, 300)
    e = oracle.extract(rects, T, None, cp)
    g = fcfs.vertices_from_rects(_dev(rects, torch.int32), T, None, _dev(cp, torch.int64))
    _assert_extract_equal(g, e)


@pytest.mark.parametrize("cfg,prec", [("c4", "fp64"), ("c4", "tf32x3"), ("c4", "f16x3"), ("c5", "fp64")])
def test_full_size_sampled_gemm_route(fcfs, route, cfg, prec):
    """The row-bucket GEMM routes (FP64 DMMA, split tcgen05) at the full BASELINE sizes: the lattice-FFT
    route is the default there, so the GEMMs are forced here (sampled outputs vs the oracle)."""
    route("gemm")
    wl = inputs.make(cfg)
    g, F = _clip_coeffs(fcfs, wl, prec)
    ms, ns = _sample_indices(wl.M, wl.N, n_rand=96 if cfg == "c5" else 160)
    idx = (ms + wl.M) * (2 * wl.N + 1) + (ns + wl.N)
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    Fr, B = oracle.coeffs(x, y, w, int(g["area"][0].item()), wl.T, ms, ns)
    _assert_parity(F[idx], Fr, B, prec, f"{cfg} gemm route sampled", ms, ns)


# ------------------------------------------------------------------ fused pairing (extraction writes the edges)

@pytest.mark.parametrize("cfg", ["c3x48", "c1", "c3big"])
def test_vertices_with_edges(fcfs, cfg):
    """fcfs_vertices_from_rects_edges: the corners equal the plain extraction's and the edges equal
    fcfs_edges' on them, on the per-clip bucket path, the general
    path (union groups) and the 2048-rect bucket variant; fcfs_coeffs_batched_edges
    with those edges gives bitwise the output of fcfs_coeffs_batched."""
    if cfg == "c3x48":
        wl = inputs.c3(clips=48)
    elif cfg == "c3big":
        wl = inputs.c3(clips=6, n_lines=1800)           # > 1344 rects per clip: the <512, 4> kernel
    else:
        wl = inputs.c1()
    rects = _dev(wl.rects, torch.int32)
    gp, cp = _dev(wl.group_ptr, torch.int64), _dev(wl.clip_ptr, torch.int64)
    G = wl.R if wl.group_ptr is None else len(wl.group_ptr) - 1
    mg = 1 if wl.group_ptr is None else int(np.diff(wl.group_ptr).max())
    vp = fcfs.VerticesPlan(wl.R, wl.T, G, wl.B, mg, grouped=wl.group_ptr is not None).enable_edges()
    K = vp.run(rects, gp, cp)
    g = fcfs.vertices_from_rects(rects, wl.T, gp, cp)
    _assert_extract_equal(g, oracle.extract(wl.rects, wl.T, wl.group_ptr, wl.clip_ptr))
    assert K == g["K"]
    for a, b in (("x", vp.x), ("y", vp.y), ("w", vp.w)):
        assert torch.equal(b[:K], g[a])
    assert torch.equal(vp.corner_ptr, g["corner_ptr"]) and torch.equal(vp.area, g["area"])
    ref = fcfs.edges(g["corner_ptr"], g["x"], g["y"], g["w"])
    assert torch.equal(vp.edges["ecnt"], ref["ecnt"])
    cpn = g["corner_ptr"].cpu().numpy()
    ec = ref["ecnt"].cpu().numpy()
    for k in ("xa", "xb", "y", "c"):
        a, b = vp.edges[k].cpu().numpy(), ref[k].cpu().numpy()
        for i in range(len(ec)):
            assert np.array_equal(a[cpn[i]:cpn[i] + ec[i]], b[cpn[i]:cpn[i] + ec[i]]), f"clip {i} {k}"
    if wl.B > 1:
        kmax = int(np.diff(cpn).max())
        plan = fcfs.BatchedPlan(wl.B, K, kmax, wl.T, wl.M, wl.N, wl.r2, "pupil", "tf32x3", form="edge")
        F1 = plan.run(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"]).clone()
        F2 = plan.run(vp.corner_ptr, vp.x[:K], vp.y[:K], vp.w[:K], vp.area, edges=vp.edges).clone()
        assert torch.equal(F1, F2)


# ------------------------------------------------------------------ seeded random sweep

@pytest.mark.parametrize("seed", list(range(32)))
def test_random_sweep(fcfs, seed):
    """Seeded random cases across the axes the paths branch on: T (power of two or not, small to
    5000), union groups or singleton rects, window M x N (M != N, zero), dense / pupil layout,
    precision, one clip (fcfs_coeffs: GEMM or FFT route) or a batch (fcfs_coeffs_batched: fused tcgen05
    kernel, edge form).  Every output against the oracle within its precision's bound."""
    rng = np.random.default_rng(1000 + seed)
    T = int(rng.choice([64, 100, 256, 1000, 2048, 4096, 5000]))
    prec = ["fp64", "tf32x3", "f16x3"][seed % 3]
    M, N = int(rng.integers(0, 49)), int(rng.integers(0, 49))
    layout = "pupil" if seed % 4 == 1 else "dense"
    r2 = float(rng.uniform(10, 2 * max(M, N, 1) ** 2)) if layout == "pupil" else -1.0
    batched = seed % 2 == 1
    B = 3 if batched else 1
    rects, cps = [], [0]
    for b in range(B):
        n = int(rng.integers(1, 60))
        r = inputs.random_rects(rng, n, T, 1, max(2, T // 6))
        rects.append(r)
        cps.append(cps[-1] + len(r))
    rects = np.concatenate(rects).astype(np.int32)
    cp = np.array(cps, np.int64)
    grouped = (not batched) and seed % 3 == 0
    gp = np.array([0, len(rects)], np.int64) if grouped else None
    e = oracle.extract(rects, T, gp, cp if batched else None)
    g = fcfs.vertices_from_rects(_dev(rects, torch.int32), T, _dev(gp, torch.int64),
                                 _dev(cp, torch.int64) if batched else None)
    _assert_extract_equal(g, e)
    ms, ns = oracle.window(M, N, r2 if layout == "pupil" else -1.0)
    if batched:
        F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], T, M, N, r2, layout,
                                prec).cpu().numpy()
        cpn = e["corner_ptr"]
        for b in range(B):
            sl = slice(cpn[b], cpn[b + 1])
            Fr, Bd = oracle.coeffs(e["x"][sl], e["y"][sl], e["w"][sl], e["area"][b], T, ms, ns)
            if layout == "dense" and r2 >= 0:
                out = (ms.astype(np.float64) ** 2 + ns.astype(np.float64) ** 2) > r2
                Fr[out] = 0
                Bd[out] = 0
            _assert_parity(F[b], Fr, Bd, prec, f"seed {seed} clip {b}", ms, ns)
    else:
        # single clip: the route the cost model picks, and (where eligible) the lattice-FFT route forced
        for route in (None, "fft"):
            F = fcfs.coeffs(g["x"], g["y"], g["w"], int(e["area"][0]), T, M, N, r2, layout, prec,
                            route=route).cpu().numpy()
            Fr, Bd = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], T, ms, ns)
            _assert_parity(F, Fr, Bd, prec, f"seed {seed} route {route}", ms, ns)


@pytest.mark.parametrize("seed", list(range(8)))
def test_haar_random_sweep(fcfs, seed):
    """Seeded random batches for fcfs_haar: T = 2 .. 512 (every level count), singleton or union
    rects, up to 3 clips with an empty one; bitwise equal to the oracle."""
    rng = np.random.default_rng(2000 + seed)
    T = int(2 ** rng.integers(1, 10))
    B = int(rng.integers(1, 4))
    rects, cps = [], [0]
    for b in range(B):
        n = 0 if (B > 1 and b == 1) else int(rng.integers(1, 40))
        r = inputs.random_rects(rng, n, T, 1, max(1, T // 3)) if n else np.zeros((0, 4), np.int32)
        rects.append(r)
        cps.append(cps[-1] + len(r))
    rects = np.concatenate(rects).astype(np.int32)
    cp = np.array(cps, np.int64)
    g = _extract_checked(fcfs, rects, T, None, cp)
    H = fcfs.haar(g["x"], g["y"], g["w"], g["area"], T, g["corner_ptr"]).cpu().numpy()
    cpn = g["corner_ptr"].cpu().numpy()
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    for b in range(B):
        sl = slice(cpn[b], cpn[b + 1])
        assert np.array_equal(H[b], oracle.haar(x[sl], y[sl], w[sl], T)), f"seed {seed} clip {b} T {T}"


@pytest.mark.parametrize("seed", list(range(8)))
def test_polygon_random_sweep(fcfs, seed):
    """Seeded random skyline-polygon batches (either orientation, collinear vertices, overlaps summed):
    extraction bit-exact against the oracle, then the batched split-TF32 coefficients of every clip."""
    rng = np.random.default_rng(3000 + seed)
    T = int(rng.choice([64, 200, 512, 2048]))
    clips = int(rng.integers(1, 5))
    ps = inputs.polygon_clips(4000 + seed, clips=clips, T=T, n_poly=int(rng.integers(1, 25)),
                              max_cols=int(rng.integers(2, 9)), collinear=float(rng.uniform(0, 0.5)))
    g = _gpu_polys(fcfs, ps)
    e = oracle.extract_polygons(ps.vx, ps.vy, ps.poly_ptr, ps.T, ps.clip_ptr)
    _assert_extract_equal(g, e)
    M, N = int(rng.integers(1, 20)), int(rng.integers(1, 20))
    F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], T, M, N, -1.0, "dense",
                            "tf32x3").cpu().numpy()
    ms, ns = oracle.window(M, N, -1.0)
    cpn = e["corner_ptr"]
    for b in range(clips):
        sl = slice(cpn[b], cpn[b + 1])
        Fr, Bd = oracle.coeffs(e["x"][sl], e["y"][sl], e["w"][sl], e["area"][b], T, ms, ns)
        _assert_parity(F[b], Fr, Bd, "tf32x3", f"seed {seed} clip {b}", ms, ns)


@pytest.mark.parametrize("seed", list(range(6)))
def test_chop_random_sweep(fcfs, seed):
    """Seeded random layouts for fcfs_chop_rects: T, tile grid and rect sizes drawn so rects span
    0 .. several tiles, some on tile boundaries; pieces and tile CSR bit-exact against the oracle."""
    rng = np.random.default_rng(5000 + seed)
    T = int(rng.choice([1, 7, 64, 100, 256]))
    tx, ty = int(rng.integers(1, 9)), int(rng.integers(1, 9))
    W, H = T * tx, T * ty
    n = int(rng.integers(0, 600))
    x0 = rng.integers(0, W, n); y0 = rng.integers(0, H, n)
    x1 = np.minimum(x0 + rng.integers(1, 3 * T + 2, n), W); y1 = np.minimum(y0 + rng.integers(1, 3 * T + 2, n), H)
    snap = rng.random(n) < 0.2                      # some corners exactly on tile lines
    x0 = np.where(snap, (x0 // T) * T, x0)
    rects = np.stack([x0, y0, x1, y1], 1).astype(np.int32).reshape(-1, 4)
    e = oracle.chop_rects(rects, T, tx, ty)
    g = fcfs.chop_rects(_dev(rects, torch.int32), T, tx, ty)
    assert g["n"] == e["n"]
    assert np.array_equal(g["rects"].cpu().numpy().reshape(-1, 4), np.asarray(e["rects"]).reshape(-1, 4))
    assert np.array_equal(g["tile_ptr"].cpu().numpy(), e["tile_ptr"])


# ---------------------------------------------------------------------------------------------
# multi-GPU single-clip path, emulated rank by rank on one GPU: y-band sharded extraction
# (fcfs_vertices_from_rects_band) and per-rank rows plans (dist.RowsSharded)
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("case", ["c4small", "c2small", "maxT"])
def test_band_extraction_concatenates_to_the_canonical_list(fcfs, case):
    from paper_1010_5562_b200 import dist as fdist
    if case == "c4small":
        wl = inputs.c4(seed=7, n_poly=20000, T=65536, M=8)
    elif case == "c2small":
        wl = inputs.c2(seed=7, n_poly=300, T=4096)
    else:   # the largest T: rects touching y = 0 and y = T (the last band holds row T)
        rng = np.random.default_rng(11)
        T = 1 << 20
        x0 = rng.integers(0, T - 10, 3000); y0 = rng.integers(0, T - 10, 3000)
        r = np.stack([x0, y0, np.minimum(x0 + rng.integers(1, 5000, 3000), T),
                      np.minimum(y0 + rng.integers(1, 5000, 3000), T)], 1).astype(np.int32)
        r[:3] = [[0, 0, 7, T], [5, T - 3, T, T], [T - 9, 0, T, 1]]
        wl = inputs.Workload("maxT", T, 4, 4, -1.0, r, None, None, ("fp64",))
    e = oracle.extract(wl.rects, wl.T, wl.group_ptr)
    rects = torch.from_numpy(wl.rects).cuda()
    gp = None if wl.group_ptr is None else torch.from_numpy(wl.group_ptr).cuda()
    G = wl.R if wl.group_ptr is None else len(wl.group_ptr) - 1
    mg = 1 if wl.group_ptr is None else int(np.diff(wl.group_ptr).max())
    for P in (1, 2, 3, 5, 8):
        xs, ys, ws, area = [], [], [], 0
        for rank in range(P):
            ex = fdist.BandExtract(wl.R, wl.T, rank, P, G=G, max_group=mg, grouped=gp is not None)
            x, y, w, K, a = ex.run(rects, gp)
            yy = y[:K].cpu().numpy()
            lo, hi = ex.band
            assert K == 0 or (yy.min() >= lo and yy.max() < hi)
            xs.append(x[:K].cpu().numpy()); ys.append(yy); ws.append(w[:K].cpu().numpy())
            area += int(a[0].item())
        assert np.array_equal(np.concatenate(xs), e["x"]), P
        assert np.array_equal(np.concatenate(ys), e["y"]), P
        assert np.array_equal(np.concatenate(ws), e["w"]), P
        assert area == int(e["area"][0]), P


def test_band_rejects_bad_band(fcfs):
    vp = fcfs.VerticesPlan(4, 64, device="cuda")
    rects = torch.tensor([[0, 0, 8, 8]] * 4, dtype=torch.int32, device="cuda")
    with pytest.raises(fcfs.FcfsError):
        vp.run_band(rects, 10, 5)
    with pytest.raises(fcfs.FcfsError):
        vp.run_band(rects, -1, 5)
    assert vp.run_band(rects, 3, 3) == 0          # an empty band is valid: no corners


@pytest.mark.parametrize("prec", ["fp64", "tf32x3"])
def test_rows_sharded_plans_reassemble_the_window(fcfs, prec):
    """Each emulated rank's RowsSharded plan (fcfs_shard ROWS, built once, run twice) gives its rows of
    the oracle window; the rank-ordered concatenation is the full window."""
    from paper_1010_5562_b200 import dist as fdist
    wl = inputs.c4(seed=2, n_poly=4000, T=65536, M=8)
    g = _gpu_extract(fcfs, wl)
    K = g["K"]
    M = N = 12
    ms, ns = oracle.window(M, N)
    e = oracle.extract(wl.rects, wl.T)
    Fr, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], wl.T, ms, ns)
    tol = 1e-12 if prec == "fp64" else 1e-5
    P = 3
    parts = []
    for rank in range(P):
        rs = fdist.RowsSharded(wl.T, M, N, prec, rank, P, device="cuda")
        loc = rs._local(g["x"], g["y"], g["w"], K, int(g["area"][0]))
        loc2 = rs._local(g["x"], g["y"], g["w"], K, int(g["area"][0]))
        torch.cuda.synchronize()
        assert len(rs.plans) == 1
        parts.append(loc2.cpu().numpy().copy())
        assert np.array_equal(loc.cpu().numpy(), parts[-1])
    F = np.concatenate(parts)
    err = np.abs(F.astype(np.complex128) - Fr)
    assert np.all(err <= tol * B + (B == 0) * 1e-7)


# ---------------------------------------------------------------------------------------------
# latency path: fcfs_small_clip (a1-a5 in one launch, no host sync, CUDA-graph capturable)
# ---------------------------------------------------------------------------------------------

def _small_case(name):
    if name == "c1":
        return inputs.c1(seed=0)
    if name == "c1s3":
        return inputs.c1(seed=3, T=3000, n_rects=90, M=20)         # T not a power of two
    if name == "singleton":
        rng = np.random.default_rng(4)
        r = inputs.random_rects(rng, 300, 8192, 4, 900)
        return inputs.Workload("singleton", 8192, 63, 40, -1.0, r, None, None, ("fp64",))
    if name == "pupil":
        w3 = inputs.c3(seed=1, clips=1, n_lines=120)
        return inputs.Workload("pupil", w3.T, w3.M, w3.N, w3.r2, w3.rects, None, None, ("tf32x3",))
    if name == "tiny":
        r = np.array([[0, 0, 1, 1], [3, 4, 7, 9]], np.int32)
        return inputs.Workload("tiny", 16, 5, 3, -1.0, r, np.array([0, 1, 2], np.int64), None, ("fp64",))
    raise KeyError(name)


@pytest.mark.parametrize("name", ["c1", "c1s3", "singleton", "pupil", "tiny"])
@pytest.mark.parametrize("prec", ["fp64", "tf32x3"])
def test_small_clip_matches_oracle(fcfs, name, prec):
    wl = _small_case(name)
    layout = "pupil" if wl.r2 >= 0 else "dense"
    gp = wl.group_ptr
    G = wl.R if gp is None else len(gp) - 1
    mg = 1 if gp is None else int(np.diff(gp).max())
    assert fcfs.SmallClipPlan.supported(wl.R, wl.T, wl.M, wl.N, wl.r2, layout, G, mg)
    plan = fcfs.SmallClipPlan(wl.R, wl.T, wl.M, wl.N, wl.r2, layout, prec, G=G, max_group=mg)
    F = plan.run(torch.from_numpy(wl.rects).cuda(), None if gp is None else torch.from_numpy(gp).cuda())
    torch.cuda.synchronize()
    e = oracle.extract(wl.rects, wl.T, gp)
    assert plan.check() == e["K"]
    ms, ns = oracle.window(wl.M, wl.N, wl.r2)
    Fr, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], wl.T, ms, ns)
    Fg = F.cpu().numpy().astype(np.complex128)
    tol = 1e-12 if prec == "fp64" else 1e-5
    err = np.abs(Fg - Fr)
    # B == 0 only at the DC, which is exact in FP64 and rounded once to complex64 otherwise
    zero_tol = 1e-15 if prec == "fp64" else 1e-7 * np.abs(Fr)
    assert np.all(err <= tol * B + (B == 0) * zero_tol), np.max(err / np.maximum(B, 1e-300))
    # the conjugate mirror is exact: F[-m, -n] == conj F[m, n]
    idx = {(int(m), int(n)): i for i, (m, n) in enumerate(zip(ms, ns))}
    Fc = F.cpu().numpy()
    for i, (m, n) in enumerate(zip(ms, ns)):
        j = idx[(-int(m), -int(n))]
        assert Fc[j] == np.conj(Fc[i])
    if prec == "fp64":
        assert Fc[idx[(0, 0)]].real == float(e["area"][0]) / (wl.T * wl.T)


def test_small_clip_graph_replay_and_status(fcfs):
    """The step is one launch with no host sync: capture it in a CUDA graph and replay it on new rects
    written into the same input buffer; device status reports a bad rect; host limits are enforced."""
    wl = inputs.c1(seed=0)
    w2 = inputs.c1(seed=9)
    assert wl.R == w2.R and len(wl.group_ptr) == len(w2.group_ptr)
    rects = torch.from_numpy(wl.rects).cuda()
    gp = torch.from_numpy(wl.group_ptr).cuda()
    plan = fcfs.SmallClipPlan(wl.R, wl.T, wl.M, wl.N, prec="fp64", G=1, max_group=wl.R)
    plan.run(rects, gp)                       # warm up (smem attribute, module load) outside the capture
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.run(rects, gp, stream=s)
    for src in (w2, wl):
        rects.copy_(torch.from_numpy(src.rects))
        g.replay()
        torch.cuda.synchronize()
        e = oracle.extract(src.rects, src.T, src.group_ptr)
        assert plan.check() == e["K"]
        ms, ns = oracle.window(src.M, src.N)
        Fr, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], src.T, ms, ns)
        assert np.all(np.abs(plan.out.cpu().numpy() - Fr) <= 1e-12 * B + (B == 0) * 1e-15)
    bad = torch.from_numpy(wl.rects).cuda()
    bad[3] = torch.tensor([5, 5, 5, 9])      # empty rect
    plan.run(bad, gp)
    torch.cuda.synchronize()
    with pytest.raises(fcfs.FcfsError):
        plan.check()
    assert not fcfs.SmallClipPlan.supported(10, 9000, 8, 8)                 # T > 8192
    assert not fcfs.SmallClipPlan.supported(600, 1024, 8, 8)                # 2400 raw corners
    with pytest.raises(fcfs.FcfsError):
        fcfs.SmallClipPlan(600, 1024, 8, 8).run(torch.zeros((600, 4), dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("route", ["gemm", "fft"])
@pytest.mark.parametrize("off", [1, 2, 3])
def test_corner_arrays_at_any_4_byte_offset(fcfs, route, off):
    """x, y, w views that start 4, 8 or 12 bytes into an allocation (e.g. rows of a gathered [3, K]
    tensor): every kernel must use vector loads only where the address itself is aligned."""
    wl = inputs.c4(seed=6, n_poly=3000, T=65536, M=8)
    g = _gpu_extract(fcfs, wl)
    K = g["K"]
    views = []
    for k in ("x", "y", "w"):
        buf = torch.zeros(K + 8, dtype=torch.int32, device="cuda")
        buf[off:off + K] = g[k][:K]
        views.append(buf[off:off + K])
    area = int(g["area"][0])
    F = fcfs.coeffs(*views, area, wl.T, 12, 12, prec="fp64", route=route)
    torch.cuda.synchronize()
    ms, ns, Fr, B = _oracle_window(g, wl.T, 12, 12)
    _assert_parity(F.cpu().numpy(), Fr, B, "fp64", f"offset {off} {route}", ms, ns)


def test_misaligned_rects_rejected(fcfs):
    wl = inputs.c1(seed=0)
    buf = torch.zeros(wl.R * 4 + 4, dtype=torch.int32, device="cuda")
    buf[1:1 + wl.R * 4] = torch.from_numpy(wl.rects).cuda().reshape(-1)
    bad = buf[1:1 + wl.R * 4].view(wl.R, 4)            # 4 bytes past a 16-byte boundary
    with pytest.raises(fcfs.FcfsError) as ex:
        fcfs.vertices_from_rects(bad, wl.T, torch.from_numpy(wl.group_ptr).cuda())
    assert ex.value.status == fcfs.E_INVALID


# ---------------------------------------------------------------------------------------------
# sync-free single-clip pipeline (fcfs_vertices_from_rects_async + fcfs_coeffs_async), graph replay
# ---------------------------------------------------------------------------------------------

@pytest.mark.parametrize("cfg,prec", [("c2", "fp64"), ("c2", "tf32x3"), ("c4", "fp64")])
def test_async_clip_pipeline_matches_oracle_and_replays(fcfs, cfg, prec):
    if cfg == "c2":
        wl = inputs.c2(seed=3, n_poly=400)
    else:
        wl = inputs.c4(seed=3, n_poly=20000, T=65536, M=48)
    gp = None if wl.group_ptr is None else torch.from_numpy(wl.group_ptr).cuda()
    G = wl.R if wl.group_ptr is None else len(wl.group_ptr) - 1
    mg = 1 if wl.group_ptr is None else int(np.diff(wl.group_ptr).max())
    rects = torch.from_numpy(wl.rects).cuda()
    plan = fcfs.AsyncClipPlan(wl.R, wl.T, wl.M, wl.N, prec=prec, G=G, max_group=mg)
    plan.run(rects, gp)
    torch.cuda.synchronize()
    e = oracle.extract(wl.rects, wl.T, wl.group_ptr)
    assert plan.check() == e["K"]
    K = e["K"]
    assert np.array_equal(plan.vp.x[:K].cpu().numpy(), e["x"]) and np.array_equal(plan.vp.w[:K].cpu().numpy(), e["w"])
    rng = np.random.default_rng(1)
    ms_all, ns_all = oracle.window(wl.M, wl.N)
    pick = rng.choice(len(ms_all), size=min(len(ms_all), 700), replace=False)
    Fr, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], wl.T, ms_all[pick], ns_all[pick])
    _assert_parity(plan.out.cpu().numpy()[pick], Fr, B, prec, f"async {cfg}", ms_all[pick], ns_all[pick])
    # capture the step and replay it on other rects written into the same buffer
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.run(rects, gp, stream=s)
    rects2 = wl.rects.copy()
    rects2[:, [0, 2]] = np.minimum(rects2[:, [0, 2]] + 3, wl.T)       # shifted in x (still valid)
    rects2 = rects2[rects2[:, 0] < rects2[:, 2]]
    if len(rects2) == wl.R:
        rects.copy_(torch.from_numpy(rects2))
        g.replay()
        torch.cuda.synchronize()
        e2 = oracle.extract(rects2, wl.T, wl.group_ptr)
        assert plan.check() == e2["K"]
        Fr2, B2 = oracle.coeffs(e2["x"], e2["y"], e2["w"], e2["area"][0], wl.T, ms_all[pick], ns_all[pick])
        _assert_parity(plan.out.cpu().numpy()[pick], Fr2, B2, prec, f"async replay {cfg}", ms_all[pick], ns_all[pick])


def test_async_clip_reports_errors_on_the_device(fcfs):
    wl = inputs.c2(seed=3, n_poly=50)
    gp = torch.from_numpy(wl.group_ptr).cuda()
    G = len(wl.group_ptr) - 1
    plan = fcfs.AsyncClipPlan(wl.R, wl.T, wl.M, wl.N, G=G, max_group=int(np.diff(wl.group_ptr).max()))
    bad = torch.from_numpy(wl.rects).cuda()
    bad[0] = torch.tensor([9, 9, 9, 20])          # empty rect
    plan.run(bad, gp)
    torch.cuda.synchronize()
    with pytest.raises(fcfs.FcfsError) as ex:
        plan.check()
    assert ex.value.status == fcfs.E_RANGE


@pytest.mark.parametrize("seed", range(10))
def test_lattice_form_random_sweep(fcfs, seed):
    """Seeded random configurations of the lattice-row form (T % 4 == 0 up to 2496, M, N in [0, 31], dense /
    pupil / masked, 1..13 clips of 0..60 rects; clip counts around the 4-clip item and chunk counts around
    the 12-row chunk and 21-chunk accumulation block) against the oracle on every clip."""
    rng = np.random.default_rng(1000 + seed)
    T = int(rng.choice([12, 48, 256, 1000, 1200, 2048, 2496, 4 * int(rng.integers(3, 600))]))
    M, N = int(rng.integers(0, 32)), int(rng.integers(0, 32))
    layout = ["dense", "pupil", "masked"][seed % 3]
    B = int(rng.integers(1, 14))
    rects, cp = _lattice_clips(rng, T, B, sizes=[int(v) for v in rng.integers(0, 61, B)])
    g = _extract_checked(fcfs, rects, T, None, cp)
    r2 = -1.0 if layout == "dense" else float(rng.uniform(0.2, 1.0) * (M * M + N * N) + 0.5)
    lay = "pupil" if layout == "pupil" else "dense"
    kmax = max(1, int(np.diff(g["corner_ptr"].cpu().numpy()).max()))
    plan = fcfs.BatchedPlan(B, g["K"], kmax, T, M, N, r2, lay, "tf32x3", form="lattice", sorted_y=True)
    assert plan.form == fcfs.FORM_LATTICE, (T, M, N)
    F = plan.run(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"]).cpu().numpy()
    ms, ns = oracle.window(M, N, r2 if lay == "pupil" else -1.0)
    cpn = g["corner_ptr"].cpu().numpy()
    x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
    area = g["area"].cpu().numpy()
    for b in range(B):
        sl = slice(cpn[b], cpn[b + 1])
        Fr, Bd = oracle.coeffs(x[sl], y[sl], w[sl], area[b], T, ms, ns)
        if layout == "masked":
            out = (ms.astype(np.float64) ** 2 + ns.astype(np.float64) ** 2) > r2
            Fr[out] = 0
            Bd[out] = 0
        _assert_parity(F[b], Fr, Bd, "tf32x3", f"lattice sweep seed {seed} T={T} M={M} N={N} clip {b}", ms, ns)


@pytest.mark.parametrize("seed", range(8))
def test_small_clip_random_sweep(fcfs, seed):
    """Seeded random small clips through fcfs_small_clip (one group of up to 100 rects, or up to 500
    singleton rects; T up to 8192 incl. non-powers of two; dense or pupil windows) against the oracle."""
    rng = np.random.default_rng(2000 + seed)
    T = int(rng.choice([16, 100, 1024, 3000, 4096, 8192]))
    M, N = int(rng.integers(0, min(64, T // 2 + 1))), int(rng.integers(0, min(200, T // 2 + 1)))
    grouped = seed % 2 == 0
    n = int(rng.integers(1, 101 if grouped else 501))
    r = inputs.random_rects(rng, n, T, 1, max(2, T // 6))
    gp = np.array([0, len(r)], np.int64) if grouped else None
    G = 1 if grouped else len(r)
    mg = len(r) if grouped else 1
    r2 = -1.0 if seed % 3 else float(rng.uniform(0.3, 1.0) * (M * M + N * N) + 0.5)
    layout = "pupil" if r2 >= 0 else "dense"
    if not fcfs.SmallClipPlan.supported(len(r), T, M, N, r2, layout, G, mg):
        pytest.skip("outside the small-clip limits")
    plan = fcfs.SmallClipPlan(len(r), T, M, N, r2, layout, "fp64", G=G, max_group=mg)
    plan.run(torch.from_numpy(r).cuda(), None if gp is None else torch.from_numpy(gp).cuda())
    torch.cuda.synchronize()
    try:
        K = plan.check()
    except fcfs.FcfsError as ex:          # a union with more than 2048 raw corners: reported, not wrong
        assert ex.status == fcfs.E_UNSUPPORTED
        return
    e = oracle.extract(r, T, gp)
    assert K == e["K"]
    ms, ns = oracle.window(M, N, r2)
    Fr, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], T, ms, ns)
    _assert_parity(plan.out.cpu().numpy(), Fr, B, "fp64", f"small sweep seed {seed}", ms, ns)


def test_c_demo_program_matches_oracle(fcfs, tmp_path):
    """The C-ABI driven from a plain C program (examples/fcfs_c_demo.c: cudaMalloc, fcfs_vertices_from_rects,
    fcfs_coeffs, no Python in the process): its FP64 window of a c1 clip equals the oracle within 1e-12 B
    and its K / area bit for bit."""
    import subprocess
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_abi_cpu import _build_c_demo
    exe = _build_c_demo(fcfs, str(tmp_path / "fcfs_c_demo"))
    wl = inputs.c1(seed=11)
    M = 16
    rects_bin, out_bin = tmp_path / "rects.bin", tmp_path / "out.bin"
    wl.rects.astype(np.int32).tofile(rects_bin)
    subprocess.check_call([exe, str(rects_bin), str(wl.R), str(wl.T), str(M), str(out_bin)], timeout=120)
    raw = np.fromfile(out_bin, dtype=np.uint8)
    nout = (2 * M + 1) ** 2
    F = raw[:nout * 16].view(np.complex128)
    K, area = raw[nout * 16:].view(np.int64)
    e = oracle.extract(wl.rects, wl.T, wl.group_ptr)
    assert K == e["K"] and area == int(e["area"][0])
    ms, ns = oracle.window(M, M)
    Fr, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], wl.T, ms, ns)
    _assert_parity(F, Fr, B, "fp64", "C demo", ms, ns)


def test_clips_async_extraction_and_graph_replay(fcfs):
    """fcfs_vertices_from_clips_async: bit-exact with the synchronising per-clip path; captured with the
    lattice-form batched coefficients in a CUDA graph and replayed on NEW rects (the graph reads the rects
    buffer); device status for a clip above max_clip_rects and for a bad rect."""
    wl = inputs.c3(seed=21, clips=24)
    rects = _dev(wl.rects, torch.int32)
    cp = _dev(wl.clip_ptr, torch.int64)
    vp = fcfs.VerticesPlan(wl.R, wl.T, None, wl.B, 1, grouped=False)
    vp.run_clips_async(rects, cp, 1200)
    torch.cuda.synchronize()
    K = vp.check_async()
    e = oracle.extract(wl.rects, wl.T, None, wl.clip_ptr)
    g = {"K": K, "x": vp.x[:K], "y": vp.y[:K], "w": vp.w[:K], "corner_ptr": vp.corner_ptr, "area": vp.area}
    _assert_extract_equal(g, e)
    kmax = int(np.diff(e["corner_ptr"]).max())
    plan = fcfs.BatchedPlan(wl.B, 4 * wl.R, 4 * 1200, wl.T, wl.M, wl.N, wl.r2, "pupil", "tf32x3", form="lattice",
                            sorted_y=True)   # upper bounds for K_total / K_max: planning only on this form
    assert plan.form == 3 and kmax <= 4 * 1200
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        vp.run_clips_async(rects, cp, 1200, stream=s)
        plan.run(vp.corner_ptr, vp.x, vp.y, vp.w, vp.area, stream=s)
    w2 = inputs.c3(seed=22, clips=24)
    for wk in (wl, w2):
        rects.copy_(_dev(wk.rects, torch.int32))   # same shapes (1200 rects per clip), new coordinates
        graph.replay()
        torch.cuda.synchronize()
        K2 = vp.check_async()
        ek = oracle.extract(wk.rects, wk.T, None, wk.clip_ptr)
        assert K2 == ek["K"]
        F = plan.out.view(wk.B, -1).cpu().numpy()
        ms, ns = oracle.window(wk.M, wk.N, wk.r2)
        for b in (0, 13, 23):
            sl = slice(ek["corner_ptr"][b], ek["corner_ptr"][b + 1])
            Fr, B = oracle.coeffs(ek["x"][sl], ek["y"][sl], ek["w"][sl], ek["area"][b], wk.T, ms, ns)
            _assert_parity(F[b], Fr, B, "tf32x3", f"graph clip {b}", ms, ns)
    # clips above the capacity the bound selects (1400 rects, bound 1200 -> the 1344-rect variant): device
    # status E_UNSUPPORTED; a bad rect: E_RANGE
    wb = inputs.c3(seed=23, clips=4, n_lines=1400)
    vb = fcfs.VerticesPlan(wb.R, wb.T, None, wb.B, 1, grouped=False)
    vb.run_clips_async(_dev(wb.rects, torch.int32), _dev(wb.clip_ptr, torch.int64), 1200)
    torch.cuda.synchronize()
    with pytest.raises(fcfs.FcfsError) as ei:
        vb.check_async()
    assert ei.value.status == fcfs.E_UNSUPPORTED
    vb.run_clips_async(_dev(wb.rects, torch.int32), _dev(wb.clip_ptr, torch.int64), 1400)   # the 2048 variant
    torch.cuda.synchronize()
    Kb = vb.check_async()
    eb = oracle.extract(wb.rects, wb.T, None, wb.clip_ptr)
    _assert_extract_equal({"K": Kb, "x": vb.x[:Kb], "y": vb.y[:Kb], "w": vb.w[:Kb], "corner_ptr": vb.corner_ptr,
                           "area": vb.area}, eb)
    bad = wl.rects.copy()
    bad[5] = [10, 10, 10, 20]
    vp.run_clips_async(_dev(bad, torch.int32), cp, 1200)
    torch.cuda.synchronize()
    with pytest.raises(fcfs.FcfsError) as ei:
        vp.check_async()
    assert ei.value.status == fcfs.E_RANGE
