"""Runs every kernel of libfcfs.so once at small sizes, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck):  compute-sanitizer --tool <t> python tools/sanitize_driver.py [subset]

Subsets: extract, c1, c3, c4, haar, misc (default: all).  Each case checks nothing itself (the parity
tests do); it only has to launch the kernels so the sanitizer sees them.  Exits 0 when every call
returned FCFS_OK."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1010_5562_b200 import fcfs, inputs  # noqa: E402


def dev(a, dt):
    return None if a is None else torch.from_numpy(np.asarray(a)).to("cuda", dt)


def case_extract():
    wl = inputs.c2(seed=1, n_poly=60, T=1024)                            # grouped unions (general path)
    fcfs.vertices_from_rects(dev(wl.rects, torch.int32), wl.T, dev(wl.group_ptr, torch.int64))
    w3 = inputs.c3(seed=0, clips=8)                                      # per-clip bucket path
    fcfs.vertices_from_rects(dev(w3.rects, torch.int32), w3.T, None, dev(w3.clip_ptr, torch.int64))
    w4 = inputs.c4(seed=0, n_poly=3000, T=65536, M=8)                    # general singleton path + band
    r4 = dev(w4.rects, torch.int32)
    fcfs.vertices_from_rects(r4, w4.T)
    vp = fcfs.VerticesPlan(w4.R, w4.T)
    vp.run_band(r4, 1000, 30000)
    ps = inputs.polygon_clips(0, clips=3, T=256, n_poly=10)               # polygons
    fcfs.vertices_from_polygons(dev(ps.vx, torch.int32), dev(ps.vy, torch.int32), dev(ps.poly_ptr, torch.int64),
                                ps.T, dev(ps.clip_ptr, torch.int64))
    lay = inputs.layout(0, T=256, tiles_x=3, tiles_y=2, lines_per_tile=40)  # chop
    fcfs.chop_rects(dev(lay.rects, torch.int32), lay.T, 3, 2)


def case_c1():
    wl = inputs.c1(seed=0)
    g = fcfs.vertices_from_rects(dev(wl.rects, torch.int32), wl.T, dev(wl.group_ptr, torch.int64))
    a = int(g["area"][0])
    for route in ("gemm", "fft"):
        for prec in ("fp64", "tf32x3", "f16x3"):
            fcfs.coeffs(g["x"], g["y"], g["w"], a, wl.T, wl.M, wl.N, prec=prec, route=route)
    fcfs.row_buckets(g["y"])


def case_c3():
    w3 = inputs.c3(seed=0, clips=8)
    g = fcfs.vertices_from_rects(dev(w3.rects, torch.int32), w3.T, None, dev(w3.clip_ptr, torch.int64))
    for form in ("lattice", "edge", "corner"):
        fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], w3.T, w3.M, w3.N, w3.r2, "pupil",
                            "tf32x3", form=form)
    fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], w3.T, w3.M, w3.N, w3.r2, "pupil", "f16x3")
    fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], w3.T, 40, 33, -1.0, "dense", "tf32x3",
                        form="edge")                                     # multi-tile edge form
    fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], w3.T, 12, 12, -1.0, "dense", "fp64")
    fcfs.edges(g["corner_ptr"], g["x"], g["y"], g["w"])


def case_c4():
    w4 = inputs.c4(seed=0, n_poly=3000, T=65536, M=8)
    g = fcfs.vertices_from_rects(dev(w4.rects, torch.int32), w4.T)
    a = int(g["area"][0])
    M = N = 40
    for route in ("gemm", "fft"):
        for prec in ("fp64", "tf32x3"):
            fcfs.coeffs(g["x"], g["y"], g["w"], a, w4.T, M, N, prec=prec, route=route)
    sh = fcfs.Shard(fcfs.SHARD_ROWS, -5, 7, 0, 0)
    fcfs.coeffs(g["x"], g["y"], g["w"], a, w4.T, M, N, prec="fp64", shard=sh)
    sh = fcfs.Shard(fcfs.SHARD_VERTEX_BLOCK, 0, 0, 100, g["K"] // 2)
    fcfs.coeffs(g["x"], g["y"], g["w"], 0, w4.T, M, N, prec="fp64", shard=sh, route="gemm")


def case_haar():
    lay = inputs.layout(0, T=64, tiles_x=2, tiles_y=2, lines_per_tile=20)
    ch = fcfs.chop_rects(dev(lay.rects, torch.int32), lay.T, 2, 2)
    g = fcfs.vertices_from_rects(ch["rects"], lay.T, None, ch["tile_ptr"])
    fcfs.haar(g["x"], g["y"], g["w"], g["area"], lay.T, g["corner_ptr"])


def case_latency():
    wl = inputs.c1(seed=0)
    rects = dev(wl.rects, torch.int32)
    gp = dev(wl.group_ptr, torch.int64)
    sp = fcfs.SmallClipPlan(wl.R, wl.T, wl.M, wl.N, G=1, max_group=wl.R)
    sp.run(rects, gp)
    torch.cuda.synchronize()
    sp.check()
    w2 = inputs.c2(seed=2, n_poly=200)
    ap = fcfs.AsyncClipPlan(w2.R, w2.T, w2.M, w2.N, G=len(w2.group_ptr) - 1, max_group=int(np.diff(w2.group_ptr).max()))
    ap.run(dev(w2.rects, torch.int32), dev(w2.group_ptr, torch.int64))
    torch.cuda.synchronize()
    ap.check()


CASES = {"extract": case_extract, "c1": case_c1, "c3": case_c3, "c4": case_c4, "haar": case_haar,
         "latency": case_latency}

if __name__ == "__main__":
    fcfs.device_check()
    print(f"sanitize_driver: library {fcfs.LIB_PATH}", flush=True)
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        torch.cuda.synchronize()
        print(f"sanitize_driver: {n} ok, launches so far {fcfs.kernel_launches()}", flush=True)
