"""Pipeline trace of the lattice kernel (diagnostic; needs libfcfs_trace.so built with -DLAT_TRACE).

Runs the c3 batched contraction once (warm) and again traced, reads CTA 0's clock64 stamps per chunk and
prints where the producers' stage waits come from: the stage's previous use (chunk g - 8) filled late by
another clip's warp (skew), or issued on time but its MMAs not yet complete (MMA latency).
Usage: FCFS_LIBRARY=paper_1010_5562_b200/libfcfs_trace.so python tools/lat_trace.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1010_5562_b200 import fcfs, inputs  # noqa: E402

wl = inputs.c3()
dev = "cuda"
rects = torch.from_numpy(wl.rects).to(dev)
cp = torch.from_numpy(wl.clip_ptr).to(dev)
vp = fcfs.VerticesPlan(wl.R, wl.T, B=wl.B, device=dev)
K = vp.run(rects, clip_ptr=cp)
corner_ptr, x, y, w, area = vp.corner_ptr, vp.x[:K], vp.y[:K], vp.w[:K], vp.area
kmax = int((corner_ptr[1:] - corner_ptr[:-1]).max().item())
plan = fcfs.BatchedPlan(wl.B, x.shape[0], kmax, wl.T, wl.M, wl.N, wl.r2, "pupil", "tf32x3", device=dev,
                        form="lattice", sorted_y=True)
for _ in range(3):
    plan.run(corner_ptr, x, y, w, area)
torch.cuda.synchronize()
lib = fcfs._lib
tr = np.zeros((8192, 12), np.int64)
trm = np.zeros((8192, 4), np.int64)
assert lib.fcfs_lat_trace_read(tr.ctypes.data_as(ctypes.c_void_p), trm.ctypes.data_as(ctypes.c_void_p)) == 0
n = int((tr[:, 8] != 0).sum())
tr, trm = tr[:n], trm[:n]
t0 = tr[:, :4].min()
ws, fs, full = tr[:, 0:4] - t0, tr[:, 4:8] - t0, tr[:, 8:12] - t0
mma = trm[:, 0] - t0
span = full.max() - ws.min()
wait = fs - ws
print(f"chunks {n}  span {span} clk  {span / n:.0f} clk/chunk")
print(f"producer wait per chunk-quadrant: mean {wait.mean():.0f}  p50 {np.median(wait):.0f}  p90 "
      f"{np.percentile(wait, 90):.0f}  total share {wait.sum() / (16 * span):.3f} of producer time")
fill = full - fs
print(f"fill time per chunk-quadrant: mean {fill.mean():.0f} p50 {np.median(fill):.0f} p90 {np.percentile(fill, 90):.0f}")
skew = full.max(1) - full.min(1)
print(f"quadrant skew of 'full' per chunk: mean {skew.mean():.0f} p90 {np.percentile(skew, 90):.0f}")
lag = mma - full.max(1)
print(f"MMA issue after last full: mean {lag.mean():.0f} p50 {np.median(lag):.0f} p90 {np.percentile(lag, 90):.0f}")
# for waits of chunk g: release time (fill start) - MMA issue of chunk g - 8
g = np.arange(8, n)
rel = fs[g].min(1) - mma[g - 8]
waited = wait[g].max(1) > 200
print(f"stage release after MMA issue of g-8 (waited chunks, {waited.sum()}): mean {rel[waited].mean():.0f} "
      f"p50 {np.median(rel[waited]):.0f} p10 {np.percentile(rel[waited], 10):.0f}")
late = (mma[g - 8] - ws[g].min(1))[waited]
print(f"  of those, MMA(g-8) issued after the wait began by: mean {late.mean():.0f} p50 {np.median(late):.0f}")
inorder = (mma[g - 8] - full[g - 8].max(1))[waited]
print(f"  MMA(g-8) issue - its own last full: mean {inorder.mean():.0f} p50 {np.median(inorder):.0f}")
prev = np.concatenate([[0], mma[:-1]])
pure = mma - np.maximum(full.max(1), prev)
print(f"MMA issue after max(own full, previous issue): mean {pure.mean():.0f} p50 {np.median(pure):.0f} "
      f"p90 {np.percentile(pure, 90):.0f}")
blocked = (prev > full.max(1)).mean()
print(f"chunks full before the previous chunk's MMA issued (in-order wait): {blocked:.2f}")
pre = trm[:, 2] - t0
bw = mma - pre
print(f"MMA warp 0: BFULL+FULL wait per chunk mean {bw.mean():.0f} p50 {np.median(bw):.0f}")
after_prev = pre - prev
print(f"MMA warp 0: loop top after previous stamp: mean {after_prev[1:].mean():.0f} p50 {np.median(after_prev[1:]):.0f}")
lastfull = full.max(1)
print(f"stamp - max(pre, lastfull): mean {(mma - np.maximum(pre, lastfull)).mean():.0f} "
      f"p50 {np.median(mma - np.maximum(pre, lastfull)):.0f}")
np.savez("gpurun_out/lat_trace.npz", tr=tr, trm=trm)
