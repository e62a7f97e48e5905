"""debug: worst err/B of the batched c3 split-TF32 path against the oracle on 8 clips (no assertion;
FCFS_EDGES / FCFS_DEBUG select kernel variants)."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle
from paper_1010_5562_b200 import fcfs, inputs
wl = inputs.c3(clips=32)
g = fcfs.vertices_from_rects(torch.from_numpy(wl.rects).cuda(), wl.T, None, torch.from_numpy(wl.clip_ptr).cuda())
F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], wl.T, wl.M, wl.N, wl.r2, "pupil", "tf32x3").cpu().numpy()
ms, ns = oracle.window(wl.M, wl.N, wl.r2)
cp = g["corner_ptr"].cpu().numpy(); x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w")); area = g["area"].cpu().numpy()
worst = 0
for b in range(0, 32, 4):
    sl = slice(cp[b], cp[b + 1])
    Fr, B = oracle.coeffs(x[sl], y[sl], w[sl], area[b], wl.T, ms, ns)
    r = np.abs(F[b] - Fr) / np.maximum(B, 1e-300)
    r[(ms == 0) & (ns == 0)] = 0
    worst = max(worst, r.max())
print(os.environ.get("FCFS_DEBUG", "0"), os.environ.get("FCFS_EDGES", "1"), "worst err/B", worst)
