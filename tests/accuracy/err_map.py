"""debug: err/B over a strided (m, n) grid of one config, printed as a tile map (max per tile)."""
import os, sys
sys.path.insert(0, os.environ.get("FCFS_PKG_ROOT", os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle
from paper_1010_5562_b200 import fcfs, inputs
cfg, prec = sys.argv[1], sys.argv[2]
wl = inputs.make(cfg)
g = fcfs.vertices_from_rects(torch.from_numpy(wl.rects).cuda(), wl.T, None if wl.group_ptr is None else torch.from_numpy(wl.group_ptr).cuda())
F = fcfs.coeffs(g["x"], g["y"], g["w"], int(g["area"][0].item()), wl.T, wl.M, wl.N, prec=prec).cpu().numpy()
st = int(sys.argv[3]) if len(sys.argv) > 3 else 16
mm, nn = np.meshgrid(np.arange(1, wl.M + 1, st), np.arange(-wl.N, wl.N + 1, st), indexing="ij")
ms, ns = mm.ravel().astype(np.int32), nn.ravel().astype(np.int32)
x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
Fr, B = oracle.coeffs(x, y, w, int(g["area"][0].item()), wl.T, ms, ns)
idx = (ms + wl.M) * (2 * wl.N + 1) + (ns + wl.N)
r = (np.abs(F[idx] - Fr) / np.maximum(B, 1e-300)).reshape(mm.shape)
print("max", r.max(), "median", np.median(r))
np.set_printoptions(linewidth=250)
print("log10 err/B, rows m = 1.., step", st, "cols n = -N.. step", st)
print(np.round(np.log10(np.maximum(r, 1e-12)), 1))
bad = np.argwhere(r > 1e-6)
print("bad (m, n):", [(int(mm[i, j]), int(nn[i, j])) for i, j in bad[:40]])
