"""debug: worst err/B of the GPU path against the oracle on a sample of one config (no assertion)."""
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
rng = np.random.default_rng(0)
ms = rng.integers(-wl.M, wl.M + 1, 600).astype(np.int32); ns = rng.integers(-wl.N, wl.N + 1, 600).astype(np.int32)
ms[:40] = np.arange(40) - 20; ns[:40] = 0
idx = (ms + wl.M) * (2 * wl.N + 1) + (ns + wl.N)
x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
Fr, B = oracle.coeffs(x, y, w, int(g["area"][0].item()), wl.T, ms, ns)
r = np.abs(F[idx] - Fr) / np.maximum(B, 1e-300)
r[(ms == 0) & (ns == 0)] = 0
i = int(np.argmax(r))
print(f"{cfg} {prec} max err/B {r.max():.3e} at (m,n)=({ms[i]},{ns[i]}); median {np.median(r):.3e}; axis max {r[:40].max():.3e}")
