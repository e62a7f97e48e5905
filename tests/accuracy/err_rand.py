"""debug: err/B on a dense random sample; list the bad entries with their tile/slot coordinates."""
import os, sys
sys.path.insert(0, os.environ.get("FCFS_PKG_ROOT", os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
sys.path.insert(1, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle
from paper_1010_5562_b200 import fcfs, inputs
cfg, prec, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
wl = inputs.make(cfg)
g = fcfs.vertices_from_rects(torch.from_numpy(wl.rects).cuda(), wl.T, None if wl.group_ptr is None else torch.from_numpy(wl.group_ptr).cuda())
F = fcfs.coeffs(g["x"], g["y"], g["w"], int(g["area"][0].item()), wl.T, wl.M, wl.N, prec=prec).cpu().numpy()
rng = np.random.default_rng(int(sys.argv[4]) if len(sys.argv) > 4 else 1)
ms = rng.integers(1, wl.M + 1, n).astype(np.int32); ns = rng.integers(-wl.N, wl.N + 1, n).astype(np.int32)
ns[ns == 0] = 1
x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
Fr, B = oracle.coeffs(x, y, w, int(g["area"][0].item()), wl.T, ms, ns)
idx = (ms + wl.M) * (2 * wl.N + 1) + (ns + wl.N)
r = np.abs(F[idx] - Fr) / np.maximum(B, 1e-300)
print("max", r.max(), "median", np.median(r), "bad>1e-7:", int((r > 1e-7).sum()))
for i in np.argsort(-r)[:25]:
    m, nn = int(ms[i]), int(ns[i]); pm, pn = m - 1, abs(nn) - 1
    print(f"  ({m},{nn}) err/B {r[i]:.2e}  A tile {pm // 32} slot {pm % 32}  B tile {pn // 32} slot {pn % 32}  |F| {abs(Fr[i]):.3e} B {B[i]:.3e}")
bad = r > 1e-7
import collections
pm, pn = ms - 1, np.abs(ns) - 1
for name, v in [("A tile", pm // 32), ("A slot", pm % 32), ("B tile", pn // 32), ("B slot", pn % 32), ("n sign", np.sign(ns))]:
    cb = collections.Counter(v[bad].tolist()); ca = collections.Counter(v.tolist())
    print(name, {k: f"{cb[k]}/{ca[k]}" for k in sorted(ca)})
