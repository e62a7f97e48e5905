"""debug: CTA-0 event trace of the batched tcgen05 kernel on configs[2] (FCFS_DEBUG bit 256 + flags).
Needs the trace compiled in: build with extra=['-DFCFS_TRACE'] (tools/_var/TR).  Events per stage sc:
10+2g+side = producer reaches its stage, 20+.. = EMPTY wait done, 30+.. = FULL arrive, 50 = MMA warp
passed the FULL waits of the pair starting at sc."""
import collections
import ctypes
import os
import sys

ROOT = os.environ.get("FCFS_PKG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ["FCFS_DEBUG"] = str(256 | int(sys.argv[1] if len(sys.argv) > 1 else 0))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1010_5562_b200 import fcfs, inputs  # noqa: E402

wl = inputs.c3(clips=148 * 4)
g = fcfs.vertices_from_rects(torch.from_numpy(wl.rects).cuda(), wl.T, None, torch.from_numpy(wl.clip_ptr).cuda())
lib = fcfs._lib
lib.fcfs_debug_trace.restype = ctypes.c_int64
buf = (ctypes.c_ulonglong * 65536)()
for rep in range(2):
    lib.fcfs_debug_trace(buf, 65536)
    fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], wl.T, wl.M, wl.N, wl.r2, "pupil", "tf32x3")
    torch.cuda.synchronize()
n = lib.fcfs_debug_trace(buf, 65536)
ev = np.array(buf[:n], dtype=np.uint64)
t = (ev >> np.uint64(24)).astype(np.int64)
e = ((ev >> np.uint64(16)) & np.uint64(0xFF)).astype(int)
s = (ev & np.uint64(0xFFFF)).astype(int)
o = np.argsort(t, kind="stable")
t, e, s = t[o] - t[o][0], e[o], s[o]
d = collections.defaultdict(dict)
for ti, ei, si in zip(t, e, s):
    d[si].setdefault(ei, ti)
rows = []
for sc in sorted(d)[100:-100]:
    x = d[sc]
    p = [k for k in x if 10 <= k < 20]
    if not p or 50 not in d.get(sc - (sc % 2), {}):
        continue
    g0 = min(p) % 10
    reach, empt, arr = x.get(10 + g0), x.get(20 + g0), x.get(30 + g0)
    arr1 = x.get(31 + g0 - (g0 % 2)) if (31 + g0 - (g0 % 2)) in x else arr
    if None in (reach, empt, arr):
        continue
    rows.append((sc, empt - reach, arr - empt, max(x.get(k, 0) for k in x if 30 <= k < 40) - empt))
r = np.array(rows)
mma = np.array(sorted(v[50] for v in d.values() if 50 in v))
print("stages", len(r), "EMPTY wait median", np.median(r[:, 1]), "wait->arrive median", np.median(r[:, 2]),
      "wait->last arrive median", np.median(r[:, 3]))
print("MMA pair spacing median", np.median(np.diff(mma)), "mean", np.mean(np.diff(mma)))
# latency from the later arrive of a stage to the MMA warp passing its FULL wait (pair start stages)
lat = []
for sc in sorted(d)[100:-100]:
    if sc % 2:
        continue
    x, y = d.get(sc, {}), d.get(sc + 1, {})
    arrs = [x[k] for k in x if 30 <= k < 40] + [y[k] for k in y if 30 <= k < 40]
    m = d.get(sc, {}).get(50)
    if arrs and m:
        lat.append(m - max(arrs))
print("last FULL arrive -> MMA passes (pair) median", np.median(lat))
