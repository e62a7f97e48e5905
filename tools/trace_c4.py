"""debug: CTA-0 event trace of the chunked split-TF32 GEMM on configs[3] (FCFS_DEBUG bit 256).
Needs a library built with the trace compiled in:  python -c "from paper_1010_5562_b200 import build; build.build(extra=['-DFCFS_TRACE'])"
"""
import ctypes, os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FCFS_DEBUG"] = str(256 | int(sys.argv[2] if len(sys.argv) > 2 else 0))
import numpy as np, torch
from paper_1010_5562_b200 import fcfs, inputs
prec = sys.argv[1] if len(sys.argv) > 1 else "tf32x3"
wl = inputs.make("c4")
g = fcfs.vertices_from_rects(torch.from_numpy(wl.rects).cuda(), wl.T)
lib = fcfs._lib
lib.fcfs_debug_trace.restype = ctypes.c_int64
buf = (ctypes.c_ulonglong * 65536)()
area = int(g["area"][0].item())
for rep in range(2):
    lib.fcfs_debug_trace(buf, 65536)
    F = fcfs.coeffs(g["x"], g["y"], g["w"], area, wl.T, wl.M, wl.N, prec=prec)
    torch.cuda.synchronize()
n = lib.fcfs_debug_trace(buf, 65536)
ev = np.array(buf[:n], dtype=np.uint64)
t = (ev >> np.uint64(24)).astype(np.int64); e = ((ev >> np.uint64(16)) & np.uint64(0xFF)).astype(int); s = (ev & np.uint64(0xFFFF)).astype(int)
o = np.argsort(t, kind="stable"); t, e, s = t[o] - t[o][0], e[o], s[o]
np.savez(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", f"trace_c4_{prec}.npz"), t=t, e=e, s=s)
print("events", n, "span", t[-1])
first = collections.defaultdict(dict)
for ti, ei, si in zip(t, e, s):
    first[si].setdefault(ei, ti)
for sc in sorted(first)[40:60]:
    d = first[sc]
    b = min(d.values())
    print(sc, " ".join(f"{k}={v - b}" for k, v in sorted(d.items())))
mf = np.sort([v[50] for v in first.values() if 50 in v])
print("mma spacing median", np.median(np.diff(mf)), "mean", np.mean(np.diff(mf)))
