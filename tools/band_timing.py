"""Per-rank cost of the y-band sharded extraction (fcfs_vertices_from_rects_band) vs the unsharded one,
emulating P ranks one after another on one GPU (c4 / c5 single clips): the a1 stage of the multi-GPU
strong-scaling model in DESIGN.md §8."""
import os
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1010_5562_b200 import dist as fdist, fcfs, inputs  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


out = {}
for cfg in ("c4", "c5"):
    wl = inputs.make(cfg)
    rects = torch.from_numpy(wl.rects).cuda()
    vp = fcfs.VerticesPlan(wl.R, wl.T)
    full = timed(lambda: vp.run(rects))
    row = {"unsharded_ms": round(full, 4)}
    for P in (2, 4, 8):
        ts = []
        for r in range(P):
            ex = fdist.BandExtract(wl.R, wl.T, r, P)
            ts.append(timed(lambda: ex.run(rects)))
        row[f"P{P}_max_rank_ms"] = round(max(ts), 4)
    out[cfg] = row
print(json.dumps(out))
