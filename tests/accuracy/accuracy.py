"""Report max |F_gpu - F_oracle| / B over whole windows (GPU vs oracle) for each config and precision."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402
from paper_1010_5562_b200 import fcfs, inputs  # noqa: E402


def dev(a, dt):
    return None if a is None else torch.as_tensor(np.asarray(a), dtype=dt).cuda()


def main():
    out = {}
    for cfg in ["c1", "c2", "c3"]:
        wl = inputs.c3(clips=8) if cfg == "c3" else inputs.make(cfg)
        g = fcfs.vertices_from_rects(dev(wl.rects, torch.int32), wl.T, dev(wl.group_ptr, torch.int64),
                                     dev(wl.clip_ptr, torch.int64))
        layout = "pupil" if wl.r2 >= 0 else "dense"
        ms, ns = oracle.window(wl.M, wl.N, wl.r2 if layout == "pupil" else -1.0)
        cp = g["corner_ptr"].cpu().numpy()
        x, y, w = (g[k].cpu().numpy() for k in ("x", "y", "w"))
        area = g["area"].cpu().numpy()
        for prec in ["fp64", "tf32x3", "f16x3"]:
            F = fcfs.coeffs_batched(g["corner_ptr"], g["x"], g["y"], g["w"], g["area"], wl.T, wl.M, wl.N, wl.r2,
                                    layout, prec).cpu().numpy().astype(np.complex128)
            worst = 0.0
            for b in range(min(wl.B, 4)):
                sl = slice(cp[b], cp[b + 1])
                Fr, B = oracle.coeffs(x[sl], y[sl], w[sl], area[b], wl.T, ms, ns)
                nz = B > 0
                worst = max(worst, float(np.max(np.abs(F[b][nz] - Fr[nz]) / B[nz])))
            out[f"{cfg}/{prec}"] = worst
            print(cfg, prec, f"max err/B = {worst:.3e}", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
