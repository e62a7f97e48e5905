"""Host-side logic of bench.py that feeds the reported numbers (no GPU): the edge count used as the
roofline's K_inner for the batched split-TF32 kernel must follow the pairing rule of include/fcfs.h
(fcfs_edges), checked here against the rule written out as a loop."""
import os
import sys
import types

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _loop_count(y, w, cp):
    out = []
    for b in range(len(cp) - 1):
        n, pos = 0, 0
        for k in range(cp[b], cp[b + 1]):
            link = k > cp[b] and y[k - 1] == y[k] and w[k - 1] == -w[k]
            pos = pos + 1 if link else 0
            n += pos % 2 == 0
        out.append(n)
    return np.array(out, np.float64)


def test_edge_counts_match_the_rule():
    import bench
    rng = np.random.default_rng(7)
    for trial in range(20):
        B = int(rng.integers(1, 6))
        sizes = rng.integers(0, 60, B)
        cp = np.zeros(B + 1, np.int64)
        cp[1:] = np.cumsum(sizes)
        K = int(cp[-1])
        y = rng.integers(0, 4, K).astype(np.int32)          # few rows: long runs
        w = rng.choice([-2, -1, 1, 2], K).astype(np.int32)
        if trial % 3 == 0:                                 # alternating chains across clip boundaries
            w = np.where(np.arange(K) % 2 == 0, 1, -1).astype(np.int32)
            y[:] = 5
        vp = types.SimpleNamespace(y=torch.from_numpy(y), w=torch.from_numpy(w))
        got = bench.edge_counts(vp, K, cp)
        assert np.array_equal(got, _loop_count(y.tolist(), w.tolist(), cp.tolist())), trial
