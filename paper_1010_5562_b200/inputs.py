"""Seeded synthetic workloads for the five BASELINE.json configs.

This module is the ONLY code shared by the CUDA path's tests/bench and the
CPU oracle.  It draws rectangles; it holds none of the FCFS arithmetic (no
corners, no phases, no coefficients).  The paper's benchmark layouts (22 nm
M1/M2/CA) are proprietary and absent, so these
generators stand in for them with BASELINE.json's shapes (recipes in
DESIGN.md "Input recipe").

Every config returns a ``Workload``:
  rects     int32 [R,4] (x0, y0, x1, y1), half-open, clipped at T (reading A13)
  group_ptr int64 [G+1] CSR over rects, or None (= every rect its own group)
  clip_ptr  int64 [B+1] CSR over groups, or None (= one clip)
  T, M, N, r2 (pupil radius^2, or -1 for the rectangular window)
PRNG: numpy ``default_rng(SeedSequence([seed, clip]))``; integer draws only.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class Workload:
    name: str
    T: int
    M: int
    N: int
    r2: float
    rects: np.ndarray
    group_ptr: np.ndarray | None
    clip_ptr: np.ndarray | None
    precisions: tuple

    @property
    def B(self) -> int:
        return 1 if self.clip_ptr is None else int(self.clip_ptr.shape[0] - 1)

    @property
    def R(self) -> int:
        return int(self.rects.shape[0])

    def clip_rect_range(self, b: int):
        """[r0, r1) rect range of clip b (groups are contiguous in rects)."""
        if self.clip_ptr is None:
            return 0, self.R
        g0, g1 = int(self.clip_ptr[b]), int(self.clip_ptr[b + 1])
        if self.group_ptr is None:
            return g0, g1
        return int(self.group_ptr[g0]), int(self.group_ptr[g1])


def _rng(seed, clip=0):
    return np.random.default_rng(np.random.SeedSequence([int(seed), int(clip)]))


def _clip(x0, y0, x1, y1, T):
    x0 = np.clip(x0, 0, T - 1)
    y0 = np.clip(y0, 0, T - 1)
    x1 = np.minimum(x1, T)
    y1 = np.minimum(y1, T)
    return np.stack([x0, y0, x1, y1], axis=1).astype(np.int32)


# NA(1+sigma)/lambda pupil of BASELINE.json configs[2]
NA, SIGMA, LAMBDA = 1.35, 0.9, 193.0


def pupil_r2(T: int) -> float:
    r = T * NA * (1.0 + SIGMA) / LAMBDA
    return r * r


def random_rects(rng, n, T, wlo, whi, hlo=None, hhi=None):
    hlo = wlo if hlo is None else hlo
    hhi = whi if hhi is None else hhi
    x0 = rng.integers(0, T, n)
    y0 = rng.integers(0, T, n)
    w = rng.integers(wlo, whi + 1, n)
    h = rng.integers(hlo, hhi + 1, n)
    return _clip(x0, y0, x0 + w, y0 + h, T)


def c1(seed: int = 0, T: int = 1024, n_rects: int = 64, M: int = 32) -> Workload:
    """configs[0]: 64 rects, corners U{0..T-1}, sides U{8..128}, one union group."""
    rng = _rng(seed)
    rects = random_rects(rng, n_rects, T, 8, 128)
    return Workload("c1", T, M, M, -1.0, rects, np.array([0, n_rects], np.int64), None, ("fp64",))


def _polygon(rng, T, lo, hi):
    """Anchor rect + U{0..4} extra rects of the same size law that overlap or touch it."""
    ax0, ay0 = rng.integers(0, T, 2)
    aw, ah = rng.integers(lo, hi + 1, 2)
    rects = [(ax0, ay0, ax0 + aw, ay0 + ah)]
    for _ in range(int(rng.integers(0, 5))):
        w, h = rng.integers(lo, hi + 1, 2)
        x0 = rng.integers(ax0 - w, ax0 + aw + 1)
        y0 = rng.integers(ay0 - h, ay0 + ah + 1)
        rects.append((x0, y0, x0 + w, y0 + h))
    r = np.array(rects, np.int64)
    return _clip(r[:, 0], r[:, 1], r[:, 2], r[:, 3], T)


def c2(seed: int = 0, T: int = 4096, n_poly: int = 2000, M: int = 64) -> Workload:
    """configs[1]: 2000 polygons, each the union of 1-5 rects (sides 16-256); one group each."""
    rng = _rng(seed)
    polys = [_polygon(rng, T, 16, 256) for _ in range(n_poly)]
    sizes = np.array([p.shape[0] for p in polys], np.int64)
    gp = np.zeros(n_poly + 1, np.int64)
    gp[1:] = np.cumsum(sizes)
    return Workload("c2", T, M, M, -1.0, np.concatenate(polys), gp, None, ("fp64", "tf32x3"))


def c3_clip(seed: int, clip: int, T: int = 2048, n_lines: int = 1200) -> np.ndarray:
    """One standard-cell-like clip: 1200 horizontal lines on 32 rows of pitch 64."""
    rng = _rng(seed, clip)
    row = rng.integers(0, 32, n_lines)
    width = rng.integers(20, 61, n_lines)
    yoff = rng.integers(0, 65 - width)            # U{0..64-width}
    length = rng.integers(40, 401, n_lines)
    x0 = rng.integers(0, T, n_lines)
    y0 = 64 * row + yoff
    return _clip(x0, y0, x0 + length, y0 + width, T)


def c3(seed: int = 0, clips: int = 4096, T: int = 2048, n_lines: int = 1200) -> Workload:
    """configs[2]: batched clips, one group per rect, pupil-disk output."""
    rects = np.concatenate([c3_clip(seed, b, T, n_lines) for b in range(clips)])
    cp = np.arange(0, clips + 1, dtype=np.int64) * n_lines
    r2 = pupil_r2(T)
    M = int(math.floor(math.sqrt(r2)))
    return Workload("c3", T, M, M, r2, rects, None, cp, ("tf32x3",))


def _wires_vias(rng, n, T, frac_via=0.2):
    nv = int(round(n * frac_via))
    nw = n - nv
    nh = nw // 2
    out = []
    # horizontal wires
    x0 = rng.integers(0, T, nh); y0 = rng.integers(0, T, nh)
    ln = rng.integers(100, 5001, nh); wd = rng.integers(20, 41, nh)
    out.append(_clip(x0, y0, x0 + ln, y0 + wd, T))
    # vertical wires
    nvv = nw - nh
    x0 = rng.integers(0, T, nvv); y0 = rng.integers(0, T, nvv)
    ln = rng.integers(100, 5001, nvv); wd = rng.integers(20, 41, nvv)
    out.append(_clip(x0, y0, x0 + wd, y0 + ln, T))
    # vias 24x24
    x0 = rng.integers(0, T, nv); y0 = rng.integers(0, T, nv)
    out.append(_clip(x0, y0, x0 + 24, y0 + 24, T))
    return np.concatenate(out)


def c4(seed: int = 0, T: int = 65536, n_poly: int = 250_000, M: int = 512) -> Workload:
    """configs[3]: routing-style tile: 80% wires (half H, half V), 20% 24x24 vias."""
    rng = _rng(seed)
    rects = _wires_vias(rng, n_poly, T, 0.2)
    return Workload("c4", T, M, M, -1.0, rects, None, None, ("fp64", "tf32x3"))


def c5(seed: int = 0, T: int = 262_144, n_rects: int = 1_000_000, M: int = 1024) -> Workload:
    """configs[4]: 50% c3-style lines, 40% c4-style wires, 10% vias; one group per rect."""
    rng = _rng(seed)
    n_lines = n_rects // 2
    row = rng.integers(0, T // 64, n_lines)
    width = rng.integers(20, 61, n_lines)
    yoff = rng.integers(0, 65 - width)
    length = rng.integers(40, 401, n_lines)
    x0 = rng.integers(0, T, n_lines)
    y0 = 64 * row + yoff
    lines = _clip(x0, y0, x0 + length, y0 + width, T)
    rest = _wires_vias(rng, n_rects - n_lines, T, 0.2)  # 40% wires + 10% vias of the total
    return Workload("c5", T, M, M, -1.0, np.concatenate([lines, rest]), None, None, ("fp64", "tf32x3"))


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def make(name: str, seed: int = 0, **kw) -> Workload:
    return CONFIGS[name](seed=seed, **kw)


def window_count(M: int, N: int, r2: float) -> int:
    """Number of output coefficients of a window (pure counting, no FCFS arithmetic)."""
    if r2 < 0:
        return (2 * M + 1) * (2 * N + 1)
    return sum(1 for m in range(-M, M + 1) for n in range(-N, N + 1) if m * m + n * n <= r2)
