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


# ------------------------------------------------------------------ polygon vertex lists

@dataclasses.dataclass
class PolygonSet:
    """Closed rectilinear polygons as vertex lists (the paper's input, Alg. 2 REQUIRE P:930-935).

    vx, vy    int32 [V] vertices; poly_ptr int64 [P+1] CSR over vertices;
    clip_ptr  int64 [B+1] CSR over polygons, or None (= one clip).
    """
    T: int
    vx: np.ndarray
    vy: np.ndarray
    poly_ptr: np.ndarray
    clip_ptr: np.ndarray | None

    @property
    def B(self) -> int:
        return 1 if self.clip_ptr is None else int(self.clip_ptr.shape[0] - 1)

    @property
    def P(self) -> int:
        return int(self.poly_ptr.shape[0] - 1)


def _pack(polys, T, per_clip=None) -> PolygonSet:
    sizes = np.array([len(p) for p in polys], np.int64)
    pp = np.zeros(len(polys) + 1, np.int64)
    pp[1:] = np.cumsum(sizes)
    V = np.concatenate([np.asarray(p, np.int64).reshape(-1, 2) for p in polys]) if polys else np.zeros((0, 2), np.int64)
    cp = None
    if per_clip is not None:
        cp = np.zeros(len(per_clip) + 1, np.int64)
        cp[1:] = np.cumsum(per_clip)
    return PolygonSet(T, V[:, 0].astype(np.int32), V[:, 1].astype(np.int32), pp, cp)


def skyline_polygon(rng, T, max_cols=6, size=None, collinear=0.0):
    """A random simple rectilinear polygon as a vertex list: a 'skyline' of 1..max_cols columns
    (widths / heights U{1..size}), in a random one of the 8 axis symmetries, placed at random inside
    [0,T]^2, listed in a random orientation from a random start vertex; with probability
    `collinear` per edge an extra vertex splits it (collinear vertices).  Pure vertex drawing."""
    size = size or max(1, T // (2 * max_cols))
    k = int(rng.integers(1, max_cols + 1))
    ws = rng.integers(1, size + 1, k)
    hs = rng.integers(1, size + 1, k)
    xs = np.concatenate([[0], np.cumsum(ws)])
    v = [(0, 0), (0, int(hs[0]))]
    for i in range(k):
        v.append((int(xs[i + 1]), int(hs[i])))
        v.append((int(xs[i + 1]), int(hs[i + 1]) if i + 1 < k else 0))
    # drop coincident consecutive vertices (equal neighbouring heights): the top edge just continues
    u = []
    for p in v:
        if not u or u[-1] != p:
            u.append(p)
    while len(u) > 1 and u[-1] == u[0]:
        u.pop()
    W, H = int(xs[-1]), int(hs.max())
    if rng.integers(0, 2):
        u = [(y, x) for x, y in u]
        W, H = H, W
    if rng.integers(0, 2):
        u = [(W - x, y) for x, y in u]
    if rng.integers(0, 2):
        u = [(x, H - y) for x, y in u]
    ox = int(rng.integers(0, T - W + 1)) if W <= T else 0
    oy = int(rng.integers(0, T - H + 1)) if H <= T else 0
    u = [(min(x + ox, T), min(y + oy, T)) for x, y in u]
    if rng.integers(0, 2):
        u = u[::-1]
    r = int(rng.integers(0, len(u)))
    u = u[r:] + u[:r]
    if collinear > 0:
        out = []
        for i, (a, b) in enumerate(u):
            out.append((a, b))
            c, d = u[(i + 1) % len(u)]
            if rng.random() < collinear and (abs(c - a) >= 2 or abs(d - b) >= 2):
                out.append(((a + c) // 2, (b + d) // 2))
        u = out
    return u


def polygon_clips(seed: int = 0, clips: int = 4, T: int = 256, n_poly: int = 20, max_cols: int = 6,
                  size=None, collinear: float = 0.2) -> PolygonSet:
    """`clips` clips of `n_poly` skyline polygons each (overlaps allowed: polygons are summed)."""
    polys = []
    for b in range(clips):
        rng = _rng(seed, b)
        polys += [skyline_polygon(rng, T, max_cols, size, collinear) for _ in range(n_poly)]
    return _pack(polys, T, [n_poly] * clips)


def rects_as_polygons(rects, T, clip_ptr=None) -> PolygonSet:
    """Every rect (x0, y0, x1, y1) as the clockwise (y up) list (x0,y1) (x1,y1) (x1,y0) (x0,y0),
    one polygon per rect; clip_ptr (over rects) carries over."""
    r = np.asarray(rects, np.int64).reshape(-1, 4)
    V = np.stack([np.stack([r[:, 0], r[:, 3]], 1), np.stack([r[:, 2], r[:, 3]], 1),
                  np.stack([r[:, 2], r[:, 1]], 1), np.stack([r[:, 0], r[:, 1]], 1)], 1).reshape(-1, 2)
    pp = np.arange(0, 4 * r.shape[0] + 1, 4, dtype=np.int64)
    cp = None if clip_ptr is None else np.asarray(clip_ptr, np.int64).copy()
    return PolygonSet(T, V[:, 0].astype(np.int32), V[:, 1].astype(np.int32), pp, cp)


# ------------------------------------------------------------------ layouts chopped into tiles (NEXT-3)

@dataclasses.dataclass
class Layout:
    """Rects over a tiles_x T x tiles_y T layout (layout coordinates), to be chopped into T x T tiles."""
    name: str
    T: int
    tiles_x: int
    tiles_y: int
    rects: np.ndarray      # int32 [R, 4], one group per rect


def layout(seed: int = 0, T: int = 2048, tiles_x: int = 64, tiles_y: int = 64, lines_per_tile: int = 1200) -> Layout:
    """c3-style standard-cell lines (rows of pitch 64 over the whole height, widths U{20..60}, lengths
    U{40..400}, x0 U{0..W-1}) at c3's density, over a layout of tiles_x x tiles_y tiles of side T; lines
    cross tile edges (the chop step splits them) and are clipped at the layout edge."""
    rng = _rng(seed, 1 << 20)
    Wd, Ht = tiles_x * T, tiles_y * T
    n = lines_per_tile * tiles_x * tiles_y
    row = rng.integers(0, Ht // 64, n)
    width = rng.integers(20, 61, n)
    yoff = rng.integers(0, 65 - width)
    length = rng.integers(40, 401, n)
    x0 = rng.integers(0, Wd, n)
    y0 = 64 * row + yoff
    x1 = np.minimum(x0 + length, Wd)
    y1 = np.minimum(y0 + width, Ht)
    r = np.stack([x0, y0, x1, y1], 1).astype(np.int32)
    return Layout("layout", T, tiles_x, tiles_y, r)


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}


def make(name: str, seed: int = 0, **kw) -> Workload:
    return CONFIGS[name](seed=seed, **kw)


def window_count(M: int, N: int, r2: float) -> int:
    """Number of output coefficients of a window (pure counting, no FCFS arithmetic)."""
    if r2 < 0:
        return (2 * M + 1) * (2 * N + 1)
    return sum(1 for m in range(-M, M + 1) for n in range(-N, N + 1) if m * m + n * n <= r2)
