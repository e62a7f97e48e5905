"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the pin of DESIGN.md "Oracle pins" (P1..P12, E1..E4) and the
PAPER.md passage ("P:n") it follows.  None of these re-types the oracle's
corner formula: every expected value comes from a different route (closed-form
rectangle integrals, rasterise + FFT with the exact cell transfer function,
per-cell brute force, numerical quadrature, the paper's own edge-length form on
polygon vertex lists, or hand values).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_1010_5562_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paper_hand_values.json")


def _window_coeffs(x, y, w, area, T, M, N):
    ms, ns = oracle.window(M, N)
    F, B = oracle.coeffs(x, y, w, area, T, ms, ns)
    return ms, ns, F, B


def _rect_closed_form(rect, T, ms, ns):
    """P2: F = (1/T^2) I(m; x0,x1) I(n; y0,y1), I(0) = L, I(m) = L e^{-i pi m (a+b)/T} sinc(m L / T)."""
    x0, y0, x1, y1 = [float(v) for v in rect]

    def I(k, a, b):
        L = b - a
        return np.where(k == 0, L + 0j, L * np.exp(-1j * np.pi * k * (a + b) / T) * np.sinc(k * L / T))

    return I(ms.astype(np.float64), x0, x1) * I(ns.astype(np.float64), y0, y1) / (T * T)


def _raster(rects, T, group_ptr=None):
    """f[a, b] = sum_groups 1[cell (a,b) in union of group] (half-open cells)."""
    img = np.zeros((T, T), np.int64)
    G = rects.shape[0] if group_ptr is None else len(group_ptr) - 1
    for g in range(G):
        r0, r1 = (g, g + 1) if group_ptr is None else (group_ptr[g], group_ptr[g + 1])
        sub = rects[r0:r1]
        if len(sub) == 0:
            continue
        bx0, by0 = sub[:, 0].min(), sub[:, 1].min()
        bx1, by1 = sub[:, 2].max(), sub[:, 3].max()
        loc = np.zeros((bx1 - bx0, by1 - by0), bool)
        for x0, y0, x1, y1 in sub:
            loc[x0 - bx0:x1 - bx0, y0 - by0:y1 - by0] = True
        img[bx0:bx1, by0:by1] += loc
    return img


def _cell_transfer(k, T):
    """S(k) = int_0^1 e^{-2 pi i k x / T} dx (unit-cell transfer function), S(0) = 1."""
    k = np.asarray(k, np.float64)
    z = 2j * np.pi * k / T
    with np.errstate(invalid="ignore", divide="ignore"):
        s = (1 - np.exp(-z)) / z
    return np.where(k == 0, 1.0 + 0j, s)


def _check(F, Fref, B, tol, what):
    err = np.abs(F - Fref)
    scale = np.maximum(B, 1e-300)
    worst = np.max(err / scale) if len(err) else 0.0
    assert np.all(err <= tol * B + 1e-300), f"{what}: max err/B = {worst:.3e} > {tol}"


# ---------------------------------------------------------------- P1: DC == area/T^2 (Eq. Fdc)

def test_P1_dc_is_exact_area():
    w = inputs.c1(seed=3)
    e = oracle.extract(w.rects, w.T, w.group_ptr)
    img = _raster(w.rects, w.T, w.group_ptr)
    assert e["area"][0] == int(img.sum())                       # area == raster pixel count
    F, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], w.T, np.array([0]), np.array([0]))
    assert F[0].real * w.T * w.T == e["area"][0] and F[0].imag == 0.0
    # disjoint rects: area == sum of rect areas (Step 1, "sum of polygon areas", Table I row 1 P:779)
    rects = np.array([[0, 0, 10, 7], [20, 3, 21, 90], [50, 50, 64, 64]], np.int32)
    e = oracle.extract(rects, 128)
    assert e["area"][0] == 70 + 87 + 196


# ---------------------------------------------------------------- P2: single rectangle closed form (Lemma 1)

@pytest.mark.parametrize("rect,T", [((3, 5, 17, 40), 64), ((0, 0, 1, 1), 8), ((100, 7, 1024, 333), 1024),
                                    ((0, 0, 64, 64), 64), ((63, 63, 64, 64), 64)])
def test_P2_single_rect_sinc_product(rect, T):
    e = oracle.extract(np.array([rect], np.int32), T)
    ms, ns, F, B = _window_coeffs(e["x"], e["y"], e["w"], e["area"][0], T, 9, 11)
    ref = _rect_closed_form(rect, T, ms, ns)
    dc = (ms == 0) & (ns == 0)
    assert F[dc][0] == ref[dc][0]
    _check(F[~dc], ref[~dc], B[~dc], 1e-13, "rect closed form")


def test_P2_far_frequencies():
    """CFS is not periodic in frequency: check m, n beyond T too."""
    rect, T = (5, 9, 12, 30), 32
    ms = np.array([33, -40, 64, 65, 100, 0, 31], np.int32)
    ns = np.array([1, 7, -3, 0, 64, 45, -95], np.int32)
    e = oracle.extract(np.array([rect], np.int32), T)
    F, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], T, ms, ns)
    _check(F, _rect_closed_form(rect, T, ms, ns), B, 1e-13, "far freq")
    # k = T, l = 0 -> 0 (SPEC cfs_query example S:319): rect closed form gives exactly 0 too
    F, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], T, np.array([T]), np.array([0]))
    assert abs(F[0]) <= 1e-15 * B[0] + 1e-300


# ---------------------------------------------------------------- P3: additivity (Prop. 2)

def test_P3_additive_over_disjoint_rects_and_groups():
    rng = np.random.default_rng(11)
    T = 256
    # disjoint rects on a coarse grid
    rects = []
    for gx in range(0, T, 32):
        for gy in range(0, T, 32):
            if rng.random() < 0.5:
                x0, y0 = gx + rng.integers(0, 8), gy + rng.integers(0, 8)
                rects.append((x0, y0, x0 + rng.integers(1, 24), y0 + rng.integers(1, 24)))
    rects = np.array(rects, np.int32)
    ms, ns = oracle.window(6, 6)
    e = oracle.extract(rects, T)
    F, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], T, ms, ns)
    acc = np.zeros_like(F)
    for r in rects:
        acc += _rect_closed_form(r, T, ms, ns)
    _check(F, acc, B, 1e-12, "sum of rects")
    # overlapping groups: F(sum of groups) == sum_g F(group g)  (signal model P:589-595, reading A5)
    w = inputs.c2(seed=1, n_poly=40, T=512)
    e = oracle.extract(w.rects, w.T, w.group_ptr)
    F, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], w.T, ms, ns)
    acc = np.zeros_like(F)
    for g in range(len(w.group_ptr) - 1):
        sub = w.rects[w.group_ptr[g]:w.group_ptr[g + 1]]
        eg = oracle.extract(sub, w.T, np.array([0, len(sub)]))
        Fg, _ = oracle.coeffs(eg["x"], eg["y"], eg["w"], eg["area"][0], w.T, ms, ns)
        acc += Fg
    _check(F, acc, B, 1e-12, "sum of groups")


# ---------------------------------------------------------------- P4: Hermitian symmetry by direct evaluation

def test_P4_conjugate_symmetry_direct():
    w = inputs.c2(seed=2, n_poly=200)
    e = oracle.extract(w.rects, w.T, w.group_ptr)
    ms, ns = oracle.window(20, 20)
    F, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], w.T, ms, ns)
    Fm, _ = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], w.T, -ms, -ns)
    _check(Fm, np.conj(F), B, 1e-15, "conj symmetry")


# ---------------------------------------------------------------- P5: translation phase

def test_P5_translation():
    w = inputs.c1(seed=5, T=1024)
    sh = w.rects.copy()
    sh = sh[(sh[:, 2] <= 900) & (sh[:, 3] <= 950)]
    dx, dy = 37, 61
    moved = sh + np.array([dx, dy, dx, dy], np.int32)
    ms, ns = oracle.window(8, 8)
    gp = np.array([0, len(sh)])
    e0 = oracle.extract(sh, 1024, gp)
    e1 = oracle.extract(moved, 1024, gp)
    F0, B0 = oracle.coeffs(e0["x"], e0["y"], e0["w"], e0["area"][0], 1024, ms, ns)
    F1, B1 = oracle.coeffs(e1["x"], e1["y"], e1["w"], e1["area"][0], 1024, ms, ns)
    ph = np.exp(-2j * np.pi * (ms * dx + ns * dy) / 1024)
    ax = (ms == 0) | (ns == 0)
    _check(F1[~ax], F0[~ax] * ph[~ax], B0[~ax], 1e-13, "translation interior")
    # axis bounds scale with coordinates; use the larger of the two bounds
    _check(F1[ax], F0[ax] * ph[ax], np.maximum(B0[ax], B1[ax]) + 1e-300, 1e-13, "translation axes")


# ---------------------------------------------------------------- P6: exact raster identity

@pytest.mark.parametrize("cfg", ["c1", "c2small"])
def test_P6_raster_fft_identity(cfg):
    if cfg == "c1":
        w = inputs.c1(seed=0)
    else:
        w = inputs.c2(seed=4, n_poly=300, T=1024)
    e = oracle.extract(w.rects, w.T, w.group_ptr)
    img = _raster(w.rects, w.T, w.group_ptr).astype(np.float64)
    D = np.fft.fft2(img)                        # D[k,l] = sum f[a,b] e^{-2 pi i (k a + l b)/T}
    ms, ns = oracle.window(24, 24)
    F, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], w.T, ms, ns)
    ref = D[ms % w.T, ns % w.T] * _cell_transfer(ms, w.T) * _cell_transfer(ns, w.T) / (w.T * w.T)
    # the FFT route carries ~ T^2 * u relative rounding; compare against |F| scale too
    tol = 1e-11
    err = np.abs(F - ref)
    assert np.all(err <= tol * (B + np.abs(ref)) + 1e-14), np.max(err)


# ---------------------------------------------------------------- P7: exact per-cell brute force (definition)

def test_P7_cell_brute_force_tiny():
    rng = np.random.default_rng(7)
    T = 12
    rects = []
    for _ in range(5):
        x0, y0 = rng.integers(0, T - 1, 2)
        rects.append((x0, y0, rng.integers(x0 + 1, T + 1), rng.integers(y0 + 1, T + 1)))
    rects = np.array(rects, np.int32)
    gp = np.array([0, 2, 5])                      # two union groups
    e = oracle.extract(rects, T, gp)
    img = _raster(rects, T, gp)
    ms, ns = oracle.window(15, 15)                # beyond T as well
    F, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], T, ms, ns)

    def cell_int(k, a):                           # int_a^{a+1} e^{-2 pi i k x / T} dx
        if k == 0:
            return 1.0
        return (np.exp(-2j * np.pi * k * (a + 1) / T) - np.exp(-2j * np.pi * k * a / T)) / (-2j * np.pi * k / T)

    ref = np.zeros(len(ms), complex)
    cells = np.argwhere(img != 0)
    for i, (m, n) in enumerate(zip(ms, ns)):
        s = 0
        for a, b in cells:
            s += img[a, b] * cell_int(m, a) * cell_int(n, b)
        ref[i] = s / (T * T)
    _check(F, ref, np.maximum(B, 1e-12), 1e-12, "cell brute force")


# ---------------------------------------------------------------- P8: midpoint quadrature converges as O(q^-2)

def test_P8_quadrature_convergence():
    T = 16
    rects = np.array([[2, 3, 9, 7], [5, 6, 12, 14], [0, 12, 3, 16]], np.int32)
    gp = np.array([0, 2, 3])
    e = oracle.extract(rects, T, gp)
    ms = np.array([1, 3, -2, 0, 5], np.int32)
    ns = np.array([2, -1, 0, 4, 5], np.int32)
    F, _ = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], T, ms, ns)
    img = _raster(rects, T, gp).astype(np.float64)
    errs = []
    for q in (4, 16, 64):
        u = (np.arange(T * q) + 0.5) / q                  # midpoints
        f = np.kron(img, np.ones((q, q)))                 # f at the midpoints
        ex = np.exp(-2j * np.pi * np.outer(ms, u) / T)    # [o, x]
        ey = np.exp(-2j * np.pi * np.outer(ns, u) / T)
        Q = np.einsum("ox,xy,oy->o", ex, f, ey) / (q * q) / (T * T)
        errs.append(np.max(np.abs(Q - F)))
    assert errs[2] < 1e-5
    assert errs[0] / errs[1] > 10 and errs[1] / errs[2] > 10      # ~16x per 4x refinement


# ---------------------------------------------------------------- P9: full tile is a delta

def test_P9_full_tile_delta():
    T = 128
    e = oracle.extract(np.array([[0, 0, T, T]], np.int32), T)
    assert e["K"] == 4 and e["area"][0] == T * T
    ms, ns, F, B = _window_coeffs(e["x"], e["y"], e["w"], e["area"][0], T, 10, 10)
    dc = (ms == 0) & (ns == 0)
    assert F[dc][0] == 1.0
    assert np.all(np.abs(F[~dc]) <= 1e-15 * B[~dc] + 1e-300)


# ---------------------------------------------------------------- P10: conservation

def test_P10_conservation():
    w = inputs.c2(seed=6, n_poly=500)
    e = oracle.extract(w.rects, w.T, w.group_ptr)
    x, y, wt = e["x"].astype(np.int64), e["y"].astype(np.int64), e["w"].astype(np.int64)
    assert wt.sum() == 0
    rng = np.random.default_rng(0)
    g = rng.integers(-1000, 1000, w.T + 1)
    h = rng.integers(-1000, 1000, w.T + 1)
    assert (wt * g[x]).sum() == 0 and (wt * h[y]).sum() == 0


# ---------------------------------------------------------------- P11: paper's edge-length form on vertex lists (Prop. 3)

_SHAPES = {
    # clockwise (y up) vertex lists starting with a horizontal edge (x_0 != x_1), Alg. 2 REQUIRE
    "square": [(0, 1), (1, 1), (1, 0), (0, 0)],
    "L": [(0, 2), (1, 2), (1, 1), (2, 1), (2, 0), (0, 0)],
    "U": [(0, 3), (1, 3), (1, 1), (2, 1), (2, 3), (3, 3), (3, 0), (0, 0)],
    "T": [(0, 3), (3, 3), (3, 2), (2, 2), (2, 0), (1, 0), (1, 2), (0, 2)],
}
# the same shapes as unions of unit-scaled rects (one union group each)
_SHAPE_RECTS = {
    "square": [(0, 0, 1, 1)],
    "L": [(0, 0, 2, 1), (0, 1, 1, 2)],
    "U": [(0, 0, 3, 1), (0, 1, 1, 3), (2, 1, 3, 3)],
    "T": [(0, 2, 3, 3), (1, 0, 2, 2)],
}


def _paper_alpha(k, l, Nx, Ny):
    if k == 0 and l == 0:
        return 1 / math.sqrt(Nx * Ny)
    if l == 0:
        return 1j / (2 * math.pi * k) * math.sqrt(Nx / Ny)
    if k == 0:
        return 1j / (2 * math.pi * l) * math.sqrt(Ny / Nx)
    return -math.sqrt(Nx * Ny) / (4 * math.pi ** 2 * k * l)


def _paper_prop3(V, k, l, T):
    """Eqs. Fdc, Fk0, F0l, Fkl with alpha, on a clockwise vertex list."""
    K = len(V)
    X = [v[0] for v in V]
    Y = [v[1] for v in V]
    wx = wy = 2 * math.pi / T
    s = 0
    for i in range(K // 2):
        a, b, c = 2 * i, (2 * i + 1) % K, (2 * i - 1) % K
        if k == 0 and l == 0:
            s += Y[a] * (X[b] - X[a])
        elif l == 0:
            s += (Y[c] - Y[a]) * np.exp(-1j * wx * k * X[a])
        elif k == 0:
            s += (X[b] - X[a]) * np.exp(-1j * wy * l * Y[a])
        else:
            s += np.exp(-1j * wy * l * Y[a]) * (np.exp(-1j * wx * k * X[b]) - np.exp(-1j * wx * k * X[a]))
    return _paper_alpha(k, l, T, T) * s


@pytest.mark.parametrize("shape", list(_SHAPES))
def test_P11_paper_edge_form_equals_T_times_corner_form(shape):
    rng = np.random.default_rng(hash(shape) % 1000)
    T = 256
    for _ in range(3):
        s = int(rng.integers(3, 40))
        ox, oy = rng.integers(0, T - 3 * s, 2)
        V = [(ox + s * a, oy + s * b) for a, b in _SHAPES[shape]]
        rects = np.array([(ox + s * a, oy + s * b, ox + s * c, oy + s * d) for a, b, c, d in _SHAPE_RECTS[shape]],
                         np.int32)
        e = oracle.extract(rects, T, np.array([0, len(rects)]))
        ms, ns = oracle.window(7, 7)
        F, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], T, ms, ns)
        ref = np.array([_paper_prop3(V, int(m), int(n), T) for m, n in zip(ms, ns)])
        _check(T * F, ref, T * B + 1e-300, 1e-13, f"Prop.3 {shape}")
        dc = (ms == 0) & (ns == 0)
        assert T * F[dc][0] == ref[dc][0].real


# ---------------------------------------------------------------- P12: hand values (golden fixture)

def test_P12_alpha_and_unit_square_hand_trace():
    g = json.load(open(GOLD))
    for a in g["alpha"]:
        assert abs(_paper_alpha(a["k"], a["l"], a["N"], a["N"]) - complex(a["re"], a["im"])) < 1e-15
    us = g["unit_square"]
    e = oracle.extract(np.array([us["rect"]], np.int32), 8)
    got = sorted(zip(e["x"].tolist(), e["y"].tolist(), e["w"].tolist()))
    assert got == sorted(tuple(c) for c in us["corners_xyw"])
    assert e["area"][0] == us["area"]
    # f_x[n] = sum_{x_k = n} w_k y_k and f_y[n] = sum_{y_k = n} w_k x_k (Steps 2-3)
    fx = {int(n): int(sum(wk * yk for xk, yk, wk in got if xk == n)) for n in (0, 1)}
    fy = {int(n): int(sum(wk * xk for xk, yk, wk in got if yk == n)) for n in (0, 1)}
    assert fx == {int(k): v for k, v in us["f_x"].items()}
    assert fy == {int(k): v for k, v in us["f_y"].items()}
    # the oracle's normalisation times T equals the paper's alpha * DFT (reading A1): alpha(2,3,4,4) example
    T = 4
    F, _ = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], T, np.array([2]), np.array([3]))
    Ex = lambda k, x: np.exp(-2j * np.pi * k * x / T)
    dft = (Ex(2, 1) - Ex(2, 0)) * (Ex(3, 1) - Ex(3, 0))      # f_xy DFT at (2,3), Step 4 P:890-904
    assert abs(T * F[0] - g["alpha"][2]["re"] * dft) < 1e-15


# ---------------------------------------------------------------- E1..E4: extraction

def _corners_from_raster(img):
    """w = mixed difference of the (zero-padded) cell raster: the corners of f."""
    T = img.shape[0]
    p = np.zeros((T + 2, T + 2), np.int64)
    p[1:T + 1, 1:T + 1] = img
    wgrid = p[1:, 1:] - p[:-1, 1:] - p[1:, :-1] + p[:-1, :-1]   # index (x, y) in [0, T]
    xs, ys = np.nonzero(wgrid)
    order = np.lexsort((xs, ys))
    return xs[order], ys[order], wgrid[xs, ys][order]


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_E1_extraction_matches_raster_corners(seed):
    rng = np.random.default_rng(seed)
    T = 96
    R = 40
    rects = inputs.random_rects(rng, R, T, 1, 40)
    cuts = np.sort(rng.choice(np.arange(1, R), 7, replace=False))
    gp = np.concatenate([[0], cuts, [R]]).astype(np.int64)
    e = oracle.extract(rects, T, gp)
    img = _raster(rects, T, gp)
    xs, ys, ws = _corners_from_raster(img)
    assert np.array_equal(e["x"], xs) and np.array_equal(e["y"], ys) and np.array_equal(e["w"], ws)
    assert e["area"][0] == img.sum()


def test_E2_batched_clips_and_order():
    w = inputs.c3(seed=0, clips=5, T=2048, n_lines=50)
    e = oracle.extract(w.rects, w.T, w.group_ptr, w.clip_ptr)
    for b in range(w.B):
        r0, r1 = w.clip_rect_range(b)
        eb = oracle.extract(w.rects[r0:r1], w.T)
        k0, k1 = e["corner_ptr"][b], e["corner_ptr"][b + 1]
        assert np.array_equal(e["x"][k0:k1], eb["x"]) and np.array_equal(e["w"][k0:k1], eb["w"])
        assert e["area"][b] == eb["area"][0]
        key = e["y"][k0:k1].astype(np.int64) * (w.T + 1) + e["x"][k0:k1]
        assert np.all(np.diff(key) > 0)                    # sorted by (y, x), unique


def test_E3_edge_cases():
    e = oracle.extract(np.zeros((0, 4), np.int32), 64, np.array([0, 0]))
    assert e["K"] == 0 and e["area"][0] == 0
    # pinch: two cells touching diagonally in one group -> |w| = 2
    e = oracle.extract(np.array([[0, 0, 1, 1], [1, 1, 2, 2]], np.int32), 4, np.array([0, 2]))
    assert sorted(zip(e["x"], e["y"], e["w"]))[1] == (1, 1, 2) or 2 in e["w"]
    # identical rects in two groups sum (weights 2), in one group union (weights 1)
    r = np.array([[1, 1, 3, 3], [1, 1, 3, 3]], np.int32)
    assert set(oracle.extract(r, 8)["w"].tolist()) == {2, -2}
    assert set(oracle.extract(r, 8, np.array([0, 2]))["w"].tolist()) == {1, -1}
    # corners on the tile boundary are kept at x = T (reading A7)
    e = oracle.extract(np.array([[5, 0, 8, 8]], np.int32), 8)
    assert 8 in e["x"].tolist() and 8 in e["y"].tolist()
    with pytest.raises(oracle.OracleError):
        oracle.extract(np.array([[3, 0, 3, 5]], np.int32), 8)          # x0 >= x1
    with pytest.raises(oracle.OracleError):
        oracle.extract(np.array([[3, 0, 9, 5]], np.int32), 8)          # x1 > T


def test_E4_window_and_pupil_counts():
    ms, ns = oracle.window(3, 2)
    assert len(ms) == 35 and ms[0] == -3 and ns[0] == -2 and ms[-1] == 3 and ns[-1] == 2
    r2 = inputs.pupil_r2(2048)
    ms, ns = oracle.window(27, 27, r2)
    g = np.arange(-27, 28)
    assert len(ms) == int(((g[:, None] ** 2 + g[None, :] ** 2) <= r2).sum()) == 2337
    assert inputs.window_count(27, 27, r2) == 2337


# ---------------------------------------------------------------- E5..E8: extraction from polygon vertex lists

def _raster_polygons(ps, b):
    """f[a, c] = sum over clip b's polygons of 1[cell centre (a+1/2, c+1/2) inside]: crossing parity of
    a ray towards +x against the polygon's vertical edges (point-in-polygon, not the corner rule)."""
    T = ps.T
    img = np.zeros((T, T), np.int64)
    cx = np.arange(T) + 0.5
    p0, p1 = (0, ps.P) if ps.clip_ptr is None else (ps.clip_ptr[b], ps.clip_ptr[b + 1])
    for p in range(p0, p1):
        a, e = ps.poly_ptr[p], ps.poly_ptr[p + 1]
        xs, ys = ps.vx[a:e].astype(np.int64), ps.vy[a:e].astype(np.int64)
        inside = np.zeros((T, T), bool)
        for i in range(len(xs)):
            j = (i + 1) % len(xs)
            if xs[i] == xs[j] and ys[i] != ys[j]:
                lo, hi = min(ys[i], ys[j]), max(ys[i], ys[j])
                inside ^= (xs[i] > cx)[:, None] & ((lo < cx) & (cx < hi))[None, :]
        img += inside
    return img


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_E5_polygon_extraction_matches_raster(seed):
    """Alg. 2 lines 9-10 on vertex lists == corners of the point-in-polygon raster, for
    skyline polygons in all 8 axis symmetries, both orientations, any start vertex, collinear
    vertices, overlapping polygons summed."""
    ps = inputs.polygon_clips(seed, clips=3, T=48, n_poly=6, max_cols=5, size=6, collinear=0.3)
    e = oracle.extract_polygons(ps.vx, ps.vy, ps.poly_ptr, ps.T, ps.clip_ptr)
    for b in range(ps.B):
        img = _raster_polygons(ps, b)
        xs, ys, ws = _corners_from_raster(img)
        k0, k1 = e["corner_ptr"][b], e["corner_ptr"][b + 1]
        assert np.array_equal(e["x"][k0:k1], xs) and np.array_equal(e["y"][k0:k1], ys)
        assert np.array_equal(e["w"][k0:k1], ws)
        assert e["area"][b] == img.sum()


@pytest.mark.parametrize("shape", list(_SHAPES))
def test_E6_polygons_equal_rect_unions(shape):
    """A polygon and the union of rects covering it have the same corners (Prop. 1),
    in every orientation / start vertex; rects given as 4-vertex polygons == rect extraction."""
    T = 64
    V = [(5 + 7 * a, 9 + 7 * c) for a, c in _SHAPES[shape]]
    rects = np.array([(5 + 7 * a, 9 + 7 * c, 5 + 7 * g, 9 + 7 * d) for a, c, g, d in _SHAPE_RECTS[shape]], np.int32)
    ref = oracle.extract(rects, T, np.array([0, len(rects)]))
    for rev in (False, True):
        for r in range(len(V)):
            u = V[::-1] if rev else V
            u = u[r:] + u[:r]
            vx = np.array([p[0] for p in u], np.int32)
            vy = np.array([p[1] for p in u], np.int32)
            e = oracle.extract_polygons(vx, vy, np.array([0, len(u)]), T)
            for k in ("x", "y", "w"):
                assert np.array_equal(e[k], ref[k]), (shape, rev, r, k)
            assert e["area"][0] == ref["area"][0]
    w = inputs.c3(seed=0, clips=3, T=2048, n_lines=40)
    ps = inputs.rects_as_polygons(w.rects, w.T, w.clip_ptr)
    e = oracle.extract_polygons(ps.vx, ps.vy, ps.poly_ptr, ps.T, ps.clip_ptr)
    ref = oracle.extract(w.rects, w.T, None, w.clip_ptr)
    for k in ("x", "y", "w", "corner_ptr", "area"):
        assert np.array_equal(e[k], ref[k]), k


def test_E7_polygon_edge_cases():
    T = 16
    ok = lambda vx, vy: oracle.extract_polygons(np.array(vx, np.int32), np.array(vy, np.int32),
                                                np.array([0, len(vx)]), T)
    # empty input; collinear vertex on every edge of the unit square is harmless
    e = oracle.extract_polygons(np.zeros(0, np.int32), np.zeros(0, np.int32), np.array([0]), T)
    assert e["K"] == 0 and e["area"][0] == 0
    e = ok([0, 1, 2, 2, 2, 1, 0, 0], [2, 2, 2, 1, 0, 0, 0, 1])
    assert e["area"][0] == 4 and e["K"] == 4
    # counter-clockwise list == clockwise list (reversed internally)
    a = ok([0, 3, 3, 0], [2, 2, 0, 0])
    b = ok([0, 0, 3, 3], [2, 0, 0, 2])
    assert all(np.array_equal(a[k], b[k]) for k in ("x", "y", "w")) and a["area"][0] == 6
    # vertices on the tile boundary (x = T) are kept (reading A7)
    e = ok([10, T, T, 10], [T, T, 3, 3])
    assert T in e["x"].tolist() and T in e["y"].tolist()
    # two overlapping copies are summed: weights +-2
    e = oracle.extract_polygons(np.array([0, 3, 3, 0] * 2, np.int32), np.array([2, 2, 0, 0] * 2, np.int32),
                                np.array([0, 4, 8]), T)
    assert set(e["w"].tolist()) == {2, -2} and e["area"][0] == 12
    for vx, vy in (([0, 3, 3, 0], [2, 2, 0, 1]),          # diagonal edge
                   ([0, 3, 3, 3, 0], [2, 2, 2, 0, 0]),    # zero-length edge
                   ([0, T + 1, T + 1, 0], [2, 2, 0, 0])):  # outside [0, T]
        with pytest.raises(oracle.OracleError):
            ok(vx, vy)


@pytest.mark.parametrize("shape", list(_SHAPES))
def test_E8_polygon_corners_give_paper_prop3(shape):
    """Coefficients of the corners extracted from the vertex list == the paper's edge-length
    Prop. 3 on the same list, x T (reading A1)."""
    rng = np.random.default_rng(7)
    T = 256
    s = int(rng.integers(3, 40))
    ox, oy = rng.integers(0, T - 3 * s, 2)
    V = [(int(ox + s * a), int(oy + s * c)) for a, c in _SHAPES[shape]]
    e = oracle.extract_polygons(np.array([p[0] for p in V], np.int32), np.array([p[1] for p in V], np.int32),
                                np.array([0, len(V)]), T)
    ms, ns = oracle.window(6, 6)
    F, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], T, ms, ns)
    ref = np.array([_paper_prop3(V, int(m), int(n), T) for m, n in zip(ms, ns)])
    _check(T * F, ref, T * B + 1e-300, 1e-13, f"Prop.3 polygon {shape}")


# ---------------------------------------------------------------- E9..E10: chopping a layout into tiles

def _layout_raster(rects, W, H):
    img = np.zeros((W, H), np.int64)
    for x0, y0, x1, y1 in rects:
        img[x0:x1, y0:y1] += 1
    return img


@pytest.mark.parametrize("seed", [0, 1])
def test_E9_chop_reassembles_the_layout_raster(seed):
    """Pieces are non-empty, inside [0,T]^2, and the tiles' rasters placed at their offsets reproduce
    the raster of the whole layout (each rect its own group: rasters add)."""
    rng = np.random.default_rng(seed)
    T, tx, ty = 16, 5, 3
    W, H = T * tx, T * ty
    x0 = rng.integers(0, W - 1, 60); y0 = rng.integers(0, H - 1, 60)
    x1 = np.minimum(x0 + rng.integers(1, 40, 60), W); y1 = np.minimum(y0 + rng.integers(1, 30, 60), H)
    rects = np.stack([x0, y0, x1, y1], 1).astype(np.int32)
    rects[0] = (0, 0, W, H)                               # spans every tile
    rects[1] = (T - 1, T - 1, T + 1, T + 1)               # a 2x2 piece at a tile corner
    ch = oracle.chop_rects(rects, T, tx, ty)
    p = ch["rects"]
    assert np.all(p[:, 0] >= 0) and np.all(p[:, 2] <= T) and np.all(p[:, 0] < p[:, 2]) and np.all(p[:, 1] < p[:, 3])
    full = _layout_raster(rects, W, H)
    re = np.zeros_like(full)
    for t in range(tx * ty):
        a, b = ch["tile_ptr"][t], ch["tile_ptr"][t + 1]
        ox, oy = (t % tx) * T, (t // tx) * T
        re[ox:ox + T, oy:oy + T] = _layout_raster(p[a:b], T, T)
    assert np.array_equal(re, full)
    assert ch["tile_ptr"][-1] == ch["n"]


def test_E10_tile_coefficients_from_chopped_pieces_match_the_cropped_raster():
    """F of one tile from its chopped pieces (extraction + coefficients) == the exact raster identity (P6)
    on the layout raster cropped to the tile."""
    lay = inputs.layout(seed=3, T=64, tiles_x=3, tiles_y=2, lines_per_tile=40)
    ch = oracle.chop_rects(lay.rects, lay.T, lay.tiles_x, lay.tiles_y)
    full = _layout_raster(lay.rects, lay.T * lay.tiles_x, lay.T * lay.tiles_y)
    T = lay.T
    for t in (0, 4):
        a, b = ch["tile_ptr"][t], ch["tile_ptr"][t + 1]
        e = oracle.extract(ch["rects"][a:b], T)
        ms, ns = oracle.window(6, 6)
        F, B = oracle.coeffs(e["x"], e["y"], e["w"], e["area"][0], T, ms, ns)
        ox, oy = (t % lay.tiles_x) * T, (t // lay.tiles_x) * T
        img = full[ox:ox + T, oy:oy + T].astype(np.float64)
        D = np.fft.fft2(img)
        ref = D[ms % T, ns % T] * _cell_transfer(ms, T) * _cell_transfer(ns, T) / (T * T)
        _check(F, ref, B + 1e-300, 1e-12, f"tile {t}")


# ---------------------------------------------------------------- H1..H4: continuous Haar transform (NEXT-4)

def _dht(img):
    """Orthonormal 2D (nonstandard) Haar filter bank on the unit-cell raster img[x, y]: the scaling
    coefficients of unit cells are the raster values (2^J / T = 1), then X_j = (sum of 4 children) / 2
    and the three details with h = (1, -1) / sqrt2, g = (1, 1) / sqrt2.  Output out[y, x]."""
    T = img.shape[0]
    out = np.zeros((T, T))
    X = img.astype(np.float64)
    n = T // 2
    while n >= 1:
        a, b, c, d = X[0::2, 0::2], X[0::2, 1::2], X[1::2, 0::2], X[1::2, 1::2]   # (n, m) = (0,0) (0,1) (1,0) (1,1)
        out[0:n, n:2 * n] = ((a + b - c - d) / 2).T    # hg: h along x
        out[n:2 * n, 0:n] = ((a - b + c - d) / 2).T    # gh
        out[n:2 * n, n:2 * n] = ((a - b - c + d) / 2).T
        X = (a + b + c + d) / 2
        n //= 2
    out[0, 0] = X[0, 0]
    return out


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_H1_haar_equals_the_discrete_haar_of_the_raster(seed):
    """CHT == DHT for rectilinear patterns on the unit lattice: the oracle (child-cell areas
    of the corner form) against the filter-bank FWT of the raster, exactly (dyadic values)."""
    rng = np.random.default_rng(seed)
    T = 32
    rects = inputs.random_rects(rng, 12, T, 1, 14)
    gp = np.array([0, 5, 12], np.int64)                 # two union groups, summed (overlaps give f = 2)
    e = oracle.extract(rects, T, gp)
    H = oracle.haar(e["x"], e["y"], e["w"], T)
    assert np.array_equal(H, _dht(_raster(rects, T, gp)))


def test_H2_parseval_and_dc():
    rng = np.random.default_rng(4)
    T = 64
    rects = inputs.random_rects(rng, 20, T, 2, 30)
    e = oracle.extract(rects, T)
    H = oracle.haar(e["x"], e["y"], e["w"], T)
    img = _raster(rects, T)
    assert H[0, 0] == e["area"][0] / T
    assert abs((H ** 2).sum() - (img.astype(np.float64) ** 2).sum()) <= 1e-9 * (img ** 2).sum()


def test_H3_hh_details_are_local_to_corners():
    """psi^(hh) of a cell is non-zero only if a corner lies strictly inside the cell (the h factor is a
    tent supported inside the cell along each axis)."""
    rng = np.random.default_rng(5)
    T = 32
    rects = inputs.random_rects(rng, 6, T, 2, 12)
    e = oracle.extract(rects, T)
    H = oracle.haar(e["x"], e["y"], e["w"], T)
    n = 1
    while n < T:
        s = T // n
        for ky in range(n):
            for kx in range(n):
                inside = np.any((e["x"] > kx * s) & (e["x"] < (kx + 1) * s) & (e["y"] > ky * s) & (e["y"] < (ky + 1) * s))
                if not inside:
                    assert H[n + ky, n + kx] == 0
        n *= 2


def test_H4_single_rect_hand_values():
    """[1,5) x [2,7) in T = 8: DC = 20/8; level 0 hg = (A00 + A01 - A10 - A11) / 8 with the 4x4 quadrant
    areas A00 = 3*2, A01 = 3*3, A10 = 1*2, A11 = 1*3 -> (6 + 9 - 2 - 3) / 8 = 1.25 (hand computation)."""
    e = oracle.extract(np.array([[1, 2, 5, 7]], np.int32), 8)
    H = oracle.haar(e["x"], e["y"], e["w"], 8)
    assert H[0, 0] == 2.5 and H[0, 1] == 1.25
    assert H[1, 0] == (6 - 9 + 2 - 3) / 8 and H[1, 1] == (6 - 9 - 2 + 3) / 8


# ---------------------------------------------------------------- B1-B4: the L1 bound B[m,n] = sum_k |term_k|
# B is the tolerance scale of every GPU parity assertion (1e-12 B / 1e-5 B), so it is pinned to values
# derived by hand from the Prop. 3 terms (reading A12), not to the oracle's own formula.
# Each term of Eq. Fkl is w_k E_x E_y / (-4 pi^2 m n) with |E| = 1, each term of Eq. Fk0 is
# i w_k y_k E_x / (2 pi m T), each of Eq. F0l i w_k x_k E_y / (2 pi n T); F[0,0] is compared exactly.

def test_B1_single_rect_hand_values():
    """[3,10) x [5,20), T = 32: corners (3,5,+1) (10,5,-1) (3,20,-1) (10,20,+1) written out by hand.
    Interior B = 4 / (4 pi^2 |m n|); n = 0: sum |w y| = 5+5+20+20 = 50 -> 50 / (2 pi |m| T);
    m = 0: sum |w x| = 3+10+3+10 = 26 -> 26 / (2 pi |n| T); B[0,0] = 0."""
    T = 32
    x = np.array([3, 10, 3, 10], np.int32)
    y = np.array([5, 5, 20, 20], np.int32)
    w = np.array([1, -1, -1, 1], np.int32)
    ms = np.array([1, -1, 3, 7, -5, 2, -9, 0, 0, 0, 4, -31], np.int32)
    ns = np.array([1, 2, -3, 5, -6, 0, 0, 4, -11, 0, 33, 1], np.int32)
    _, B = oracle.coeffs(x, y, w, 7 * 15, T, ms, ns)
    pi = math.pi
    for i, (m, n) in enumerate(zip(ms.tolist(), ns.tolist())):
        if m == 0 and n == 0:
            want = 0.0
        elif n == 0:
            want = 50.0 / (2 * pi * abs(m) * T)
        elif m == 0:
            want = 26.0 / (2 * pi * abs(n) * T)
        else:
            want = 4.0 / (4 * pi * pi * abs(m * n))
        assert B[i] == pytest.approx(want, rel=1e-14, abs=0.0), (m, n, B[i], want)


def test_B2_weights_beyond_one_hand_values():
    """A hand corner list with |w| = 2 and 3 (pinch points / summed groups, reading A6), T = 16:
    (1,1,+2) (4,1,-1) (2,3,-3) (7,7,+2).  sum |w| = 8; sum |w y| = 2+1+9+14 = 26; sum |w x| = 2+4+6+14 = 26."""
    T = 16
    x = np.array([1, 4, 2, 7], np.int32)
    y = np.array([1, 1, 3, 7], np.int32)
    w = np.array([2, -1, -3, 2], np.int32)
    ms = np.array([1, 2, -3, 5, 0, 6], np.int32)
    ns = np.array([1, -4, 0, 0, 3, -7], np.int32)
    _, B = oracle.coeffs(x, y, w, 0, T, ms, ns)
    pi = math.pi
    want = [8 / (4 * pi * pi * 1), 8 / (4 * pi * pi * 8), 26 / (2 * pi * 3 * T), 26 / (2 * pi * 5 * T),
            26 / (2 * pi * 3 * T), 8 / (4 * pi * pi * 42)]
    assert np.allclose(B, want, rtol=1e-14, atol=0.0)


@pytest.mark.parametrize("corner", [(0, 0, 1), (5, 9, -1), (13, 2, 3), (31, 31, -2)])
def test_B3_single_corner_bound_is_attained(corner):
    """One term: |F[m,n]| equals B[m,n] exactly (|E| = 1), so a B scaled by any constant != 1 fails.
    Axis entries need a non-zero coordinate weight (x, y > 0) to be non-trivial."""
    T = 32
    x = np.array([corner[0]], np.int32)
    y = np.array([corner[1]], np.int32)
    w = np.array([corner[2]], np.int32)
    ms, ns = oracle.window(9, 7)
    F, B = oracle.coeffs(x, y, w, 0, T, ms, ns)
    nz = ~((ms == 0) & (ns == 0))
    assert np.allclose(np.abs(F[nz]), B[nz], rtol=1e-14, atol=1e-300)


@pytest.mark.parametrize("cfg", ["c1", "c2s"])
def test_B4_triangle_inequality(cfg):
    """|F[m,n]| <= B[m,n] at every window entry (triangle inequality over the terms), and B > 0 off DC
    for a clip whose corner weights do not all vanish."""
    wl = inputs.c1(seed=2) if cfg == "c1" else inputs.c2(seed=5, n_poly=80)
    e = oracle.extract(wl.rects, wl.T, wl.group_ptr)
    ms, ns, F, B = _window_coeffs(e["x"], e["y"], e["w"], e["area"][0], wl.T, 24, 20)
    nz = ~((ms == 0) & (ns == 0))
    assert np.all(np.abs(F[nz]) <= B[nz] * (1 + 1e-12))
    assert np.all(B[nz] > 0)
