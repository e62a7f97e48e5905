"""CPU oracle for the FCFS hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1010_5562_b200`` never imports it, and it never imports the product
package: the two share no code (the seeded generators in
``paper_1010_5562_b200/inputs.py`` hold no FCFS arithmetic and are the only
common module).

The arithmetic lives in ``fcfs_oracle.c`` (plain C, ``long double``,
Neumaier sums, one exact integer phase + one table lookup per term); see its
header for the PAPER.md passages each function follows.  Every function is
pinned by ``tests/test_oracle_pins.py`` (pins P1..P12 of DESIGN.md).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fcfs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_E_INVALID, OR_E_RANGE, OR_E_CAPACITY, OR_E_SELFCHECK, OR_E_NOMEM = 0, 1, 2, 3, 7, 8


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (-O2 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        lib.oracle_extract.argtypes = [P, i64, P, i64, P, i64, i32, P, P, P, i64, P, P, P]
        lib.oracle_extract.restype = ctypes.c_int
        lib.oracle_extract_polygons.argtypes = [P, P, P, i64, P, i64, i32, P, P, P, i64, P, P, P]
        lib.oracle_extract_polygons.restype = ctypes.c_int
        lib.oracle_chop_rects.argtypes = [P, i64, i32, i32, i32, P, i64, P, P]
        lib.oracle_chop_rects.restype = ctypes.c_int
        lib.oracle_haar.argtypes = [P, P, P, i64, i32, P]
        lib.oracle_haar.restype = ctypes.c_int
        lib.oracle_coeffs.argtypes = [P, P, P, i64, i64, i32, P, P, i64, P, P, P, ctypes.c_int]
        lib.oracle_coeffs.restype = ctypes.c_int
        lib.oracle_window.argtypes = [i32, i32, ctypes.c_double, P, P, i64]
        lib.oracle_window.restype = i64
        lib.oracle_max_threads.argtypes = []
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    pass


def extract(rects, T, group_ptr=None, clip_ptr=None):
    """Signed corners of f = sum_groups 1[union of group] per clip.

    rects: int32 [R,4] (x0,y0,x1,y1).  group_ptr: int64 [G+1] or None (each rect
    its own group).  clip_ptr: int64 [B+1] over groups or None (one clip).
    Returns dict(x, y, w (int32), corner_ptr (int64 [B+1]), area (int64 [B]), K).
    """
    lib = _load()
    rects = np.ascontiguousarray(rects, dtype=np.int32).reshape(-1, 4)
    R = rects.shape[0]
    if group_ptr is not None:
        group_ptr = np.ascontiguousarray(group_ptr, dtype=np.int64)
        G = group_ptr.shape[0] - 1
    else:
        G = R
    if clip_ptr is not None:
        clip_ptr = np.ascontiguousarray(clip_ptr, dtype=np.int64)
        B = clip_ptr.shape[0] - 1
    else:
        B = 1
    cptr = np.zeros(B + 1, np.int64)
    area = np.zeros(B, np.int64)
    K = ctypes.c_int64(0)
    cap = 0
    rc = lib.oracle_extract(_ptr(rects), R, _ptr(group_ptr), G, _ptr(clip_ptr), B, int(T),
                            None, None, None, 0, _ptr(cptr), _ptr(area), ctypes.byref(K))
    if rc not in (OR_OK, OR_E_CAPACITY):
        raise OracleError(f"oracle_extract failed rc={rc}")
    cap = K.value
    x = np.zeros(max(cap, 1), np.int32)
    y = np.zeros(max(cap, 1), np.int32)
    w = np.zeros(max(cap, 1), np.int32)
    rc = lib.oracle_extract(_ptr(rects), R, _ptr(group_ptr), G, _ptr(clip_ptr), B, int(T),
                            _ptr(x), _ptr(y), _ptr(w), cap, _ptr(cptr), _ptr(area), ctypes.byref(K))
    if rc != OR_OK:
        raise OracleError(f"oracle_extract failed rc={rc}")
    return dict(x=x[:cap], y=y[:cap], w=w[:cap], corner_ptr=cptr, area=area, K=cap)


def extract_polygons(vx, vy, poly_ptr, T, clip_ptr=None):
    """Signed corners of f = sum of the polygons' indicators per clip (Alg. 2 on vertex lists).

    vx, vy: int32 [V] vertices; poly_ptr: int64 [P+1] CSR over vertices (closed polygons, either
    orientation); clip_ptr: int64 [B+1] over polygons or None (one clip).
    Returns dict(x, y, w (int32), corner_ptr (int64 [B+1]), area (int64 [B]), K).
    """
    lib = _load()
    vx = np.ascontiguousarray(vx, dtype=np.int32)
    vy = np.ascontiguousarray(vy, dtype=np.int32)
    poly_ptr = np.ascontiguousarray(poly_ptr, dtype=np.int64)
    P = poly_ptr.shape[0] - 1
    if clip_ptr is not None:
        clip_ptr = np.ascontiguousarray(clip_ptr, dtype=np.int64)
        B = clip_ptr.shape[0] - 1
    else:
        B = 1
    cptr = np.zeros(B + 1, np.int64)
    area = np.zeros(B, np.int64)
    K = ctypes.c_int64(0)
    args = (_ptr(vx), _ptr(vy), _ptr(poly_ptr), P, _ptr(clip_ptr), B, int(T))
    rc = lib.oracle_extract_polygons(*args, None, None, None, 0, _ptr(cptr), _ptr(area), ctypes.byref(K))
    if rc not in (OR_OK, OR_E_CAPACITY):
        raise OracleError(f"oracle_extract_polygons failed rc={rc}")
    cap = K.value
    x = np.zeros(max(cap, 1), np.int32)
    y = np.zeros(max(cap, 1), np.int32)
    w = np.zeros(max(cap, 1), np.int32)
    rc = lib.oracle_extract_polygons(*args, _ptr(x), _ptr(y), _ptr(w), cap, _ptr(cptr), _ptr(area), ctypes.byref(K))
    if rc != OR_OK:
        raise OracleError(f"oracle_extract_polygons failed rc={rc}")
    return dict(x=x[:cap], y=y[:cap], w=w[:cap], corner_ptr=cptr, area=area, K=cap)


def chop_rects(rects, T, tiles_x, tiles_y):
    """Rects (layout coordinates) chopped into T x T tiles: dict(rects (int32 [n,4], tile-local),
    tile_ptr (int64 [tiles+1], row-major tiles), n)."""
    lib = _load()
    rects = np.ascontiguousarray(rects, dtype=np.int32).reshape(-1, 4)
    nt = int(tiles_x) * int(tiles_y)
    tp = np.zeros(nt + 1, np.int64)
    n = ctypes.c_int64(0)
    rc = lib.oracle_chop_rects(_ptr(rects), rects.shape[0], int(T), int(tiles_x), int(tiles_y), None, 0, _ptr(tp),
                               ctypes.byref(n))
    if rc not in (OR_OK, OR_E_CAPACITY):
        raise OracleError(f"oracle_chop_rects failed rc={rc}")
    out = np.zeros((max(n.value, 1), 4), np.int32)
    rc = lib.oracle_chop_rects(_ptr(rects), rects.shape[0], int(T), int(tiles_x), int(tiles_y), _ptr(out), n.value,
                               _ptr(tp), ctypes.byref(n))
    if rc != OR_OK:
        raise OracleError(f"oracle_chop_rects failed rc={rc}")
    return dict(rects=out[:n.value], tile_ptr=tp, n=n.value)


def haar(x, y, w, T):
    """Continuous Haar transform of one clip's corners: float64 [T, T] in the layout of reading A18."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.int32)
    y = np.ascontiguousarray(y, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.int32)
    out = np.zeros((int(T), int(T)), np.float64)
    rc = lib.oracle_haar(_ptr(x), _ptr(y), _ptr(w), x.shape[0], int(T), _ptr(out))
    if rc != OR_OK:
        raise OracleError(f"oracle_haar failed rc={rc}")
    return out


def window(M, N, r2=-1.0):
    """(ms, ns) in the output order: m-major, then n; pupil m^2+n^2 <= r2 if r2 >= 0."""
    lib = _load()
    cnt = lib.oracle_window(int(M), int(N), float(r2), None, None, 0)
    ms = np.zeros(cnt, np.int32)
    ns = np.zeros(cnt, np.int32)
    lib.oracle_window(int(M), int(N), float(r2), _ptr(ms), _ptr(ns), cnt)
    return ms, ns


def coeffs(x, y, w, area, T, ms, ns, nthreads=0):
    """F[m,n] (complex128) and the L1 bound B[m,n] at each listed signed (m, n)."""
    lib = _load()
    x = np.ascontiguousarray(x, dtype=np.int32)
    y = np.ascontiguousarray(y, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.int32)
    ms = np.ascontiguousarray(ms, dtype=np.int32)
    ns = np.ascontiguousarray(ns, dtype=np.int32)
    n = ms.shape[0]
    re = np.zeros(n, np.float64)
    im = np.zeros(n, np.float64)
    bd = np.zeros(n, np.float64)
    rc = lib.oracle_coeffs(_ptr(x), _ptr(y), _ptr(w), x.shape[0], int(area), int(T),
                           _ptr(ms), _ptr(ns), n, _ptr(re), _ptr(im), _ptr(bd), int(nthreads))
    if rc != OR_OK:
        raise OracleError(f"oracle_coeffs failed rc={rc}")
    return re + 1j * im, bd


def max_threads() -> int:
    return int(_load().oracle_max_threads())
