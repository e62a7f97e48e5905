"""ctypes binding of libfcfs.so (include/fcfs.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only
allocates torch tensors (device memory, workspaces), passes raw pointers and the
current CUDA stream, and raises ``FcfsError`` on a non-OK status.  There is no CPU
fallback: importing this module fails loudly if ``libfcfs.so`` is missing.

Names follow the C-ABI: ``vertices_from_rects`` (a1), ``coeffs`` (a2-a5, one clip,
optional shard), ``coeffs_batched`` (many clips), ``pupil_indices``, ``window_size``.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FCFS_LIBRARY (tests only) selects another build of the same ABI, e.g. libfcfs_checked.so (the
# device-side invariant checks of tools/checked_run.sh); the default is the in-tree libfcfs.so.
LIB_PATH = os.environ.get("FCFS_LIBRARY") or os.path.join(_HERE, "libfcfs.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{os.path.basename(LIB_PATH)} not found at {LIB_PATH}: build it with "
                      "`python -m paper_1010_5562_b200.build` (no CPU fallback exists)")

_lib = ctypes.CDLL(LIB_PATH)

FCFS_OK, E_INVALID, E_RANGE, E_CAPACITY, E_WORKSPACE, E_UNSUPPORTED, E_CUDA = range(7)
FP64, TF32X3, F16X3 = 0, 1, 2
LAYOUT_DENSE, LAYOUT_PUPIL = 0, 1
SHARD_NONE, SHARD_ROWS, SHARD_VERTEX_BLOCK = 0, 1, 2
ROUTE_AUTO, ROUTE_GEMM, ROUTE_FFT = 0, 1, 2
FORM_AUTO, FORM_EDGE, FORM_CORNER, FORM_LATTICE = 0, 1, 2, 3
_ROUTE = {"auto": ROUTE_AUTO, "gemm": ROUTE_GEMM, "fft": ROUTE_FFT, None: ROUTE_AUTO,
          ROUTE_AUTO: ROUTE_AUTO, ROUTE_GEMM: ROUTE_GEMM, ROUTE_FFT: ROUTE_FFT}
_FORM = {"auto": FORM_AUTO, "edge": FORM_EDGE, "corner": FORM_CORNER, "lattice": FORM_LATTICE, None: FORM_AUTO,
         FORM_AUTO: FORM_AUTO, FORM_EDGE: FORM_EDGE, FORM_CORNER: FORM_CORNER, FORM_LATTICE: FORM_LATTICE}
_PREC = {"fp64": FP64, "tf32x3": TF32X3, "f16x3": F16X3, FP64: FP64, TF32X3: TF32X3, F16X3: F16X3}
_LAYOUT = {"dense": LAYOUT_DENSE, "pupil": LAYOUT_PUPIL, LAYOUT_DENSE: LAYOUT_DENSE, LAYOUT_PUPIL: LAYOUT_PUPIL}


class Window(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int32), ("N", ctypes.c_int32), ("pupil_r2", ctypes.c_double),
                ("layout", ctypes.c_int32)]


class Shard(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("m_lo", ctypes.c_int32), ("m_hi", ctypes.c_int32),
                ("k_lo", ctypes.c_int64), ("k_hi", ctypes.c_int64)]


class Options(ctypes.Structure):
    _fields_ = [("route", ctypes.c_int32), ("form", ctypes.c_int32), ("sorted_y", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 5)]


def make_options(route=None, form=None, sorted_y=False):
    """fcfs_options: route "auto" | "gemm" | "fft" (fcfs_coeffs), form "auto" | "edge" | "corner" | "lattice"
    (fcfs_coeffs_batched, split precisions), sorted_y: the caller guarantees y-sorted clips (as
    fcfs_vertices_from_* emit them; skips the lattice form's device check and its stream sync)."""
    return Options(_ROUTE[route], _FORM[form], 1 if sorted_y else 0)


_P, _i64, _i32, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
_WP, _SP, _OP = ctypes.POINTER(Window), ctypes.POINTER(Shard), ctypes.POINTER(Options)

_lib.fcfs_status_string.argtypes = [_i32]
_lib.fcfs_status_string.restype = ctypes.c_char_p
_lib.fcfs_last_error.argtypes = []
_lib.fcfs_last_error.restype = ctypes.c_char_p
_lib.fcfs_device_check.argtypes = []
_lib.fcfs_device_check.restype = _i32
_lib.fcfs_kernel_launches.argtypes = []
_lib.fcfs_kernel_launches.restype = _i32
_lib.fcfs_window_size.argtypes = [_WP]
_lib.fcfs_window_size.restype = _i64
_lib.fcfs_pupil_indices.argtypes = [_i32, _i32, ctypes.c_double, _P, _P, _i64]
_lib.fcfs_pupil_indices.restype = _i64
_lib.fcfs_vertices_workspace_bytes.argtypes = [_i64, _i64, _i64, _i64]
_lib.fcfs_vertices_workspace_bytes.restype = _sz
_lib.fcfs_vertices_from_rects.argtypes = [_P, _i64, _P, _i64, _P, _i64, _i32, _i64, _P, _P, _P, _i64, _P, _P,
                                          ctypes.POINTER(_i64), _P, _sz, _P]
_lib.fcfs_vertices_from_rects.restype = _i32
_lib.fcfs_vertices_from_rects_edges.argtypes = [_P, _i64, _P, _i64, _P, _i64, _i32, _i64, _P, _P, _P, _i64, _P, _P,
                                                ctypes.POINTER(_i64), _P, _P, _P, _P, _P, _P, _sz, _P]
_lib.fcfs_vertices_from_rects_edges.restype = _i32
_lib.fcfs_vertices_from_rects_band.argtypes = [_P, _i64, _P, _i64, _i32, _i64, _i32, _i32, _P, _P, _P, _i64, _P,
                                               _P, ctypes.POINTER(_i64), _P, _sz, _P]
_lib.fcfs_vertices_from_rects_band.restype = _i32
_lib.fcfs_polygons_workspace_bytes.argtypes = [_i64, _i64, _i64]
_lib.fcfs_polygons_workspace_bytes.restype = _sz
_lib.fcfs_vertices_from_polygons.argtypes = [_P, _P, _i64, _P, _i64, _P, _i64, _i32, _P, _P, _P, _i64, _P, _P,
                                             ctypes.POINTER(_i64), _P, _sz, _P]
_lib.fcfs_vertices_from_polygons.restype = _i32
_lib.fcfs_coeffs_workspace_bytes.argtypes = [_i64, _i32, _WP, _i32, _SP, _OP]
_lib.fcfs_coeffs_workspace_bytes.restype = _sz
_lib.fcfs_haar_workspace_bytes.argtypes = [_i64, _i32]
_lib.fcfs_haar_workspace_bytes.restype = _sz
_lib.fcfs_haar.argtypes = [_P, _i64, _i64, _P, _P, _P, _P, _i32, _P, _P, _sz, _P]
_lib.fcfs_haar.restype = _i32
_lib.fcfs_chop_workspace_bytes.argtypes = [_i64, _i64, _i32, _i32]
_lib.fcfs_chop_workspace_bytes.restype = _sz
_lib.fcfs_chop_rects.argtypes = [_P, _i64, _i32, _i32, _i32, _P, _i64, _P, ctypes.POINTER(_i64), _P, _sz, _P]
_lib.fcfs_chop_rects.restype = _i32
_lib.fcfs_coeffs_route.argtypes = [_i64, _i32, _WP, _i32, _SP, _OP]
_lib.fcfs_coeffs_route.restype = _i32
_lib.fcfs_coeffs.argtypes = [_P, _P, _P, _i64, _i64, _i32, _WP, _i32, _SP, _OP, _P, _P, _sz, _P]
_lib.fcfs_coeffs.restype = _i32
_lib.fcfs_coeffs_rows_to_peers.argtypes = [_P, _P, _P, _i64, _i64, _i32, _WP, _i32, _SP, _OP,
                                           ctypes.POINTER(ctypes.c_void_p), _i32, _P, _sz, _P]
_lib.fcfs_coeffs_rows_to_peers.restype = _i32
_lib.fcfs_batched_workspace_bytes.argtypes = [_i64, _i64, _i64, _i32, _WP, _i32, _OP]
_lib.fcfs_batched_workspace_bytes.restype = _sz
_lib.fcfs_coeffs_batched_form.argtypes = [_i64, _i64, _i64, _i32, _WP, _i32, _OP]
_lib.fcfs_coeffs_batched_form.restype = _i32
_lib.fcfs_coeffs_batched.argtypes = [_P, _i64, _i64, _i64, _P, _P, _P, _P, _i32, _WP, _i32, _OP, _P, _P, _sz, _P]
_lib.fcfs_coeffs_batched_edges.argtypes = [_P, _i64, _i64, _i64, _P, _P, _P, _P, _P, _P, _P, _P, _P, _i32, _WP,
                                           _i32, _OP, _P, _P, _sz, _P]
_lib.fcfs_coeffs_batched_edges.restype = _i32
_lib.fcfs_coeffs_batched.restype = _i32

_lib.fcfs_row_buckets_workspace_bytes.argtypes = [_i64, _i64]
_lib.fcfs_row_buckets_workspace_bytes.restype = _sz
_lib.fcfs_row_buckets.argtypes = [_P, _P, _i64, _i64, _i32, _P, _P, _P, ctypes.POINTER(_i64), _P, _sz, _P]
_lib.fcfs_row_buckets.restype = _i32

_lib.fcfs_vertices_from_rects_async.argtypes = [_P, _i64, _P, _i64, _P, _i64, _i32, _i64, _P, _P, _P, _i64, _P, _P, _P,
                                                _P, _P, _sz, _P]
_lib.fcfs_vertices_from_rects_async.restype = _i32
_lib.fcfs_coeffs_async.argtypes = [_P, _P, _P, _P, _i64, _P, _i32, _WP, _i32, _P, _P, _P, _sz, _P]
_lib.fcfs_vertices_from_clips_async.argtypes = [_P, _i64, _P, _i64, _i32, _i64, _P, _P, _P, _i64, _P, _P, _P, _P, _P,
                                                _sz, _P]
_lib.fcfs_vertices_from_clips_async.restype = _i32
_lib.fcfs_coeffs_async.restype = _i32
_lib.fcfs_small_clip_supported.argtypes = [_i64, _i64, _i32, _i64, _WP]
_lib.fcfs_small_clip_supported.restype = _i32
_lib.fcfs_small_clip.argtypes = [_P, _i64, _P, _i64, _i32, _i64, _WP, _i32, _P, _P, _P, _P]
_lib.fcfs_small_clip.restype = _i32

_lib.fcfs_profile_enable.argtypes = [_i32]
_lib.fcfs_profile_enable.restype = _i32
_lib.fcfs_profile_read.argtypes = [_P, _P, _i32]
_lib.fcfs_profile_read.restype = _i32
_lib.fcfs_edges.argtypes = [_P, _P, _P, _P, _i64, _P, _P, _P, _P, _P, _P]
_lib.fcfs_edges.restype = _i32

EXPORTED = ["fcfs_vertices_workspace_bytes", "fcfs_vertices_from_rects", "fcfs_coeffs_workspace_bytes",
            "fcfs_coeffs", "fcfs_batched_workspace_bytes", "fcfs_coeffs_batched", "fcfs_window_size",
            "fcfs_pupil_indices", "fcfs_status_string", "fcfs_last_error", "fcfs_device_check",
            "fcfs_kernel_launches", "fcfs_profile_enable", "fcfs_profile_read", "fcfs_row_buckets_workspace_bytes",
            "fcfs_row_buckets", "fcfs_polygons_workspace_bytes", "fcfs_vertices_from_polygons",
            "fcfs_coeffs_route", "fcfs_chop_workspace_bytes", "fcfs_chop_rects",
            "fcfs_haar_workspace_bytes", "fcfs_haar", "fcfs_edges", "fcfs_vertices_from_rects_edges",
            "fcfs_coeffs_batched_edges", "fcfs_coeffs_batched_form", "fcfs_vertices_from_rects_band",
            "fcfs_small_clip_supported", "fcfs_small_clip", "fcfs_vertices_from_rects_async",
            "fcfs_coeffs_async", "fcfs_coeffs_rows_to_peers", "fcfs_vertices_from_clips_async"]
STAGES = ("extract", "contract", "epilogue", "pairing")


class FcfsError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        name = _lib.fcfs_status_string(status).decode()
        detail = _lib.fcfs_last_error().decode()
        super().__init__(f"{where}: {name}: {detail}")


def _check(st, where):
    if st != FCFS_OK:
        raise FcfsError(st, where)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _ws(nbytes, device):
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def make_window(M, N, r2=-1.0, layout="dense"):
    return Window(int(M), int(N), float(r2), _LAYOUT[layout])


def window_size(M, N, r2=-1.0, layout="dense"):
    w = make_window(M, N, r2, layout)
    n = _lib.fcfs_window_size(ctypes.byref(w))
    if n < 0:
        raise FcfsError(E_INVALID, "window_size")
    return int(n)


def pupil_indices(M, N, r2):
    """(ms, ns) int32 host tensors of the packed pupil order (m-major, then n)."""
    cnt = _lib.fcfs_pupil_indices(int(M), int(N), float(r2), None, None, 0)
    ms = torch.zeros(cnt, dtype=torch.int32)
    ns = torch.zeros(cnt, dtype=torch.int32)
    _lib.fcfs_pupil_indices(int(M), int(N), float(r2), _ptr(ms), _ptr(ns), cnt)
    return ms, ns


def device_check():
    _check(_lib.fcfs_device_check(), "device_check")


def kernel_launches() -> int:
    return int(_lib.fcfs_kernel_launches())


def profile_enable(on=True):
    _check(_lib.fcfs_profile_enable(1 if on else 0), "fcfs_profile_enable")


def profile_read():
    """{stage: (ms_total, launches)} of the CUDA-event-timed stages since the last read."""
    n = len(STAGES)
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_int64 * n)()
    _check(_lib.fcfs_profile_read(ms, cnt, n), "fcfs_profile_read")
    return {STAGES[i]: (float(ms[i]), int(cnt[i])) for i in range(n)}


def _max_group_host(group_ptr):
    if group_ptr is None:
        return 1
    d = group_ptr[1:] - group_ptr[:-1]
    return int(d.max().item()) if d.numel() else 1


def vertices_from_rects(rects, T, group_ptr=None, clip_ptr=None, max_group=None, stream=None):
    """a1: canonical signed corners.  rects int32 [R,4] cuda; group_ptr/clip_ptr int64 cuda or None.

    Returns dict(x, y, w (int32 cuda [K]), corner_ptr (int64 cuda [B+1]), area (int64 cuda [B]), K).
    """
    dev = rects.device
    rects = rects.contiguous()
    R = rects.shape[0]
    G = R if group_ptr is None else group_ptr.shape[0] - 1
    B = 1 if clip_ptr is None else clip_ptr.shape[0] - 1
    mg = _max_group_host(group_ptr) if max_group is None else int(max_group)
    cap = 4 * R if group_ptr is None else 4 * R * max(mg, 1)
    x = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    y = torch.empty_like(x)
    w = torch.empty_like(x)
    cptr = torch.empty(B + 1, dtype=torch.int64, device=dev)
    area = torch.empty(B, dtype=torch.int64, device=dev)
    ws = _ws(_lib.fcfs_vertices_workspace_bytes(R, G, B, mg), dev)
    K = ctypes.c_int64(0)
    st = _lib.fcfs_vertices_from_rects(_ptr(rects), R, _ptr(group_ptr), G, _ptr(clip_ptr), B, int(T), mg,
                                       _ptr(x), _ptr(y), _ptr(w), cap, _ptr(cptr), _ptr(area), ctypes.byref(K),
                                       _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "fcfs_vertices_from_rects")
    k = K.value
    return dict(x=x[:k], y=y[:k], w=w[:k], corner_ptr=cptr, area=area, K=k)


def vertices_from_polygons(vx, vy, poly_ptr, T, clip_ptr=None, stream=None):
    """a1 from polygon vertex lists.  vx, vy int32 cuda [V]; poly_ptr int64 cuda [P+1];
    clip_ptr int64 cuda [B+1] over polygons or None.  At most one corner per vertex.

    Returns dict(x, y, w (int32 cuda [K]), corner_ptr (int64 cuda [B+1]), area (int64 cuda [B]), K).
    """
    dev = poly_ptr.device
    vx, vy = vx.contiguous(), vy.contiguous()
    V = vx.shape[0]
    P = poly_ptr.shape[0] - 1
    B = 1 if clip_ptr is None else clip_ptr.shape[0] - 1
    x = torch.empty(max(V, 1), dtype=torch.int32, device=dev)
    y = torch.empty_like(x)
    w = torch.empty_like(x)
    cptr = torch.empty(B + 1, dtype=torch.int64, device=dev)
    area = torch.empty(B, dtype=torch.int64, device=dev)
    ws = _ws(_lib.fcfs_polygons_workspace_bytes(V, P, B), dev)
    K = ctypes.c_int64(0)
    st = _lib.fcfs_vertices_from_polygons(_ptr(vx), _ptr(vy), V, _ptr(poly_ptr), P, _ptr(clip_ptr), B, int(T),
                                          _ptr(x), _ptr(y), _ptr(w), V, _ptr(cptr), _ptr(area), ctypes.byref(K),
                                          _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "fcfs_vertices_from_polygons")
    k = K.value
    return dict(x=x[:k], y=y[:k], w=w[:k], corner_ptr=cptr, area=area, K=k)


class HaarPlan:
    """Pre-allocated workspace + output for repeated ``fcfs_haar`` calls (B clips of side T)."""

    def __init__(self, B, T, device="cuda"):
        self.B, self.T = int(B), int(T)
        nb = _lib.fcfs_haar_workspace_bytes(self.B, self.T)
        if nb == 0:
            raise FcfsError(E_INVALID, "fcfs_haar_workspace_bytes")
        self.ws = _ws(nb, device)
        self.ws.zero_()                      # fcfs_haar: the scatter scratch is zeroed once, left zero by every call
        self.scratch_bytes = self.B * 5 * (self.T * self.T - 1) // 3 * 8
        self.out = torch.empty((self.B, self.T, self.T), dtype=torch.float64, device=device)

    def run(self, x, y, w, area, corner_ptr=None, stream=None):
        st = _lib.fcfs_haar(_ptr(corner_ptr), self.B, int(x.shape[0]), _ptr(x), _ptr(y), _ptr(w), _ptr(area), self.T,
                            _ptr(self.out), _ptr(self.ws), self.ws.numel(), _stream(stream))
        _check(st, "fcfs_haar")
        return self.out


def haar(x, y, w, area, T, corner_ptr=None, stream=None):
    """Continuous Haar transform: float64 cuda [B, T, T] (reading A18 layout, exact values)."""
    B = 1 if corner_ptr is None else corner_ptr.shape[0] - 1
    return HaarPlan(B, T, device=area.device).run(x, y, w, area, corner_ptr, stream)


class ChopPlan:
    """Pre-allocated outputs + workspace for repeated ``fcfs_chop_rects`` calls (layout -> tiles).
    cap: piece capacity (default R + R/2 + 1024; a call that needs more raises E_CAPACITY)."""

    def __init__(self, R, T, tiles_x, tiles_y, cap=None, device="cuda"):
        self.R, self.T, self.tx, self.ty = int(R), int(T), int(tiles_x), int(tiles_y)
        self.cap = int(cap) if cap is not None else self.R + self.R // 2 + 1024
        self.out = torch.empty((max(self.cap, 1), 4), dtype=torch.int32, device=device)
        self.tile_ptr = torch.empty(self.tx * self.ty + 1, dtype=torch.int64, device=device)
        self.ws = _ws(_lib.fcfs_chop_workspace_bytes(self.R, self.cap, self.tx, self.ty), device)
        self.n = 0

    def run(self, rects, stream=None):
        n = ctypes.c_int64(0)
        st = _lib.fcfs_chop_rects(_ptr(rects), self.R, self.T, self.tx, self.ty, _ptr(self.out), self.cap,
                                  _ptr(self.tile_ptr), ctypes.byref(n), _ptr(self.ws), self.ws.numel(),
                                  _stream(stream))
        self.n = n.value
        _check(st, "fcfs_chop_rects")
        return self.n


def chop_rects(rects, T, tiles_x, tiles_y, stream=None):
    """Layout rects (int32 cuda [R,4]) cut into T x T tiles: dict(rects (tile-local pieces in tile order),
    tile_ptr (int64 [tiles+1]), n).  Retries once with the exact capacity if the default is too small."""
    R = rects.shape[0]
    plan = ChopPlan(R, T, tiles_x, tiles_y, device=rects.device)
    try:
        plan.run(rects.contiguous(), stream)
    except FcfsError as ex:
        if ex.status != E_CAPACITY:
            raise
        plan = ChopPlan(R, T, tiles_x, tiles_y, cap=plan.n if plan.n else None, device=rects.device)
        plan.run(rects.contiguous(), stream)
    return dict(rects=plan.out[:plan.n], tile_ptr=plan.tile_ptr, n=plan.n)


class PolygonsPlan:
    """Pre-allocated outputs + workspace for repeated ``fcfs_vertices_from_polygons`` calls."""

    def __init__(self, V, P, T, B=1, device="cuda"):
        self.V, self.P, self.T, self.B = int(V), int(P), int(T), int(B)
        self.cap = self.V
        self.x = torch.empty(max(self.cap, 1), dtype=torch.int32, device=device)
        self.y = torch.empty_like(self.x)
        self.w = torch.empty_like(self.x)
        self.corner_ptr = torch.empty(self.B + 1, dtype=torch.int64, device=device)
        self.area = torch.empty(self.B, dtype=torch.int64, device=device)
        self.ws = _ws(_lib.fcfs_polygons_workspace_bytes(self.V, self.P, self.B), device)
        self.K = 0

    def run(self, vx, vy, poly_ptr, clip_ptr=None, stream=None):
        K = ctypes.c_int64(0)
        st = _lib.fcfs_vertices_from_polygons(_ptr(vx), _ptr(vy), self.V, _ptr(poly_ptr), self.P, _ptr(clip_ptr),
                                              self.B, self.T, _ptr(self.x), _ptr(self.y), _ptr(self.w), self.cap,
                                              _ptr(self.corner_ptr), _ptr(self.area), ctypes.byref(K), _ptr(self.ws),
                                              self.ws.numel(), _stream(stream))
        _check(st, "fcfs_vertices_from_polygons")
        self.K = K.value
        return self.K


class VerticesPlan:
    """Pre-allocated outputs + workspace for repeated ``fcfs_vertices_from_rects`` calls."""

    def __init__(self, R, T, G=None, B=1, max_group=1, grouped=False, device="cuda"):
        self.R, self.T, self.B = int(R), int(T), int(B)
        self.G = self.R if G is None else int(G)
        self.mg = max(int(max_group), 1)
        self.cap = 4 * self.R * (self.mg if grouped else 1)
        self.x = torch.empty(max(self.cap, 1), dtype=torch.int32, device=device)
        self.y = torch.empty_like(self.x)
        self.w = torch.empty_like(self.x)
        self.corner_ptr = torch.empty(self.B + 1, dtype=torch.int64, device=device)
        self.area = torch.empty(self.B, dtype=torch.int64, device=device)
        self.ws = _ws(_lib.fcfs_vertices_workspace_bytes(self.R, self.G, self.B, self.mg), device)
        self.K = 0
        self.edges = None

    def enable_edges(self):
        """Also write the edge pairing of the corners (fcfs_vertices_from_rects_edges) into self.edges."""
        n = max(self.cap, 1)
        self.edges = {k: torch.empty(n, dtype=torch.int32, device=self.x.device) for k in ("xa", "xb", "y", "c")}
        self.edges["ecnt"] = torch.empty(self.B, dtype=torch.int32, device=self.x.device)
        return self

    def run(self, rects, group_ptr=None, clip_ptr=None, stream=None):
        K = ctypes.c_int64(0)
        if self.edges is None:
            st = _lib.fcfs_vertices_from_rects(_ptr(rects), self.R, _ptr(group_ptr), self.G, _ptr(clip_ptr), self.B,
                                               self.T, self.mg, _ptr(self.x), _ptr(self.y), _ptr(self.w), self.cap,
                                               _ptr(self.corner_ptr), _ptr(self.area), ctypes.byref(K), _ptr(self.ws),
                                               self.ws.numel(), _stream(stream))
        else:
            e = self.edges
            st = _lib.fcfs_vertices_from_rects_edges(
                _ptr(rects), self.R, _ptr(group_ptr), self.G, _ptr(clip_ptr), self.B, self.T, self.mg, _ptr(self.x),
                _ptr(self.y), _ptr(self.w), self.cap, _ptr(self.corner_ptr), _ptr(self.area), ctypes.byref(K),
                _ptr(e["xa"]), _ptr(e["xb"]), _ptr(e["y"]), _ptr(e["c"]), _ptr(e["ecnt"]), _ptr(self.ws),
                self.ws.numel(), _stream(stream))
        _check(st, "fcfs_vertices_from_rects")
        self.K = K.value
        return self.K

    def run_clips_async(self, rects, clip_ptr, max_clip_rects, stream=None):
        """B clips of singleton groups with no host synchronisation (fcfs_vertices_from_clips_async): K and the
        outcome stay on the device (self.K_dev, self.status; ``check_async()`` reads them after the stream's
        work), so the call can be captured in a CUDA graph."""
        if not hasattr(self, "K_dev"):
            self.K_dev = torch.zeros(1, dtype=torch.int64, device=self.x.device)
            self.status = torch.zeros(1, dtype=torch.int32, device=self.x.device)
        st = _lib.fcfs_vertices_from_clips_async(_ptr(rects), self.R, _ptr(clip_ptr), self.B, self.T,
                                                 int(max_clip_rects), _ptr(self.x), _ptr(self.y), _ptr(self.w),
                                                 self.cap, _ptr(self.corner_ptr), _ptr(self.area), _ptr(self.K_dev),
                                                 _ptr(self.status), _ptr(self.ws), self.ws.numel(), _stream(stream))
        _check(st, "fcfs_vertices_from_clips_async")

    def check_async(self):
        """The device-side outcome of run_clips_async (raises on an error status); returns K."""
        st = int(self.status.item())
        if st != FCFS_OK:
            raise FcfsError(st, "fcfs_vertices_from_clips_async (device status)")
        self.K = int(self.K_dev.item())
        return self.K

    def run_band(self, rects, y_lo, y_hi, group_ptr=None, stream=None):
        """One clip's corners with y_lo <= y < y_hi (fcfs_vertices_from_rects_band); self.area[0] is the
        band's share of the area.  Needs B == 1."""
        if self.B != 1:
            raise FcfsError(E_INVALID, "run_band needs a single-clip plan")
        K = ctypes.c_int64(0)
        st = _lib.fcfs_vertices_from_rects_band(_ptr(rects), self.R, _ptr(group_ptr), self.G, self.T, self.mg,
                                                int(y_lo), int(y_hi), _ptr(self.x), _ptr(self.y), _ptr(self.w),
                                                self.cap, _ptr(self.corner_ptr), _ptr(self.area), ctypes.byref(K),
                                                _ptr(self.ws), self.ws.numel(), _stream(stream))
        _check(st, "fcfs_vertices_from_rects_band")
        self.K = K.value
        return self.K


def _out_dtype(prec):
    return torch.complex128 if _PREC[prec] == FP64 else torch.complex64


class CoeffsPlan:
    """Pre-allocated workspace + output for repeated ``fcfs_coeffs`` calls on one clip.
    route: "auto" (the cost model), "gemm" or "fft" (fcfs_options.route)."""

    def __init__(self, K, T, M, N, r2=-1.0, layout="dense", prec="fp64", shard=None, device="cuda", route=None):
        self.K, self.T, self.prec = int(K), int(T), _PREC[prec]
        self.win = make_window(M, N, r2, layout)
        self.shard = shard
        self.opt = make_options(route=route)
        sp = ctypes.byref(shard) if shard is not None else None
        nbytes = _lib.fcfs_coeffs_workspace_bytes(self.K, self.T, ctypes.byref(self.win), self.prec, sp,
                                                  ctypes.byref(self.opt))
        if nbytes == 0:
            raise FcfsError(E_INVALID, "fcfs_coeffs_workspace_bytes")
        self.ws = _ws(nbytes, device)
        if shard is not None and shard.kind == SHARD_ROWS:
            n_out = (shard.m_hi - shard.m_lo + 1) * (2 * int(N) + 1)
        else:
            n_out = window_size(M, N, r2, layout)
        self.out = torch.empty(n_out, dtype=_out_dtype(prec), device=device)

    def run(self, x, y, w, area, stream=None, out=None):
        out = self.out if out is None else out
        sp = ctypes.byref(self.shard) if self.shard is not None else None
        st = _lib.fcfs_coeffs(_ptr(x), _ptr(y), _ptr(w), self.K, int(area), self.T, ctypes.byref(self.win),
                              self.prec, sp, ctypes.byref(self.opt), _ptr(out), _ptr(self.ws), self.ws.numel(),
                              _stream(stream))
        _check(st, "fcfs_coeffs")
        return out

    def run_to_peers(self, x, y, w, area, peers, stream=None):
        """ROWS shard with its all_gather fused into the epilogue (fcfs_coeffs_rows_to_peers): this rank's rows
        are stored at their full-window positions into every buffer of ``peers`` (device pointers or tensors
        of the full DENSE window: this rank's own and the other ranks' mapped into this process)."""
        ptrs = [p if isinstance(p, int) else p.data_ptr() for p in peers]
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        st = _lib.fcfs_coeffs_rows_to_peers(_ptr(x), _ptr(y), _ptr(w), self.K, int(area), self.T,
                                            ctypes.byref(self.win), self.prec, ctypes.byref(self.shard),
                                            ctypes.byref(self.opt), arr, len(ptrs), _ptr(self.ws), self.ws.numel(),
                                            _stream(stream))
        _check(st, "fcfs_coeffs_rows_to_peers")


def coeffs_route(K, T, M, N, r2=-1.0, layout="dense", prec="fp64", shard=None, route=None):
    """1 if fcfs_coeffs takes the lattice-FFT route for these sizes (y-sorted corners), else 0."""
    win = make_window(M, N, r2, layout)
    sp = ctypes.byref(shard) if shard is not None else None
    opt = make_options(route=route)
    return int(_lib.fcfs_coeffs_route(int(K), int(T), ctypes.byref(win), _PREC[prec], sp, ctypes.byref(opt)))


def coeffs(x, y, w, area, T, M, N, r2=-1.0, layout="dense", prec="fp64", shard=None, stream=None, route=None):
    """a2-a5 for one clip.  Returns complex128 (fp64) or complex64 (tf32x3) cuda tensor."""
    plan = CoeffsPlan(x.shape[0], T, M, N, r2, layout, prec, shard, device=x.device, route=route)
    return plan.run(x, y, w, area, stream=stream)


class AsyncClipPlan:
    """One clip's a1-a5 with no host synchronisation (fcfs_vertices_from_rects_async + fcfs_coeffs_async
    on the lattice-FFT route): K, the area and the outcome stay on the device, so the whole step can be
    captured in a CUDA graph.  ``check()`` (after the stream's work) raises on a device-reported error and
    returns K."""

    def __init__(self, R, T, M, N, r2=-1.0, layout="dense", prec="fp64", G=None, max_group=1, device="cuda"):
        self.vp = VerticesPlan(R, T, G, 1, max_group, grouped=max_group > 1 or (G is not None and G != R),
                               device=device)
        self.T, self.prec = int(T), _PREC[prec]
        self.win = make_window(M, N, r2, layout)
        self.K_cap = max(self.vp.cap, 1)
        self.opt = make_options(route="fft")
        nbytes = _lib.fcfs_coeffs_workspace_bytes(self.K_cap, self.T, ctypes.byref(self.win), self.prec, None,
                                                  ctypes.byref(self.opt))
        if nbytes == 0:
            raise FcfsError(E_INVALID, "fcfs_coeffs_workspace_bytes")
        self.ws = _ws(nbytes, device)
        self.out = torch.empty(window_size(M, N, r2, layout), dtype=_out_dtype(prec), device=device)
        self.K = torch.zeros(1, dtype=torch.int64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)

    def run(self, rects, group_ptr=None, stream=None):
        vp = self.vp
        st = _lib.fcfs_vertices_from_rects_async(_ptr(rects), vp.R, _ptr(group_ptr), vp.G, None, 1, vp.T, vp.mg,
                                                 _ptr(vp.x), _ptr(vp.y), _ptr(vp.w), vp.cap, _ptr(vp.corner_ptr),
                                                 _ptr(vp.area), _ptr(self.K), _ptr(self.status), _ptr(vp.ws),
                                                 vp.ws.numel(), _stream(stream))
        _check(st, "fcfs_vertices_from_rects_async")
        st = _lib.fcfs_coeffs_async(_ptr(vp.x), _ptr(vp.y), _ptr(vp.w), _ptr(self.K), self.K_cap, _ptr(vp.area),
                                    self.T, ctypes.byref(self.win), self.prec, _ptr(self.out), _ptr(self.status),
                                    _ptr(self.ws), self.ws.numel(), _stream(stream))
        _check(st, "fcfs_coeffs_async")
        return self.out

    def check(self):
        st = int(self.status.item())
        if st != FCFS_OK:
            raise FcfsError(st, "AsyncClipPlan (device status)")
        return int(self.K.item())


class SmallClipPlan:
    """fcfs_small_clip: a1-a5 of one small clip in one kernel launch, no host synchronisation (the step
    can be captured in a CUDA graph).  ``status`` / ``K`` are device tensors written by the kernel."""

    def __init__(self, R, T, M, N, r2=-1.0, layout="dense", prec="fp64", G=None, max_group=1, device="cuda"):
        self.R, self.T, self.prec = int(R), int(T), _PREC[prec]
        self.G = self.R if G is None else int(G)
        self.mg = max(int(max_group), 1)
        self.win = make_window(M, N, r2, layout)
        self.out = torch.empty(window_size(M, N, r2, layout), dtype=_out_dtype(prec), device=device)
        self.K = torch.zeros(1, dtype=torch.int64, device=device)
        self.status = torch.full((1,), -1, dtype=torch.int32, device=device)

    @staticmethod
    def supported(R, T, M, N, r2=-1.0, layout="dense", G=None, max_group=1):
        win = make_window(M, N, r2, layout)
        return bool(_lib.fcfs_small_clip_supported(int(R), int(R if G is None else G), int(T), int(max_group),
                                                   ctypes.byref(win)))

    def run(self, rects, group_ptr=None, stream=None):
        st = _lib.fcfs_small_clip(_ptr(rects), self.R, _ptr(group_ptr), self.G, self.T, self.mg,
                                  ctypes.byref(self.win), self.prec, _ptr(self.out), _ptr(self.K),
                                  _ptr(self.status), _stream(stream))
        _check(st, "fcfs_small_clip")
        return self.out

    def check(self):
        """After the stream's work completed: raise if the kernel reported an error."""
        st = int(self.status.item())
        if st != FCFS_OK:
            raise FcfsError(st, "fcfs_small_clip (device status)")
        return int(self.K.item())


class BatchedPlan:
    """Pre-allocated workspace + output for repeated ``fcfs_coeffs_batched`` calls.
    form: "auto", "edge", "corner" or "lattice" (fcfs_options.form; split precisions); sorted_y: see
    make_options."""

    def __init__(self, B, K_total, K_max, T, M, N, r2=-1.0, layout="dense", prec="tf32x3", device="cuda",
                 form=None, sorted_y=False):
        self.B, self.K_total, self.K_max, self.T, self.prec = int(B), int(K_total), int(K_max), int(T), _PREC[prec]
        self.win = make_window(M, N, r2, layout)
        self.opt = make_options(form=form, sorted_y=sorted_y)
        nbytes = _lib.fcfs_batched_workspace_bytes(self.B, self.K_total, self.K_max, self.T,
                                                   ctypes.byref(self.win), self.prec, ctypes.byref(self.opt))
        if nbytes == 0:
            raise FcfsError(E_INVALID, "fcfs_batched_workspace_bytes")
        self.ws = _ws(nbytes, device)
        self.per_clip = window_size(M, N, r2, layout)
        self.out = torch.empty(self.B * self.per_clip, dtype=_out_dtype(prec), device=device)
        self.form = int(_lib.fcfs_coeffs_batched_form(self.B, self.K_total, self.K_max, self.T,
                                                      ctypes.byref(self.win), self.prec, ctypes.byref(self.opt)))

    def run(self, corner_ptr, x, y, w, area, stream=None, out=None, edges=None):
        """edges: the pairing of these corners (dict xa, xb, y, c, ecnt from ``edges`` or
        ``VerticesPlan.enable_edges``) to contract over instead of pairing again, or None."""
        out = self.out if out is None else out
        if edges is None:
            st = _lib.fcfs_coeffs_batched(_ptr(corner_ptr), self.B, self.K_total, self.K_max, _ptr(x), _ptr(y),
                                          _ptr(w), _ptr(area), self.T, ctypes.byref(self.win), self.prec,
                                          ctypes.byref(self.opt), _ptr(out), _ptr(self.ws), self.ws.numel(),
                                          _stream(stream))
        else:
            st = _lib.fcfs_coeffs_batched_edges(
                _ptr(corner_ptr), self.B, self.K_total, self.K_max, _ptr(x), _ptr(y), _ptr(w), _ptr(area),
                _ptr(edges["xa"]), _ptr(edges["xb"]), _ptr(edges["y"]), _ptr(edges["c"]), _ptr(edges["ecnt"]),
                self.T, ctypes.byref(self.win), self.prec, ctypes.byref(self.opt), _ptr(out), _ptr(self.ws),
                self.ws.numel(), _stream(stream))
        _check(st, "fcfs_coeffs_batched")
        return out.view(self.B, self.per_clip)


def coeffs_batched(corner_ptr, x, y, w, area, T, M, N, r2=-1.0, layout="dense", prec="tf32x3", K_max=None,
                   stream=None, form=None, sorted_y=False):
    B = corner_ptr.shape[0] - 1
    if K_max is None:
        K_max = int((corner_ptr[1:] - corner_ptr[:-1]).max().item()) if B > 0 else 0
    plan = BatchedPlan(B, x.shape[0], K_max, T, M, N, r2, layout, prec, device=x.device, form=form,
                       sorted_y=sorted_y)
    return plan.run(corner_ptr, x, y, w, area, stream=stream)


def edges(corner_ptr, x, y, w, stream=None):
    """Edge pairing of a corner list (fcfs_edges): dict xa, xb, y, c (int32 [K], clip b's edges at
    [corner_ptr[b], corner_ptr[b] + ecnt[b])) and ecnt (int32 [B])."""
    K = int(x.shape[0])
    B = int(corner_ptr.shape[0]) - 1
    dev = x.device
    out = {k: torch.full((max(K, 1),), -7, dtype=torch.int32, device=dev) for k in ("xa", "xb", "y", "c")}
    ecnt = torch.empty(max(B, 1), dtype=torch.int32, device=dev)
    _check(_lib.fcfs_edges(_ptr(x), _ptr(y), _ptr(w), _ptr(corner_ptr), B, _ptr(out["xa"]), _ptr(out["xb"]),
                           _ptr(out["y"]), _ptr(out["c"]), _ptr(ecnt), _stream(stream)), "fcfs_edges")
    out["ecnt"] = ecnt[:B]
    return out


def row_buckets(y, corner_ptr=None, cap=32, stream=None):
    """Row buckets of a corner list (fcfs_row_buckets): dict bptr [nb+1], by [nb], clip_bptr [B+1], nb."""
    K = int(y.shape[0])
    B = 1 if corner_ptr is None else int(corner_ptr.shape[0]) - 1
    dev = y.device
    bptr = torch.empty(K + 1, dtype=torch.int32, device=dev)
    by = torch.empty(max(K, 1), dtype=torch.int32, device=dev)
    clip_bptr = torch.empty(B + 1, dtype=torch.int64, device=dev)
    ws = _ws(_lib.fcfs_row_buckets_workspace_bytes(K, B), dev)
    nb = _i64(0)
    _check(_lib.fcfs_row_buckets(_ptr(y), _ptr(corner_ptr), B, K, int(cap), _ptr(bptr), _ptr(by), _ptr(clip_bptr),
                                 ctypes.byref(nb), _ptr(ws), ws.numel(), _stream(stream)), "fcfs_row_buckets")
    n = int(nb.value)
    return {"bptr": bptr[:n + 1], "by": by[:n], "clip_bptr": clip_bptr, "nb": n}
