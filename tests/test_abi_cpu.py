"""C-ABI checks that need no GPU: the library loads, exports every symbol the header
declares, struct layouts match, and the host helpers agree with the oracle's window
enumeration.  No compute entry point is called here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_1010_5562_b200 import inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fcfs.h")


@pytest.fixture(scope="module")
def fcfs():
    from paper_1010_5562_b200 import build
    build.build()
    from paper_1010_5562_b200 import fcfs as f
    return f


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fcfs_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported(fcfs):
    declared = _declared_functions()
    assert len(declared) >= 12
    lib = ctypes.CDLL(fcfs.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/fcfs.h but not exported"
    assert sorted(fcfs.EXPORTED) == declared


def test_library_is_sm100a_only(fcfs):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", fcfs.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def test_struct_layouts(fcfs):
    assert ctypes.sizeof(fcfs.Window) == 24 and fcfs.Window.pupil_r2.offset == 8 and fcfs.Window.layout.offset == 16
    assert ctypes.sizeof(fcfs.Shard) == 32 and fcfs.Shard.k_lo.offset == 16 and fcfs.Shard.k_hi.offset == 24
    assert ctypes.sizeof(fcfs.Options) == 32 and fcfs.Options.form.offset == 4 and fcfs.Options.sorted_y.offset == 8 \
        and fcfs.Options.reserved.offset == 12


def test_window_helpers_match_oracle(fcfs):
    r2 = inputs.pupil_r2(2048)
    assert fcfs.window_size(27, 27, r2, "pupil") == 2337
    assert fcfs.window_size(32, 32) == 65 * 65
    assert fcfs.window_size(3, 5, 10.0, "dense") == 7 * 11
    ms, ns = fcfs.pupil_indices(27, 27, r2)
    oms, ons = oracle.window(27, 27, r2)
    assert np.array_equal(ms.numpy(), oms) and np.array_equal(ns.numpy(), ons)
    ms, ns = fcfs.pupil_indices(5, 3, 9.0)
    oms, ons = oracle.window(5, 3, 9.0)
    assert np.array_equal(ms.numpy(), oms) and np.array_equal(ns.numpy(), ons)
    with pytest.raises(fcfs.FcfsError):
        fcfs.window_size(3, 3, -1.0, "pupil")


def test_status_strings_and_no_gpu_behaviour(fcfs):
    assert fcfs._lib.fcfs_status_string(0) == b"FCFS_OK"
    assert fcfs._lib.fcfs_status_string(5) == b"FCFS_E_UNSUPPORTED"
    import torch
    if not torch.cuda.is_available():
        st = fcfs._lib.fcfs_device_check()
        assert st != 0                      # fails loudly without an sm_100 device


def test_workspace_queries_are_positive(fcfs):
    w = fcfs.make_window(512, 512)
    assert fcfs._lib.fcfs_coeffs_workspace_bytes(1_000_000, 65536, ctypes.byref(w), 0, None, None) > 0
    assert fcfs._lib.fcfs_vertices_workspace_bytes(250_000, 250_000, 1, 1) > 250_000 * 4 * 8
    wp = fcfs.make_window(27, 27, inputs.pupil_r2(2048), "pupil")
    assert fcfs._lib.fcfs_batched_workspace_bytes(4096, 4096 * 4800, 5000, 2048, ctypes.byref(wp), 1, None) > 0


def test_options_are_validated_and_route_forcing_is_explicit(fcfs):
    """The library reads no environment variable: routes and forms are fcfs_options fields, and a bad
    option (unknown enum, non-zero reserved word) is rejected by the planning queries (no device needed)."""
    import subprocess
    out = subprocess.run(["strings", fcfs.LIB_PATH], capture_output=True, text=True).stdout
    for env in ("FCFS_DEBUG", "FCFS_EDGES", "FCFS_ROUTE"):
        assert env not in out
    w = fcfs.make_window(512, 512)
    good = fcfs.make_options(route="fft")
    assert fcfs._lib.fcfs_coeffs_route(1_000_000, 65536, ctypes.byref(w), 0, None, ctypes.byref(good)) == 1
    gemm = fcfs.make_options(route="gemm")
    assert fcfs._lib.fcfs_coeffs_route(1_000_000, 65536, ctypes.byref(w), 0, None, ctypes.byref(gemm)) == 0
    bad = fcfs.make_options()
    bad.reserved[3] = 1
    assert fcfs._lib.fcfs_coeffs_workspace_bytes(1000, 4096, ctypes.byref(w), 0, None, ctypes.byref(bad)) == 0
    bad = fcfs.Options(7, 0)
    assert fcfs._lib.fcfs_coeffs_route(1000, 4096, ctypes.byref(w), 0, None, ctypes.byref(bad)) == 0
    wp = fcfs.make_window(27, 27, inputs.pupil_r2(2048), "pupil")
    form = fcfs._lib.fcfs_coeffs_batched_form
    assert form(4096, 1 << 24, 5000, 2048, ctypes.byref(wp), 1, None) == fcfs.FORM_LATTICE     # c3: dense clips
    assert form(4096, 4096 * 40, 50, 2048, ctypes.byref(wp), 1, None) == fcfs.FORM_EDGE       # sparse clips
    e = fcfs.make_options(form="edge")
    assert form(4096, 1 << 24, 5000, 2048, ctypes.byref(wp), 1, ctypes.byref(e)) == fcfs.FORM_EDGE
    lat = fcfs.make_options(form="lattice")
    assert form(4096, 4096 * 40, 50, 2048, ctypes.byref(wp), 1, ctypes.byref(lat)) == fcfs.FORM_LATTICE
    assert form(4096, 1 << 24, 5000, 2050, ctypes.byref(wp), 1, ctypes.byref(lat)) == fcfs.FORM_EDGE   # T % 4
    wide = fcfs.make_window(40, 27)
    assert form(16, 1 << 16, 5000, 2048, ctypes.byref(wide), 1, ctypes.byref(lat)) == fcfs.FORM_EDGE  # M > 31
    c = fcfs.make_options(form="corner")
    assert form(4096, 1 << 24, 5000, 2048, ctypes.byref(wp), 1, ctypes.byref(c)) == fcfs.FORM_CORNER
    assert form(4096, 1 << 24, 5000, 2048, ctypes.byref(wp), 2, None) == fcfs.FORM_CORNER


def _build_c_demo(fcfs, out):
    """gcc, plain C: include/fcfs.h is a C header and libfcfs.so is usable without Python."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    lib_dir = os.path.dirname(fcfs.LIB_PATH)
    cuda = "/usr/local/cuda"
    subprocess.check_call([gcc, "-O2", "-Wall", "-Werror", "-std=c11", os.path.join(ROOT, "examples", "fcfs_c_demo.c"),
                           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
                           "-L", lib_dir, "-lfcfs", "-L", os.path.join(cuda, "lib64"), "-lcudart",
                           f"-Wl,-rpath,{lib_dir}:{os.path.join(cuda, 'lib64')}", "-o", out])
    return out


def test_c_demo_compiles_and_links(fcfs, tmp_path):
    exe = _build_c_demo(fcfs, str(tmp_path / "fcfs_c_demo"))
    assert os.path.exists(exe)
