"""Build libfcfs.so in-tree with nvcc for sm_100a (explicit -gencode; no torch arch list)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libfcfs.so")
CHECKED_LIB = os.path.join(HERE, "libfcfs_checked.so")
SOURCES = ["fcfs_abi.cu", "extract.cu", "buckets.cu", "contract_fp64.cu", "contract_tf32.cu", "epilogue.cu", "fft_route.cu", "chop.cu", "haar.cu", "edges.cu", "lattice.cu", "small.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src, os.path.join(CSRC, "common.cuh"), os.path.join(ROOT, "include", "fcfs.h")]
    deps += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, extra=(), checked: bool = False) -> str:
    """libfcfs.so; checked=True builds libfcfs_checked.so instead: the same sources with -DFCFS_CHECKED
    (device-side FCFS_DCHECK invariants, common.cuh), for tests only."""
    lib = CHECKED_LIB if checked else LIB
    if checked:
        extra = (*extra, "-DFCFS_CHECKED")
    objdir = os.path.join(HERE, "build_obj_checked" if checked else "build_obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        objs.append(obj)
        if _stale(obj, src):
            cmd = [NVCC, *FLAGS, *extra, "-c", src, "-o", obj]
            if verbose:
                print(" ".join(cmd), flush=True)
            procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for s, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose and out:
            sys.stderr.write(out.decode())
    if procs or not os.path.exists(lib):
        tmp = lib + f".tmp{os.getpid()}"
        subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
                               "-cudart", "static"])
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(verbose=True, checked="--checked" in sys.argv))
