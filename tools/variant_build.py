"""A/B builds of one source file: compile csrc/<file> with extra -D flags and link it with the other objects of
the default build into paper_1010_5562_b200/variants/libfcfs_<tag>.so (git-ignored; travels to the GPU box with
the snapshot).  Select one at run time with FCFS_LIBRARY=<path> (tests / bench only).

usage: python tools/variant_build.py <file.cu> <tag> [-DNAME[=V] ...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1010_5562_b200 import build as b  # noqa: E402


def main():
    src, tag, *defs = sys.argv[1:]
    b.build()
    objdir = os.path.join(b.HERE, "build_obj")
    outdir = os.path.join(b.HERE, "variants")
    os.makedirs(outdir, exist_ok=True)
    obj = os.path.join(outdir, f"{src.replace('.cu', '')}_{tag}.o")
    subprocess.check_call([b.NVCC, *b.FLAGS, *defs, "-c", os.path.join(b.CSRC, src), "-o", obj])
    objs = [obj if s == src else os.path.join(objdir, s.replace(".cu", ".o")) for s in b.SOURCES]
    lib = os.path.join(outdir, f"libfcfs_{tag}.so")
    subprocess.check_call([b.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs,
                           "-cudart", "static"])
    print(lib)


if __name__ == "__main__":
    main()
