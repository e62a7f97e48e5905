"""B200-native fast continuous Fourier series (FCFS) of rectilinear polygons (arXiv 1010.5562).

Submodules:
  inputs  seeded synthetic workloads (no FCFS arithmetic; shared with the oracle tests)
  fcfs    ctypes binding of the C-ABI library libfcfs.so (include/fcfs.h); loading it
          fails loudly if the CUDA library is missing — there is no CPU fallback.
"""
__all__ = ["inputs", "fcfs"]
