"""B200-native data-parallel wavefront ray tracer (arxiv 2407.00179, "Data-Parallel ANARI").

The product is libdpr.so (C ABI in include/dpr.h: sm_100a CUDA kernels + NCCL); this
package holds its sources (csrc/), the build script and the thin ctypes binding (dpr.py).
"""
from . import dpr  # noqa: F401

__all__ = ["dpr"]
