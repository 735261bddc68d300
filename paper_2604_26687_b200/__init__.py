"""paper_2604_26687_b200 — B200-native online GNS estimation (COPUS,
arXiv 2604.26687) behind the reference's coadapt API.

Layout:
  csrc/        sm_100a kernels (kernels.cu), the C-ABI (cabi.cu) and the C++20
               implementation of the reference headers (host/*.cpp) ->
               lib/libcoadapt_b200.so
  _lib.py      ctypes binding of include/coadapt_cuda.h + coadapt_host.h
  gns.py       Python mirror of gns.hpp / goodput.hpp / decide
  device.py    device plan + step accumulator handles (the hot path)
  layout.py    model shapes and (d,t,p) shard layouts with dedup weights
"""
from . import _lib
from ._lib import (CudaError, GnsResult, GnsState, InternalError, NcclError, StepStats,
                   ValidationError, lib)

__all__ = ["CudaError", "GnsResult", "GnsState", "InternalError", "NcclError", "StepStats",
           "ValidationError", "lib", "_lib"]
