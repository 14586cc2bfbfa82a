"""B200-native segmental-refinement full multigrid (Adams, Brown, Knepley, Samtaney,
arXiv 1406.7808): the FMG+SR solve of the cell-centred 7-point 3D Poisson problem.

The product is the C-ABI shared library `libsrfmg.so` (include/sr_fmg.h) built from
`csrc/` for sm_100a; `Solver` is its ctypes front end.  Importing this package fails if the
library has not been built -- there is no CPU fallback.
"""
from ._lib import LIB_PATH, SrError, kernel_names  # noqa: F401  (raises if .so missing)
from .api import HostStore, LevelInfo, Solver, nccl_unique_id, partition  # noqa: F401

__all__ = ["Solver", "LevelInfo", "SrError", "kernel_names", "LIB_PATH", "partition",
           "nccl_unique_id", "HostStore"]
