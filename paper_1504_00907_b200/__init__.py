"""B200-native DDG-preconditioned CG (arXiv:1504.00907) behind the C ABI of libddg.

The package holds only what the hot path needs: csrc/ (sm_100a kernels, host
setup, C ABI), build.py (in-tree nvcc build) and ddg.py (ctypes binding).
"""
from .ddg import DDGError, Solver, load  # noqa: F401

__all__ = ["Solver", "DDGError", "load"]
