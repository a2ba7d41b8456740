"""B200-native (sm_100a) GMG + multi-color LU-SGS hot path of arXiv 2509.06347.

The product is libgmg.so (C ABI in include/gmg.h); `gmg` is its thin ctypes
binding.  No CPU fallback exists: compute calls fail loudly without the
extension or a CUDA device.
"""
from .gmg import (ABI_SYMBOLS, GmgError, Options, Solver, lib)  # noqa: F401

__all__ = ["ABI_SYMBOLS", "GmgError", "Options", "Solver", "lib"]
