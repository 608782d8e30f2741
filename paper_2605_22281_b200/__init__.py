"""B200-native sketched flexible Golub-Kahan step (sFLSQR / sFLSMR, arXiv 2605.22281).

The product is the C-ABI library ``lib/libsflsqr.so`` (include/sflsqr.h) built
from ``csrc/`` for sm_100a; ``sflsqr.py`` is its thin ctypes binding.
"""
from ._build import LIB_PATH, build_library  # noqa: F401
from .sflsqr import SFLSQR, SflsqrError, load_library, solve, solver_for_problem  # noqa: F401

__all__ = ["SFLSQR", "SflsqrError", "load_library", "solve", "solver_for_problem", "build_library", "LIB_PATH"]
