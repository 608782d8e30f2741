"""Operators A and T (= A^T or an unmatched B ~ A^T) for the oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md L23-31 (eq. inverseproblem): b = A x_true + e; the methods only touch A
through products A z and A^T w (or A# w for an unmatched transpose, L86-87,
L1640-1647).
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "oracle_csr.c")
_LIB = os.path.join(_HERE, "liboracle_csr.so")
_lib = None


def build_lib(force: bool = False) -> str:
    """gcc -O2 -ffp-contract=off: plain single-threaded C, no BLAS."""
    stale = (not os.path.exists(_LIB)) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC)
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", _SRC, "-o", tmp],
                       check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _get():
    global _lib
    if _lib is None:
        build_lib()
        lib = ctypes.CDLL(_LIB)
        i64p, i32p, f64p = (ctypes.POINTER(t) for t in (ctypes.c_int64, ctypes.c_int32, ctypes.c_double))
        lib.oracle_csr_matvec.argtypes = [ctypes.c_int64, i64p, i32p, f64p, f64p, f64p]
        lib.oracle_csr_matvec.restype = None
        lib.oracle_csr_transpose.argtypes = [ctypes.c_int64, ctypes.c_int64, i64p, i32p, f64p, i64p, i32p, f64p]
        lib.oracle_csr_transpose.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class OracleCSR:
    """CSR matrix with a plain single-threaded product."""

    def __init__(self, nrows, ncols, rowptr, col, val):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int32)
        self.val = np.ascontiguousarray(val, dtype=np.float64)

    def matvec(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.ncols,):
            raise ValueError("dimension mismatch")
        y = np.empty(self.nrows)
        _get().oracle_csr_matvec(self.nrows, _p(self.rowptr, ctypes.c_int64), _p(self.col, ctypes.c_int32),
                                 _p(self.val, ctypes.c_double), _p(x, ctypes.c_double), _p(y, ctypes.c_double))
        return y

    def transpose(self) -> "OracleCSR":
        nnz = int(self.rowptr[-1])
        trp = np.empty(self.ncols + 1, dtype=np.int64)
        tcol = np.empty(nnz, dtype=np.int32)
        tval = np.empty(nnz, dtype=np.float64)
        rc = _get().oracle_csr_transpose(self.nrows, self.ncols, _p(self.rowptr, ctypes.c_int64),
                                         _p(self.col, ctypes.c_int32), _p(self.val, ctypes.c_double),
                                         _p(trp, ctypes.c_int64), _p(tcol, ctypes.c_int32),
                                         _p(tval, ctypes.c_double))
        if rc != 0:
            raise ValueError("transpose failed")
        return OracleCSR(self.ncols, self.nrows, trp, tcol, tval)


class CSROperator:
    """A as CSR; T = A^T (built here by the oracle's own transpose) or a given B."""

    def __init__(self, A: OracleCSR, T: OracleCSR = None):
        self.A = A
        self.T = T if T is not None else A.transpose()
        self.m, self.n = A.nrows, A.ncols
        if (self.T.nrows, self.T.ncols) != (self.n, self.m):
            raise ValueError("T must be n x m")

    def matvec(self, z):
        return self.A.matvec(z)

    def tmatvec(self, w):
        return self.T.matvec(w)


class DenseOperator:
    """Tiny dense A with T = A^T or a given dense B (pins P4-P6)."""

    def __init__(self, A, T=None):
        self.Ad = np.asarray(A, dtype=np.float64)
        self.Td = self.Ad.T.copy() if T is None else np.asarray(T, dtype=np.float64)
        self.m, self.n = self.Ad.shape

    def matvec(self, z):
        return self.Ad @ z

    def tmatvec(self, w):
        return self.Td @ w


def blur_taps(sigma: float, radius: int) -> np.ndarray:
    """1-D Gaussian taps g_t ~ exp(-t^2 / (2 sigma^2)), t = -radius..radius, sum 1 (reading R15)."""
    t = np.arange(-radius, radius + 1, dtype=np.float64)
    g = np.exp(-(t * t) / (2.0 * sigma * sigma))
    return g / np.sum(g)


class BlurOperator:
    """Gaussian PSF blur with zero boundary (BASELINE.json config 2).

    Plain 2-D definition: Y[i,j] = sum_{u,v=-r..r} g_u g_v X[i+u, j+v], X = 0
    outside the H x W image; x, y are row-major vectorisations.  The PSF
    outer(g, g) is symmetric, so A^T = A (T = A).
    """

    def __init__(self, H, W, sigma, radius):
        self.H, self.W, self.r = int(H), int(W), int(radius)
        self.g = blur_taps(sigma, radius)
        self.m = self.n = self.H * self.W

    def matvec(self, x):
        r, H, W = self.r, self.H, self.W
        Xp = np.zeros((H + 2 * r, W + 2 * r))
        Xp[r:r + H, r:r + W] = np.asarray(x).reshape(H, W)
        Y = np.zeros((H, W))
        for u in range(-r, r + 1):
            for v in range(-r, r + 1):
                Y += (self.g[u + r] * self.g[v + r]) * Xp[r + u:r + u + H, r + v:r + v + W]
        return Y.reshape(-1)

    def tmatvec(self, w):
        return self.matvec(w)


def operator_from_problem(prob) -> object:
    """Oracle operator for a gen.Problem: CSR (T built by the oracle, or the given B) or blur."""
    if prob.t_mode == "same":
        bl = prob.blur
        return BlurOperator(bl["H"], bl["W"], bl["sigma"], bl["radius"])
    A = OracleCSR(prob.A.nrows, prob.A.ncols, prob.A.rowptr, prob.A.col, prob.A.val)
    T = None
    if prob.t_mode == "given":
        T = OracleCSR(prob.T.nrows, prob.T.ncols, prob.T.rowptr, prob.T.col, prob.T.val)
    return CSROperator(A, T)
