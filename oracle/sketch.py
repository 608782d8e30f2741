"""Sparse-sign sketch S (d x dim) for the oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper uses a Gaussian sketch and CountSketch
(L1390, L1615-1616); BASELINE.json asks for a sparse-sign sketch with d rows and
s nonzeros per column.  Reading R5/R6:

  * column i (the GLOBAL, original-order coordinate index of the sketched vector)
    has exactly s distinct rows, each with an independent sign, value +-1/sqrt(s);
  * the t-th nonzero (t = 0..s-1) of column i is drawn by Philox4x32-10 with
    key = (seed_lo32, seed_hi32), counter = (i_lo32, i_hi32, t, attempt):
        row  = (w0 * d) >> 32          (w0, w1 the first two output words)
        sign = -1 if (w1 & 1) else +1
    starting at attempt = 0 and incrementing attempt while row equals one of the
    rows already chosen for nonzeros 0..t-1 of the same column.
  * s = 1 is CountSketch.
"""
import numpy as np

from .philox import philox4x32_10


def sparse_sign_table(seed: int, d: int, s: int, col0: int, ncols: int):
    """Return (rows int32 (ncols, s), signs int8 (ncols, s)) for columns col0..col0+ncols-1."""
    if not (1 <= s <= d):
        raise ValueError("need 1 <= s <= d")
    i = np.arange(col0, col0 + ncols, dtype=np.uint64)
    key = np.array([seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF], dtype=np.uint64)
    rows = np.empty((ncols, s), dtype=np.int64)
    signs = np.empty((ncols, s), dtype=np.int8)
    ilo = i & np.uint64(0xFFFFFFFF)
    ihi = i >> np.uint64(32)
    for t in range(s):
        attempt = np.zeros(ncols, dtype=np.uint64)
        todo = np.arange(ncols)
        while todo.size:
            ctr = np.stack([ilo[todo], ihi[todo], np.full(todo.size, t, dtype=np.uint64), attempt[todo]], axis=-1)
            w = philox4x32_10(ctr, key).astype(np.uint64)
            r = ((w[:, 0] * np.uint64(d)) >> np.uint64(32)).astype(np.int64)
            sg = np.where((w[:, 1] & np.uint64(1)) == 1, -1, 1).astype(np.int8)
            dup = np.zeros(todo.size, dtype=bool)
            for u in range(t):
                dup |= rows[todo, u] == r
            ok = ~dup
            rows[todo[ok], t] = r[ok]
            signs[todo[ok], t] = sg[ok]
            attempt[todo[dup]] += np.uint64(1)
            todo = todo[dup]
    return rows.astype(np.int32), signs


class SparseSignSketch:
    """S in R^{d x dim}; apply(v) = S v, with the table generated once."""

    def __init__(self, seed: int, d: int, s: int, dim: int):
        self.seed, self.d, self.s, self.dim = seed, d, s, dim
        self.rows, self.signs = sparse_sign_table(seed, d, s, 0, dim)
        self.scale = 1.0 / np.sqrt(s)

    def apply(self, v: np.ndarray) -> np.ndarray:
        """S v: y[row(i,t)] += sign(i,t) * v_i / sqrt(s), accumulated in (i, t) order."""
        y = np.zeros(self.d)
        contrib = (self.signs.astype(np.float64) * self.scale) * v[:, None]
        np.add.at(y, self.rows.reshape(-1), contrib.reshape(-1))
        return y

    def dense(self) -> np.ndarray:
        S = np.zeros((self.d, self.dim))
        cols = np.repeat(np.arange(self.dim), self.s)
        S[self.rows.reshape(-1), cols] = self.signs.reshape(-1) * self.scale
        return S


class IdentitySketch:
    """S = I (d = dim): the unsketched reduction used by pins P4a-P4c."""

    def __init__(self, dim: int):
        self.d = self.dim = dim

    def apply(self, v):
        return np.array(v, dtype=np.float64, copy=True)


class DenseSketch:
    """Explicit dense S (e.g. S A^T for the Remark of PAPER.md L810-822, pin P5)."""

    def __init__(self, S: np.ndarray):
        self.S = np.asarray(S, dtype=np.float64)
        self.d, self.dim = self.S.shape

    def apply(self, v):
        return self.S @ v


GAUSS_DOMAIN = 0x47415553   # 'GAUS': counter word 3 of the Gaussian draws (reading R21)


def gaussian_table(seed: int, d: int, col0: int, ncols: int) -> np.ndarray:
    """Gaussian sketch entries S[r, i] for columns i in [col0, col0+ncols), shape (d, ncols).

    Reading R21: the paper's Gaussian sketch (Theorem 2.1 /
    Corollary L1011-1121) with i.i.d. N(0, 1/d) entries, drawn by a counter-based
    generator so that any rank can produce any column: for the pair t of rows (2t, 2t+1)
    of column i, (w0, w1, w2, w3) = Philox4x32-10(key = (seed_lo, seed_hi),
    counter = (i_lo, i_hi, t, 'GAUS')); u1 = (((w1 << 32) | w0) >> 11 + 1/2) 2^-53,
    u2 likewise from (w3, w2); Box-Muller: g_2t = sqrt(-2 ln u1) cos(2 pi u2),
    g_2t+1 = sqrt(-2 ln u1) sin(2 pi u2); S[r, i] = g_r / sqrt(d).
    """
    npair = (d + 1) // 2
    i = np.arange(col0, col0 + ncols, dtype=np.uint64)
    key = np.array([seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF], dtype=np.uint64)
    S = np.empty((d, ncols))
    for t in range(npair):
        ctr = np.stack([i & np.uint64(0xFFFFFFFF), i >> np.uint64(32), np.full(ncols, t, dtype=np.uint64),
                        np.full(ncols, GAUSS_DOMAIN, dtype=np.uint64)], axis=-1)
        w = philox4x32_10(ctr, key).astype(np.uint64)
        a = ((w[:, 1] << np.uint64(32)) | w[:, 0]) >> np.uint64(11)
        b = ((w[:, 3] << np.uint64(32)) | w[:, 2]) >> np.uint64(11)
        u1 = (a.astype(np.float64) + 0.5) * 2.0 ** -53
        u2 = (b.astype(np.float64) + 0.5) * 2.0 ** -53
        r = np.sqrt(-2.0 * np.log(u1))
        th = (2.0 * np.pi) * u2
        S[2 * t] = r * np.cos(th)
        if 2 * t + 1 < d:
            S[2 * t + 1] = r * np.sin(th)
    return S / np.sqrt(d)


class GaussianSketch:
    """Dense Gaussian S in R^{d x dim} (reading R21); apply(v) = S v (row-wise dot products)."""

    def __init__(self, seed: int, d: int, dim: int):
        self.seed, self.d, self.dim = seed, d, dim
        self.S = gaussian_table(seed, d, 0, dim)

    def apply(self, v: np.ndarray) -> np.ndarray:
        return self.S @ np.asarray(v, dtype=np.float64)

    def dense(self) -> np.ndarray:
        return self.S
