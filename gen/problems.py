"""Workload recipes for BASELINE.json configs 1-5.

Every input is seeded and synthetic.  The paper's own images (``house``,
ASTRA Shepp-Logan phantoms) are not available;
these generators stand in for them at the shapes BASELINE.json fixes.

Seeds: master seed ``260522281 + config_index`` split by ``SeedSequence`` into the
named streams (A, xtrue, noise); sketch seed ``0x5F1A5D + config_index``.
Noise is scaled to its exact norm, ``e = g * delta*||A x_true|| / ||g||``
(reading R9; PAPER.md L50-54 defines delta = ||e|| / ||A x_true||).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsflsqr_gen.so")
_SRC = os.path.join(_HERE, "csrc", "gen.cpp")
_lib = None

MASTER_SEED = 260522281
SKETCH_SEED_BASE = 0x5F1A5D
LOWRANK_SEED_BASE = 0x10C0A5


def build_lib(force: bool = False) -> str:
    """Compile gen/csrc/gen.cpp into gen/libsflsqr_gen.so (g++, -O3, no FMA contraction)."""
    stale = (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)
    if force or stale:
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-shared", "-pthread", "-ffp-contract=off",
               _SRC, "-o", tmp]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _get_lib():
    global _lib
    if _lib is None:
        build_lib()
        lib = ctypes.CDLL(_LIB_PATH)
        i64p = ctypes.POINTER(ctypes.c_int64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        f64p = ctypes.POINTER(ctypes.c_double)
        ci = ctypes.c_int
        for nm in ("gen_siddon_rownnz", "gen_pixbp_rownnz"):
            getattr(lib, nm).argtypes = [ci, ci, ci, i64p, ci]
            getattr(lib, nm).restype = ci
        for nm in ("gen_siddon_fill", "gen_pixbp_fill"):
            getattr(lib, nm).argtypes = [ci, ci, ci, i64p, i32p, f64p, ci]
            getattr(lib, nm).restype = ci
        i64 = ctypes.c_int64
        for nm in ("gen_siddon_rownnz_range", "gen_pixbp_rownnz_range"):
            getattr(lib, nm).argtypes = [ci, ci, ci, ci, i64, i64, i64p, ci]
            getattr(lib, nm).restype = ci
        for nm in ("gen_siddon_fill_range", "gen_pixbp_fill_range"):
            getattr(lib, nm).argtypes = [ci, ci, ci, ci, i64, i64, i64p, i32p, f64p, ci]
            getattr(lib, nm).restype = ci
        lib.gen_csr_matvec.argtypes = [ctypes.c_int64, i64p, i32p, f64p, f64p, f64p, ci]
        lib.gen_csr_matvec.restype = ci
        _lib = lib
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


@dataclass
class CSR:
    """Canonical CSR: int64 rowptr (nrows+1), int32 col, float64 val."""
    nrows: int
    ncols: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def matvec(self, x: np.ndarray, nthreads: int = 0) -> np.ndarray:
        """Generator-side y = M x (used only to form b = A x_true)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.nrows, dtype=np.float64)
        _get_lib().gen_csr_matvec(self.nrows, _p(self.rowptr, ctypes.c_int64), _p(self.col, ctypes.c_int32),
                                  _p(self.val, ctypes.c_double), _p(x, ctypes.c_double),
                                  _p(y, ctypes.c_double), nthreads)
        return y

    @staticmethod
    def from_dense(M: np.ndarray) -> "CSR":
        M = np.asarray(M, dtype=np.float64)
        r, c = M.shape
        rowptr = np.arange(0, r * c + 1, c, dtype=np.int64)
        col = np.tile(np.arange(c, dtype=np.int32), r)
        return CSR(r, c, rowptr, col, np.ascontiguousarray(M.reshape(-1)))

    def to_dense(self) -> np.ndarray:
        D = np.zeros((self.nrows, self.ncols))
        for i in range(self.nrows):
            s, e = self.rowptr[i], self.rowptr[i + 1]
            D[i, self.col[s:e]] += self.val[s:e]
        return D


def _rowptr_from_counts(cnt: np.ndarray) -> np.ndarray:
    rp = np.zeros(cnt.size + 1, dtype=np.int64)
    np.cumsum(cnt, out=rp[1:])
    return rp


def siddon_csr(N: int, n_angles: int, nb: int, nthreads: int = 0, tile: int = 0) -> CSR:
    """Siddon ray-pixel intersection-length matrix, m = n_angles*nb rows, n = N*N columns
    (pixel order: row-major, or tile x tile tiles when tile > 0; reading R16)."""
    return _rows_block("siddon", N, n_angles, nb, 0, n_angles * nb, nthreads, tile)


def pixbp_csr(N: int, n_angles: int, nb: int, nthreads: int = 0, tile: int = 0) -> CSR:
    """Pixel-driven linear-interpolation backprojector B (n x m), B ~ A^T but unmatched."""
    return _rows_block("pixbp", N, n_angles, nb, 0, N * N, nthreads, tile)


def _rows_block(kind, N, n_angles, nb, r0, r1, nthreads=0, tile=0):
    """Rows [r0, r1) of the Siddon A (kind 'siddon') or the pixel-driven B ('pixbp') as a
    CSR block (local rowptr from 0, global columns) - the same rows make_problem builds."""
    lib = _get_lib()
    cnt = np.empty(r1 - r0, dtype=np.int64)
    f_cnt = lib.gen_siddon_rownnz_range if kind == "siddon" else lib.gen_pixbp_rownnz_range
    f_fill = lib.gen_siddon_fill_range if kind == "siddon" else lib.gen_pixbp_fill_range
    if f_cnt(N, tile, n_angles, nb, r0, r1, _p(cnt, ctypes.c_int64), nthreads) != 0:
        raise RuntimeError("row count failed")
    rp = _rowptr_from_counts(cnt)
    col = np.empty(int(rp[-1]), dtype=np.int32)
    val = np.empty(int(rp[-1]), dtype=np.float64)
    if f_fill(N, tile, n_angles, nb, r0, r1, _p(rp, ctypes.c_int64), _p(col, ctypes.c_int32),
              _p(val, ctypes.c_double), nthreads) != 0:
        raise RuntimeError("row fill failed")
    ncols = N * N if kind == "siddon" else n_angles * nb
    return CSR(r1 - r0, ncols, rp, col, val)


def row_nnz(kind, N, n_angles, nb, nthreads=0, tile=0):
    """Nonzeros of every row (for the nnz-balanced partition) without storing the matrix."""
    lib = _get_lib()
    nrows = n_angles * nb if kind == "siddon" else N * N
    cnt = np.empty(nrows, dtype=np.int64)
    f = lib.gen_siddon_rownnz_range if kind == "siddon" else lib.gen_pixbp_rownnz_range
    if f(N, tile, n_angles, nb, 0, nrows, _p(cnt, ctypes.c_int64), nthreads) != 0:
        raise RuntimeError("row count failed")
    return cnt


def tiled_order(N: int, tile: int) -> np.ndarray:
    """perm with x_tiled = x_rowmajor[perm] (tile x tile tiles, row-major tiles and interior)."""
    if tile <= 0:
        return np.arange(N * N)
    p = np.arange(N * N)
    tt, ntx = tile * tile, N // tile
    t, r = np.divmod(p, tt)
    iy = (t // ntx) * tile + r // tile
    ix = (t % ntx) * tile + r % tile
    return iy * N + ix


def ellipse_phantom(N: int, rng: np.random.Generator, n_ell: int = 10) -> np.ndarray:
    """Random-ellipse phantom (BASELINE.json configs 3-5; reading R15).

    Centres uniform-by-area in the inscribed disk, semi-axes U[0.02,0.6]*N/2,
    rotation U[0,pi), additive intensities U[-0.3,1]; sum, then clip >= 0.
    Returns the row-major vectorised image (n = N*N).
    """
    half = 0.5 * N
    c = np.arange(N, dtype=np.float64) + 0.5 - half
    X, Y = np.meshgrid(c, c)  # X varies along ix (columns), Y along iy (rows)
    img = np.zeros((N, N))
    for _ in range(n_ell):
        r = half * np.sqrt(rng.uniform())
        phi = 2.0 * np.pi * rng.uniform()
        cx, cy = r * np.cos(phi), r * np.sin(phi)
        a = rng.uniform(0.02, 0.6) * half
        b = rng.uniform(0.02, 0.6) * half
        rot = rng.uniform(0.0, np.pi)
        inten = rng.uniform(-0.3, 1.0)
        xr = (X - cx) * np.cos(rot) + (Y - cy) * np.sin(rot)
        yr = -(X - cx) * np.sin(rot) + (Y - cy) * np.cos(rot)
        img[(xr / a) ** 2 + (yr / b) ** 2 <= 1.0] += inten
    np.maximum(img, 0.0, out=img)
    return img.reshape(-1)


def rect_image(N: int, rng: np.random.Generator, n_rect: int = 4) -> np.ndarray:
    """Piecewise-constant N x N image: n_rect axis-aligned rectangles, values U[0,1],
    overwritten in order on a zero background (config 1; reading R15)."""
    img = np.zeros((N, N))
    for _ in range(n_rect):
        y0, y1 = np.sort(rng.integers(0, N, size=2))
        x0, x1 = np.sort(rng.integers(0, N, size=2))
        img[y0:y1 + 1, x0:x1 + 1] = rng.uniform(0.0, 1.0)
    return img.reshape(-1)


def star_field(N: int, rng: np.random.Generator, frac: float = 0.02) -> np.ndarray:
    """Sparse star field: round(frac*n) distinct pixels with values U[0.5,1] (config 2)."""
    n = N * N
    k = int(round(frac * n))
    x = np.zeros(n)
    idx = rng.choice(n, size=k, replace=False)
    x[idx] = rng.uniform(0.5, 1.0, size=k)
    return x


def gen_blur_taps(sigma: float, radius: int) -> np.ndarray:
    t = np.arange(-radius, radius + 1, dtype=np.float64)
    g = np.exp(-t * t / (2.0 * sigma * sigma))
    return g / g.sum()


def gen_blur_apply(x: np.ndarray, H: int, W: int, sigma: float, radius: int) -> np.ndarray:
    """Generator-side separable Gaussian blur, zero boundary (used only to form b)."""
    from scipy.ndimage import correlate1d
    g = gen_blur_taps(sigma, radius)
    X = x.reshape(H, W)
    Y = correlate1d(X, g, axis=1, mode="constant", cval=0.0)
    Y = correlate1d(Y, g, axis=0, mode="constant", cval=0.0)
    return Y.reshape(-1)


def lowrank_image(N: int, rng: np.random.Generator, n_rect: int = 12) -> np.ndarray:
    """Synthetic stand-in for the `house` image (config 8): a smooth separable background plus
    n_rect additive axis-aligned rectangles (rank <= n_rect + 1), row-major."""
    t = np.linspace(0.0, 1.0, N)
    img = 0.2 * np.outer(0.5 + 0.5 * np.sin(np.pi * t), 0.5 + 0.5 * np.cos(0.5 * np.pi * t))
    for _ in range(n_rect):
        y0, y1 = np.sort(rng.integers(0, N, size=2))
        x0, x1 = np.sort(rng.integers(0, N, size=2))
        img[y0:y1 + 1, x0:x1 + 1] += rng.uniform(0.1, 0.5)
    return img.reshape(-1)


def blur_mask_csr(N: int, sigma: float, radius: int, keep: np.ndarray) -> CSR:
    """Rows `keep` of the zero-boundary separable Gaussian blur of an N x N image (row-major):
    blurring composed with subsampling."""
    g = gen_blur_taps(sigma, radius)
    iy, ix = keep // N, keep % N
    cols, vals, cnt = [], [], np.zeros(keep.size, dtype=np.int64)
    offs = [(dy, dx) for dy in range(-radius, radius + 1) for dx in range(-radius, radius + 1)]
    for dy, dx in offs:
        yy, xx = iy + dy, ix + dx
        ok = (yy >= 0) & (yy < N) & (xx >= 0) & (xx < N)
        cols.append(np.where(ok, yy * N + xx, -1))
        vals.append(np.full(keep.size, g[dy + radius] * g[dx + radius]))
    C = np.stack(cols, axis=1)
    V = np.stack(vals, axis=1)
    ok = C >= 0
    cnt = ok.sum(axis=1)
    rowptr = np.zeros(keep.size + 1, dtype=np.int64)
    np.cumsum(cnt, out=rowptr[1:])
    return CSR(keep.size, N * N, rowptr, C[ok].astype(np.int32), np.ascontiguousarray(V[ok]))


@dataclass
class SolverSpec:
    method: str          # "sflsqr" | "sflsmr"
    maxit: int
    window: int          # orthogonalisation window ell
    d: int               # sketch rows
    s_nz: int            # nonzeros per sketch column
    precond: str         # "irn" | "nonneg" | "identity"
    p: float = 1.0       # IRN exponent (l_p prior)
    eps_rel: float = 1e-3
    eta: float = 0.0     # discrepancy safety factor (0 = off)
    tol: float = 0.0
    orth_mode: str = "P"
    sketch: str = "sparse"   # "sparse" (sparse-sign, R5/R6) | "gaussian" (dense N(0, 1/d), R21)
    lowrank: Optional[dict] = None  # tau_r setup for precond "lowrank" / "lowrank_rnd": N, r, oversample, seed


@dataclass
class Problem:
    name: str
    config_index: int
    m: int
    n: int
    A: Optional[CSR]                 # None for the matrix-free blur
    T: Optional[CSR]                 # given transpose-side operator (B) or None
    t_mode: str                      # "build" (A^T) | "given" (B) | "same" (symmetric blur)
    blur: Optional[dict]
    x_true: np.ndarray
    b: np.ndarray
    e: np.ndarray
    delta: float
    delta_e: float
    sketch_seed: int
    solvers: list = field(default_factory=list)
    geometry: dict = field(default_factory=dict)


CONFIGS = {
    1: dict(name="c1_dense256", kind="dense", N=16, delta=0.01,
            solvers=[("sflsqr", 40, 2, 80, 4, "irn", 1.01), ("sflsmr", 40, 2, 80, 4, "irn", 1.01)]),
    2: dict(name="c2_blur256", kind="blur", N=256, sigma=2.5, radius=7, delta=0.01,
            solvers=[("sflsqr", 100, 3, 200, 8, "irn", 0.0)]),
    3: dict(name="c3_ct512", kind="ct", N=512, n_angles=360, nb=725, delta=0.02, matched=True, tile=4,
            solvers=[("sflsqr", 150, 3, 300, 8, "nonneg", 0.0), ("sflsmr", 150, 3, 300, 8, "nonneg", 0.0)]),
    4: dict(name="c4_ct1024_unmatched", kind="ct", N=1024, n_angles=720, nb=1449, delta=0.01, matched=False, tile=4,
            solvers=[("sflsqr", 200, 4, 400, 8, "identity", 0.0)]),
    5: dict(name="c5_ct2048", kind="ct", N=2048, n_angles=1440, nb=2897, delta=0.01, matched=True, tile=4,
            solvers=[("sflsqr", 300, 5, 600, 8, "irn", 0.0), ("sflsmr", 300, 5, 600, 8, "irn", 0.0)]),
    # the paper's synthetic family:
    # A 1024 x 512 with singular values rho^(1-i), rho = 1.01, x_true = ones, ||b_true|| = 1,
    # white noise ||e|| = delta in {1%, 10%}; Gaussian sketch with s = 2k + 1 rows (k = maxit
    # = 50, not stated in the paper); sLSQR / sLSMR = sFLSQR / sFLSMR with tau = id and no
    # truncation (full window, L1150-1152).
    6: dict(name="c6_decay_rho1.01_noise1", kind="decay", m=1024, n=512, rho=1.01, delta=0.01, sketch="gaussian",
            solvers=[("sflsqr", 50, 50, 101, 1, "identity", 0.0), ("sflsmr", 50, 50, 101, 1, "identity", 0.0)]),
    # deblurring + inpainting with low-rank truncation (PAPER.md L98-109,
    # L1601-1636): 512 x 512 image, Gaussian PSF of variance 0.25 (sigma 0.5 px, 5 x 5, zero
    # boundary), half of the pixels dropped (rows removed), 5 % noise; 50 iterations, rank r = 30,
    # CountSketch with d = 101.  The `house` image is missing: a synthetic low-rank image (sum of
    # rectangles on a smooth separable background) stands in (reading R22).
    8: dict(name="c8_deblur_inpaint512", kind="inpaint", N=512, sigma=0.5, radius=2, keep=0.5, delta=0.05,
            lowrank=dict(r=30, oversample=10),
            solvers=[("sflsqr", 50, 3, 101, 1, "lowrank_rnd", 0.0), ("sflsmr", 50, 3, 101, 1, "lowrank_rnd", 0.0)]),
    7: dict(name="c7_decay_rho1.01_noise10", kind="decay", m=1024, n=512, rho=1.01, delta=0.10, sketch="gaussian",
            solvers=[("sflsqr", 50, 50, 101, 1, "identity", 0.0), ("sflsmr", 50, 50, 101, 1, "identity", 0.0)]),
}


def make_problem(config_index: int, N: Optional[int] = None, n_angles: Optional[int] = None,
                 nb: Optional[int] = None, nthreads: int = 0, seed_offset: int = 0) -> Problem:
    """Build the seeded problem for a BASELINE.json config (1-based index).

    ``N``/``n_angles``/``nb`` override the geometry to produce reduced-size
    variants of the same recipe (parity tests); defaults are BASELINE.json's.
    """
    cfg = CONFIGS[config_index]
    ss = np.random.SeedSequence(MASTER_SEED + config_index + seed_offset)
    s_A, s_x, s_e = ss.spawn(3)
    rA, rx, re = (np.random.Generator(np.random.PCG64(s)) for s in (s_A, s_x, s_e))
    kind = cfg["kind"]
    geometry = {}
    A = T = None
    blur = None
    if kind == "dense":
        Nimg = N or cfg["N"]
        n = Nimg * Nimg
        U = np.linalg.qr(rA.standard_normal((n, n)))[0]
        V = np.linalg.qr(rA.standard_normal((n, n)))[0]
        sig = 10.0 ** (-6.0 * np.arange(n) / (n - 1))
        Ad = (U * sig) @ V.T
        A = CSR.from_dense(Ad)
        t_mode = "build"
        x_true = rect_image(Nimg, rx)
        m = n
        geometry = dict(N=Nimg, sigma_min=float(sig[-1]))
        Ax = A.matvec(x_true)
    elif kind == "blur":
        Nimg = N or cfg["N"]
        n = m = Nimg * Nimg
        blur = dict(H=Nimg, W=Nimg, sigma=cfg["sigma"], radius=cfg["radius"])
        t_mode = "same"
        x_true = star_field(Nimg, rx)
        geometry = dict(N=Nimg)
        Ax = gen_blur_apply(x_true, Nimg, Nimg, cfg["sigma"], cfg["radius"])
    elif kind == "ct":
        Nimg = N or cfg["N"]
        na = n_angles or cfg["n_angles"]
        nbins = nb or cfg["nb"]
        tile = cfg.get("tile", 0) if Nimg % max(cfg.get("tile", 1), 1) == 0 else 0
        A = siddon_csr(Nimg, na, nbins, nthreads, tile)
        if cfg["matched"]:
            t_mode = "build"
        else:
            T = pixbp_csr(Nimg, na, nbins, nthreads, tile)
            t_mode = "given"
        m, n = A.nrows, A.ncols
        x_true = ellipse_phantom(Nimg, rx)[tiled_order(Nimg, tile)]
        geometry = dict(N=Nimg, n_angles=na, nb=nbins, tile=tile)
        Ax = A.matvec(x_true, nthreads)
    elif kind == "inpaint":
        Nimg = N or cfg["N"]
        n = Nimg * Nimg
        keep = np.sort(rA.choice(n, size=int(round(cfg["keep"] * n)), replace=False))
        A = blur_mask_csr(Nimg, cfg["sigma"], cfg["radius"], keep)
        t_mode = "build"
        m = A.nrows
        x_true = lowrank_image(Nimg, rx)
        geometry = dict(N=Nimg, keep=cfg["keep"], sigma=cfg["sigma"])
        Ax = A.matvec(x_true)
    elif kind == "decay":
        m, n = cfg["m"], cfg["n"]
        U = np.linalg.qr(rA.standard_normal((m, n)))[0]
        V = np.linalg.qr(rA.standard_normal((n, n)))[0]
        sig = cfg["rho"] ** (-np.arange(n, dtype=np.float64))          # rho^(1-i), i = 1..n
        Ad = (U * sig) @ V.T
        x_true = np.ones(n)
        Ad = Ad / np.linalg.norm(Ad @ x_true)                           # ||b_true|| = 1 (L546)
        A = CSR.from_dense(Ad)
        t_mode = "build"
        geometry = dict(rho=cfg["rho"], sigma_min=float(sig[-1]))
        Ax = A.matvec(x_true)
    else:
        raise ValueError(kind)
    g = re.standard_normal(m)
    e = g * (cfg["delta"] * np.linalg.norm(Ax) / np.linalg.norm(g))
    b = Ax + e
    lowrank = None
    if "lowrank" in cfg:
        lowrank = dict(cfg["lowrank"], N=geometry["N"], seed=LOWRANK_SEED_BASE + config_index)
    solvers = [SolverSpec(method=s[0], maxit=s[1], window=s[2], d=s[3], s_nz=s[4], precond=s[5], eta=s[6],
                          sketch=cfg.get("sketch", "sparse"), lowrank=lowrank)
               for s in cfg["solvers"]]
    return Problem(name=cfg["name"], config_index=config_index, m=m, n=n, A=A, T=T, t_mode=t_mode,
                   blur=blur, x_true=x_true, b=b, e=e, delta=cfg["delta"], delta_e=float(np.linalg.norm(e)),
                   sketch_seed=SKETCH_SEED_BASE + config_index, solvers=solvers, geometry=geometry)


@dataclass
class ShardProblem:
    """One rank's share of a CT config: its A row block (and B row block), its slice
    of b, and the global metadata (the multi-GPU bench)."""
    name: str
    config_index: int
    m: int
    n: int
    a_rows: tuple
    t_rows: Optional[tuple]
    A_loc: CSR
    T_loc: Optional[CSR]
    t_mode: str
    b_loc: np.ndarray
    delta_e: float
    sketch_seed: int
    solvers: list


def _ct_geometry(cfg, N=None, n_angles=None, nb=None):
    Nimg = N or cfg["N"]
    tile = cfg.get("tile", 0) if Nimg % max(cfg.get("tile", 1), 1) == 0 else 0
    return Nimg, n_angles or cfg["n_angles"], nb or cfg["nb"], tile


def ct_row_nnz(config_index: int, nthreads: int = 0, N=None, n_angles=None, nb=None):
    """Row lengths of A (and B when unmatched) for the nnz-balanced partition (geometry overrides
    as in make_problem)."""
    cfg = CONFIGS[config_index]
    Nimg, na, nbins, tile = _ct_geometry(cfg, N, n_angles, nb)
    a = row_nnz("siddon", Nimg, na, nbins, nthreads, tile)
    t = None if cfg["matched"] else row_nnz("pixbp", Nimg, na, nbins, nthreads, tile)
    return a, t


def make_ct_shard(config_index: int, a_rows: tuple, t_rows: Optional[tuple], allreduce_sum,
                  nthreads: int = 0, N=None, n_angles=None, nb=None) -> ShardProblem:
    """The rows [a_rows) of A (and [t_rows) of B) of make_problem(config_index), and the
    matching slice of b = A x_true + e.  The same seeded streams as make_problem;
    ||A x_true|| is the allreduce of the ranks' partial squares (allreduce_sum(float))."""
    cfg = CONFIGS[config_index]
    if cfg["kind"] != "ct":
        raise ValueError("sharded generation is for the CT configs")
    N, na, nb, tile = _ct_geometry(cfg, N, n_angles, nb)
    ss = np.random.SeedSequence(MASTER_SEED + config_index)
    s_A, s_x, s_e = ss.spawn(3)
    rx, re = (np.random.Generator(np.random.PCG64(s)) for s in (s_x, s_e))
    m, n = na * nb, N * N
    A_loc = _rows_block("siddon", N, na, nb, a_rows[0], a_rows[1], nthreads, tile)
    T_loc = None
    t_mode = "build"
    if not cfg["matched"]:
        T_loc = _rows_block("pixbp", N, na, nb, t_rows[0], t_rows[1], nthreads, tile)
        t_mode = "given"
    x_true = ellipse_phantom(N, rx)[tiled_order(N, tile)]
    Ax_loc = A_loc.matvec(x_true, nthreads)
    norm_ax = float(np.sqrt(allreduce_sum(float(Ax_loc @ Ax_loc))))
    g = re.standard_normal(m)
    scale = cfg["delta"] * norm_ax / np.linalg.norm(g)
    b_loc = Ax_loc + g[a_rows[0]:a_rows[1]] * scale
    solvers = [SolverSpec(method=s[0], maxit=s[1], window=s[2], d=s[3], s_nz=s[4], precond=s[5], eta=s[6])
               for s in cfg["solvers"]]
    return ShardProblem(name=cfg["name"], config_index=config_index, m=m, n=n, a_rows=tuple(a_rows),
                        t_rows=None if t_rows is None else tuple(t_rows), A_loc=A_loc, T_loc=T_loc, t_mode=t_mode,
                        b_loc=b_loc, delta_e=cfg["delta"] * norm_ax, sketch_seed=SKETCH_SEED_BASE + config_index,
                        solvers=solvers)
