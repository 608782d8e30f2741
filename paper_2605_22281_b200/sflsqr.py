"""Thin ctypes binding of libsflsqr.so (include/sflsqr.h).

Argument marshalling only: every step of the method runs in the library's
CUDA kernels.  Method names mirror the C ABI without the ``sflsqr_`` prefix.
Arrays may be NumPy (host) or CUDA ``torch.Tensor`` (device; passed by
pointer with SFLSQR_MEM_DEVICE).  PyTorch supplies the stream
(``torch.cuda.current_stream()``) when it is importable with CUDA.

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from ._build import LIB_PATH

OK = 0
E_INVALID, E_DIM, E_NONFINITE, E_ZERO_RHS, E_STATE, E_CUDA, E_OOM, E_UNSUPPORTED = -1, -2, -3, -4, -5, -6, -7, -8
METHOD_SFLSQR, METHOD_SFLSMR, METHOD_FLSQR, METHOD_FLSMR, METHOD_LSQR, METHOD_LSMR = 0, 1, 2, 3, 4, 5
METHODS = {"sflsqr": METHOD_SFLSQR, "sflsmr": METHOD_SFLSMR, "flsqr": METHOD_FLSQR, "flsmr": METHOD_FLSMR,
           "lsqr": METHOD_LSQR, "lsmr": METHOD_LSMR}
ORTH_P, ORTH_Z = 0, 1
ORTHK_AUTO, ORTHK_MGS = 0, 1
RUNNING, MAXIT, TOL, DISCREPANCY, BREAKDOWN = 0, 1, 2, 3, 4
PRECOND_IDENTITY, PRECOND_IRN, PRECOND_NONNEG, PRECOND_LOWRANK_RND = 0, 1, 2, 3
T_BUILD, T_GIVEN = 0, 1
MEM_HOST, MEM_DEVICE, MEM_BORROW = 0, 1, 2
X_GATHERED = 4          # sflsqr_get_x: the whole x, all-gathered over the ranks
HIST_TRUE_RES = 1
KC_NAMES = ["spmv_A", "spmv_T", "orth", "tau", "sketch", "ls", "xupd", "res", "stop"]

EXPORTED = [
    "sflsqr_version", "sflsqr_create", "sflsqr_get_unique_id", "sflsqr_debug_nccl_selftest", "sflsqr_local_group_create",
    "sflsqr_local_group_destroy", "sflsqr_set_operator_shard", "sflsqr_set_operator", "sflsqr_set_operator_blur", "sflsqr_set_sketch",
    "sflsqr_set_precond", "sflsqr_set_rhs", "sflsqr_iterate", "sflsqr_get_x", "sflsqr_get_residual_norms",
    "sflsqr_get_info", "sflsqr_debug_sketch_table", "sflsqr_debug_apply", "sflsqr_debug_basis", "sflsqr_debug_state",
    "sflsqr_debug_set_tuning", "sflsqr_set_sketch_gaussian", "sflsqr_debug_sketch_dense",
    "sflsqr_set_precond_lowrank",
    "sflsqr_set_profiling", "sflsqr_reset_profile", "sflsqr_get_profile", "sflsqr_last_error", "sflsqr_destroy",
]


COMM_NCCL, COMM_LOCAL, COMM_IPC = 0, 1, 2

# opts.knobs (include/sflsqr.h SFLSQR_KNOB_*): scheduling / storage-format switches, 0 = defaults
KNOBS = {"no_pdl": 0x1, "sketch_main": 0x2, "no_interp": 0x4, "no_sell": 0x8, "cgs_always2": 0x10,
         "full_spmv_grid": 0x20, "res_main": 0x40, "res_side": 0x80, "p2p_on": 0x100, "p2p_off": 0x200,
         "keep_csr": 0x400, "debug_poison": 0x800, "no_ell_c16": 0x1000, "half_warp_rows": 0x2000,
         "tma": 0x4000, "wnorm_sep": 0x8000}


def knob_bits(knobs):
    """int bits, or an iterable of names of KNOBS."""
    if knobs is None:
        return 0
    if isinstance(knobs, int):
        return knobs
    bits = 0
    for k in knobs:
        bits |= KNOBS[k]
    return bits


class Opts(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int32), ("window", ctypes.c_int32), ("maxit", ctypes.c_int32),
                ("orth_mode", ctypes.c_int32), ("tol", ctypes.c_double), ("eta", ctypes.c_double),
                ("delta_e", ctypes.c_double), ("history", ctypes.c_int32), ("device", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("use_graph", ctypes.c_int32), ("comm_kind", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("local_group", ctypes.c_void_p), ("orth_kernel", ctypes.c_int32), ("knobs", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 2)]


class Info(ctypes.Structure):
    _fields_ = [("k_done", ctypes.c_int32), ("k_x", ctypes.c_int32), ("status", ctypes.c_int32),
                ("rank_flag", ctypes.c_int32), ("m", ctypes.c_int64), ("n", ctypes.c_int64),
                ("nnz_a", ctypes.c_int64), ("nnz_t", ctypes.c_int64), ("launches", ctypes.c_int64),
                ("beta", ctypes.c_double), ("m0", ctypes.c_int64), ("m_loc", ctypes.c_int64),
                ("n0", ctypes.c_int64), ("n_loc", ctypes.c_int64), ("delta_e", ctypes.c_double),
                ("bytes_model", ctypes.c_double), ("a_pairs", ctypes.c_int64), ("t_pairs", ctypes.c_int64),
                ("a_fmt", ctypes.c_int32), ("t_fmt", ctypes.c_int32), ("knobs", ctypes.c_int32),
                ("csr_kept", ctypes.c_int32), ("graph", ctypes.c_int32), ("reserved_i", ctypes.c_int32)]


class Profile(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 9), ("launches", ctypes.c_int64 * 9), ("bytes", ctypes.c_double * 9)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libsflsqr.so (raises OSError if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"{path} not found: run __graft_entry__.build() (no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    vp, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "sflsqr_version": ([], ctypes.c_int),
        "sflsqr_create": ([ctypes.POINTER(vp), ctypes.POINTER(Opts)], ctypes.c_int),
        "sflsqr_set_operator": ([vp, i64, i64, vp, vp, vp, i32, vp, vp, vp, i32], ctypes.c_int),
        "sflsqr_set_operator_shard": ([vp, i64, i64, i64, i64, vp, vp, vp, i32, i64, i64, vp, vp, vp], ctypes.c_int),
        "sflsqr_get_unique_id": ([vp], ctypes.c_int),
        "sflsqr_debug_nccl_selftest": ([i32], ctypes.c_int),
        "sflsqr_local_group_create": ([ctypes.POINTER(vp), i32, i32], ctypes.c_int),
        "sflsqr_local_group_destroy": ([vp], None),
        "sflsqr_set_operator_blur": ([vp, i32, i32, f64, i32], ctypes.c_int),
        "sflsqr_set_sketch": ([vp, ctypes.c_uint64, i32, i32], ctypes.c_int),
        "sflsqr_set_sketch_gaussian": ([vp, ctypes.c_uint64, i32], ctypes.c_int),
        "sflsqr_set_precond_lowrank": ([vp, i32, i32, i32, i32, ctypes.c_uint64], ctypes.c_int),
        "sflsqr_debug_sketch_dense": ([vp, i64, i64, vp], ctypes.c_int),
        "sflsqr_set_precond": ([vp, i32, f64, f64], ctypes.c_int),
        "sflsqr_set_rhs": ([vp, vp, i64, i32], ctypes.c_int),
        "sflsqr_iterate": ([vp, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)], ctypes.c_int),
        "sflsqr_get_x": ([vp, vp, i64, i32], ctypes.c_int),
        "sflsqr_get_residual_norms": ([vp, vp, vp, i64, ctypes.POINTER(i64)], ctypes.c_int),
        "sflsqr_get_info": ([vp, ctypes.POINTER(Info)], ctypes.c_int),
        "sflsqr_debug_sketch_table": ([vp, i64, i64, vp, vp], ctypes.c_int),
        "sflsqr_debug_apply": ([vp, i32, vp, vp], ctypes.c_int),
        "sflsqr_debug_basis": ([vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "sflsqr_debug_state": ([vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "sflsqr_debug_set_tuning": ([vp, i32, i32], ctypes.c_int),
        "sflsqr_set_profiling": ([vp, i32], ctypes.c_int),
        "sflsqr_reset_profile": ([vp], ctypes.c_int),
        "sflsqr_get_profile": ([vp, ctypes.POINTER(Profile)], ctypes.c_int),
        "sflsqr_last_error": ([vp], ctypes.c_char_p),
        "sflsqr_destroy": ([vp], None),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


class SflsqrError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"libsflsqr error {code}: {msg}")
        self.code = code


def _ptr(a):
    """(pointer, is_device, keepalive) for a numpy array or torch tensor (or None)."""
    if a is None:
        return None, False, None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            a = np.ascontiguousarray(a)
        return a.ctypes.data, False, a
    mod = type(a).__module__
    if mod.startswith("torch"):
        if not a.is_contiguous():
            a = a.contiguous()
        return a.data_ptr(), bool(a.is_cuda), a
    raise TypeError(f"unsupported array type {type(a)}")


def _torch_stream(device):
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream(device).cuda_stream
    except Exception:
        pass
    return None


class SFLSQR:
    """One solver handle (sflsqr_create ... sflsqr_destroy)."""

    def __init__(self, method="sflsqr", window=2, maxit=10, orth_mode="P", tol=0.0, eta=0.0, delta_e=0.0,
                 history=HIST_TRUE_RES, device=0, stream=None, use_graph=True, rank=0, world=1, nccl_id=None,
                 local_group=None, orth_kernel="auto", knobs=0, ipc_name=None):
        self.lib = load_library()
        o = Opts()
        o.knobs = knob_bits(knobs)
        o.method = METHODS.get(method, -1)
        o.orth_kernel = ORTHK_MGS if orth_kernel == "mgs" else ORTHK_AUTO
        o.window, o.maxit = int(window), int(maxit)
        o.orth_mode = ORTH_P if orth_mode == "P" else ORTH_Z
        o.tol, o.eta, o.delta_e = float(tol), float(eta), float(delta_e)
        o.history, o.device = int(history), int(device)
        # NULL / the legacy default stream -> the library creates its own non-blocking stream
        o.stream = stream if stream is not None else _torch_stream(device)
        o.rank, o.world, o.use_graph = int(rank), int(world), 1 if use_graph else 0
        self._id_buf = None
        if int(world) > 1:
            if local_group is not None:
                o.comm_kind, o.local_group = COMM_LOCAL, local_group.ptr
            elif ipc_name is not None:
                # SFLSQR_COMM_IPC: process ranks, POSIX shm rendezvous + CUDA-IPC peer memory
                o.comm_kind = COMM_IPC
                self._id_buf = ctypes.create_string_buffer(str(ipc_name).encode(), 128)
                o.nccl_id = ctypes.addressof(self._id_buf)
            else:
                o.comm_kind = COMM_NCCL
                self._id_buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
                o.nccl_id = ctypes.addressof(self._id_buf)
        self.maxit = int(maxit)
        h = ctypes.c_void_p()
        rc = self.lib.sflsqr_create(ctypes.byref(h), ctypes.byref(o))
        if rc != OK:
            raise SflsqrError(rc, self.lib.sflsqr_last_error(None).decode())
        self.h = h
        self._keep = []
        self.m = self.n = None

    # ------------------------------------------------------------------
    def _check(self, rc):
        if rc != OK:
            raise SflsqrError(rc, self.lib.sflsqr_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.sflsqr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------------ ABI mirrors
    def set_operator(self, m, n, a_rowptr, a_col, a_val, t=None, borrow=False):  # noqa: D401
        """t = None -> T_BUILD (A^T formed by the library); t = (rowptr, col, val) -> T_GIVEN."""
        pa = [_ptr(x) for x in (a_rowptr, a_col, a_val)]
        dev = pa[0][1]
        if t is None:
            pt = [(None, dev, None)] * 3
            mode = T_BUILD
        else:
            pt = [_ptr(x) for x in t]
            mode = T_GIVEN
        flags = (MEM_DEVICE if dev else MEM_HOST) | (MEM_BORROW if borrow else 0)
        if borrow:
            self._keep += [p[2] for p in pa + pt]
        self._check(self.lib.sflsqr_set_operator(self.h, int(m), int(n), pa[0][0], pa[1][0], pa[2][0], mode,
                                                 pt[0][0], pt[1][0], pt[2][0], flags))
        self.m, self.n = int(m), int(n)

    def set_operator_shard(self, m, n, a_row0, a_row1, a_rowptr, a_col, a_val, t=None, t_rows=(0, 0)):
        """This rank's block of A rows [a_row0, a_row1) (local rowptr, global columns); t = None ->
        COLSHARD (T = (A block)^T built locally), t = (rowptr, col, val) of T rows t_rows -> ROWSHARD."""
        pa = [_ptr(np.ascontiguousarray(x)) for x in (a_rowptr, a_col, a_val)]
        if t is None:
            pt, mode = [(None, False, None)] * 3, T_BUILD
        else:
            pt, mode = [_ptr(np.ascontiguousarray(x)) for x in t], T_GIVEN
        self._check(self.lib.sflsqr_set_operator_shard(self.h, int(m), int(n), int(a_row0), int(a_row1), pa[0][0],
                                                       pa[1][0], pa[2][0], mode, int(t_rows[0]), int(t_rows[1]),
                                                       pt[0][0], pt[1][0], pt[2][0]))
        inf = self.get_info()
        self.m_glob, self.n_glob = int(m), int(n)
        self.m, self.n = inf["m_loc"], inf["n_loc"]
        self.n_global = inf["n"]

    def set_operator_blur(self, H, W, sigma, radius):
        self._check(self.lib.sflsqr_set_operator_blur(self.h, int(H), int(W), float(sigma), int(radius)))
        self.m = self.n = int(H) * int(W)

    def set_sketch(self, seed, d, s_nz):
        self._check(self.lib.sflsqr_set_sketch(self.h, int(seed), int(d), int(s_nz)))

    def set_sketch_gaussian(self, seed, d):
        self._check(self.lib.sflsqr_set_sketch_gaussian(self.h, int(seed), int(d)))
        self._gauss_d = int(d)

    def debug_sketch_dense(self, col0, ncols):
        out = np.empty((self._gauss_d, int(ncols)))
        self._check(self.lib.sflsqr_debug_sketch_dense(self.h, int(col0), int(ncols), out.ctypes.data))
        return out

    def set_precond_lowrank(self, H, W, r, oversample=10, seed=0):
        self._check(self.lib.sflsqr_set_precond_lowrank(self.h, int(H), int(W), int(r), int(oversample), int(seed)))

    def set_precond(self, kind="identity", p=1.0, eps_rel=1e-3):
        k = {"identity": PRECOND_IDENTITY, "irn": PRECOND_IRN, "nonneg": PRECOND_NONNEG}.get(kind, kind)
        self._check(self.lib.sflsqr_set_precond(self.h, int(k), float(p), float(eps_rel)))

    def set_rhs(self, b):
        p, dev, keep = _ptr(b)
        n = b.numel() if hasattr(b, "numel") else b.size
        self._check(self.lib.sflsqr_set_rhs(self.h, p, int(n), MEM_DEVICE if dev else MEM_HOST))

    def iterate(self, k):
        done, status = ctypes.c_int32(), ctypes.c_int32()
        self._check(self.lib.sflsqr_iterate(self.h, int(k), ctypes.byref(done), ctypes.byref(status)))
        return bool(done.value), int(status.value)

    def get_x(self, out=None, gathered=False):
        """This rank's slice of x_k (the whole x on one rank); gathered=True: the whole x on every
        rank (a collective over the group)."""
        n = getattr(self, "n_global", self.n) if gathered else self.n
        if out is None:
            out = np.empty(n)
        p, dev, _ = _ptr(out)
        flags = (MEM_DEVICE if dev else MEM_HOST) | (X_GATHERED if gathered else 0)
        self._check(self.lib.sflsqr_get_x(self.h, p, int(n), flags))
        return out

    def get_residual_norms(self):
        cap = self.maxit
        tr, sk = np.empty(cap), np.empty(cap)
        cnt = ctypes.c_int64()
        self._check(self.lib.sflsqr_get_residual_norms(self.h, tr.ctypes.data, sk.ctypes.data, cap,
                                                       ctypes.byref(cnt)))
        c = int(cnt.value)
        return tr[:c].copy(), sk[:c].copy()

    def get_info(self):
        inf = Info()
        self._check(self.lib.sflsqr_get_info(self.h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in Info._fields_}

    def debug_sketch_table(self, col0, ncols, s_nz):
        rows = np.empty((ncols, s_nz), dtype=np.int32)
        signs = np.empty((ncols, s_nz), dtype=np.int8)
        self._check(self.lib.sflsqr_debug_sketch_table(self.h, int(col0), int(ncols), rows.ctypes.data,
                                                       signs.ctypes.data))
        return rows, signs

    def debug_apply(self, which, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.m if which == 0 else self.n)
        self._check(self.lib.sflsqr_debug_apply(self.h, int(which), x.ctypes.data, y.ctypes.data))
        return y

    def debug_basis(self):
        info = self.get_info()
        kd, kx = info["k_done"], info["k_x"]
        H = np.zeros((kd + 1, kd), order="F")
        Tm = np.zeros((kd, kd), order="F")
        Z = np.zeros((self.n, kd), order="F")
        W = np.zeros((self.m, kd + 1), order="F")
        y = np.zeros(kx)
        self._check(self.lib.sflsqr_debug_basis(self.h, H.ctypes.data, Tm.ctypes.data, Z.ctypes.data,
                                                W.ctypes.data, y.ctypes.data))
        return dict(H=H, T=Tm, Z=Z, W=W, y=y)

    def debug_state(self, window, d, method):
        info = self.get_info()
        kd = info["k_done"]
        z, x = np.zeros(self.n), np.zeros(self.n)
        ring = np.zeros((window, self.n))
        nc = kd if method == "sflsqr" else kd + 1 if method == "sflsmr" else 0
        cols = np.zeros((d, max(nc, 1)), order="F")
        rhs = np.zeros(d)
        self._check(self.lib.sflsqr_debug_state(self.h, z.ctypes.data, x.ctypes.data, ring.ctypes.data,
                                                cols.ctypes.data, rhs.ctypes.data))
        return dict(z=z, x=x, p_ring=ring, sketch_cols=cols[:, :nc], rhs=rhs)

    def debug_set_tuning(self, spmv_mode=-1, band_shift=16):
        self._check(self.lib.sflsqr_debug_set_tuning(self.h, int(spmv_mode), int(band_shift)))

    def set_profiling(self, on=True):
        self._check(self.lib.sflsqr_set_profiling(self.h, 1 if on else 0))

    def reset_profile(self):
        self._check(self.lib.sflsqr_reset_profile(self.h))

    def get_profile(self):
        p = Profile()
        self._check(self.lib.sflsqr_get_profile(self.h, ctypes.byref(p)))
        return {KC_NAMES[i]: dict(ms=p.ms[i], launches=int(p.launches[i]), bytes=p.bytes[i]) for i in range(9)}


def get_unique_id() -> bytes:
    """128-byte NCCL id (rank 0); broadcast it with the caller's process group."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    rc = lib.sflsqr_get_unique_id(buf)
    if rc != OK:
        raise SflsqrError(rc, lib.sflsqr_last_error(None).decode())
    return buf.raw


def nccl_selftest(device=0) -> None:
    """sflsqr_debug_nccl_selftest: the NCCL transport on a one-rank communicator, eagerly and captured."""
    lib = load_library()
    rc = lib.sflsqr_debug_nccl_selftest(int(device))
    if rc != OK:
        raise SflsqrError(rc, lib.sflsqr_last_error(None).decode())


class LocalGroup:
    """In-process rank group (SFLSQR_COMM_LOCAL): world handles on one device, one host thread each."""

    def __init__(self, world, device=0):
        self.lib = load_library()
        p = ctypes.c_void_p()
        rc = self.lib.sflsqr_local_group_create(ctypes.byref(p), int(world), int(device))
        if rc != OK:
            raise SflsqrError(rc, self.lib.sflsqr_last_error(None).decode())
        self.ptr, self.world = p.value, int(world)

    def close(self):
        if self.ptr:
            self.lib.sflsqr_local_group_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solver_for_problem(prob, spec, maxit=None, history=HIST_TRUE_RES, use_graph=True, eta=None, device=0,
                       operator_on_device=False, method=None, orth_kernel="auto", knobs=0):
    """Configure an SFLSQR handle for a gen.Problem / gen.SolverSpec (marshalling only).
    method overrides spec.method (e.g. "flsqr" / "flsmr" on a config's operator)."""
    mx = maxit or spec.maxit
    s = SFLSQR(method=method or spec.method, window=spec.window, maxit=mx, orth_mode=spec.orth_mode, tol=spec.tol,
               eta=spec.eta if eta is None else eta, delta_e=prob.delta_e, history=history, device=device,
               use_graph=use_graph, orth_kernel=orth_kernel, knobs=knobs)
    if prob.t_mode == "same":
        bl = prob.blur
        s.set_operator_blur(bl["H"], bl["W"], bl["sigma"], bl["radius"])
    else:
        A = prob.A
        t = None if prob.t_mode == "build" else (prob.T.rowptr, prob.T.col, prob.T.val)
        s.set_operator(A.nrows, A.ncols, A.rowptr, A.col, A.val, t=t)
    if getattr(spec, "sketch", "sparse") == "gaussian":
        s.set_sketch_gaussian(prob.sketch_seed, spec.d)
    else:
        s.set_sketch(prob.sketch_seed, spec.d, spec.s_nz)
    if (method or spec.method) in ("lsqr", "lsmr"):
        s.set_precond("identity")          # GKB methods take no flexible preconditioner
    elif spec.precond == "lowrank_rnd":
        lr = spec.lowrank
        s.set_precond_lowrank(lr["N"], lr["N"], lr["r"], lr["oversample"], lr["seed"])
    else:
        s.set_precond(spec.precond, spec.p, spec.eps_rel)
    return s


def _csr_arrays(M):
    """(nrows, ncols, rowptr int64, col int32, val float64) of a scipy.sparse matrix or a
    (rowptr, col, val, shape) tuple."""
    if hasattr(M, "tocsr"):
        C = M.tocsr()
        return (C.shape[0], C.shape[1], np.ascontiguousarray(C.indptr, dtype=np.int64),
                np.ascontiguousarray(C.indices, dtype=np.int32), np.ascontiguousarray(C.data, dtype=np.float64))
    rowptr, col, val, shape = M
    return (int(shape[0]), int(shape[1]), np.ascontiguousarray(rowptr, dtype=np.int64),
            np.ascontiguousarray(col, dtype=np.int32), np.ascontiguousarray(val, dtype=np.float64))


def solve(A, b, method="sflsqr", T=None, maxit=50, window=3, sketch=("sparse", None, 8, 0), precond="identity",
          p=1.0, eps_rel=1e-3, lowrank=None, tol=0.0, eta=0.0, delta_e=0.0, orth_mode="P", device=0,
          use_graph=True):
    """One-call solve through the C ABI (argument marshalling only).

    A: scipy.sparse matrix or (rowptr, col, val, (m, n)); T: the transpose-side operator B ~ A^T
    in the same forms (None: A^T formed by the library).  method: sflsqr | sflsmr | flsqr | flsmr |
    lsqr | lsmr.  sketch: ("sparse", d, s_nz, seed) or ("gaussian", d, seed); d = None -> 2 maxit + 1.
    precond: identity | irn | nonneg | lowrank_rnd (lowrank = dict(H, W, r, oversample, seed)).
    Returns dict(x, status, k, true_res, sketch_res, info)."""
    m, n, rp, col, val = _csr_arrays(A)
    s = SFLSQR(method=method, window=window, maxit=maxit, orth_mode=orth_mode, tol=tol, eta=eta, delta_e=delta_e,
               device=device, use_graph=use_graph)
    try:
        if T is None:
            s.set_operator(m, n, rp, col, val)
        else:
            tn, tm, trp, tcol, tval = _csr_arrays(T)
            if (tn, tm) != (n, m):
                raise ValueError("T must be n x m")
            s.set_operator(m, n, rp, col, val, t=(trp, tcol, tval))
        if method in ("sflsqr", "sflsmr"):
            kind = sketch[0]
            d = sketch[1] if sketch[1] is not None else 2 * maxit + 1
            if kind == "gaussian":
                s.set_sketch_gaussian(sketch[2] if len(sketch) > 2 else 0, d)
            else:
                s.set_sketch(sketch[3] if len(sketch) > 3 else 0, d, sketch[2])
        if precond == "lowrank_rnd":
            lr = lowrank or {}
            s.set_precond_lowrank(lr["H"], lr["W"], lr["r"], lr.get("oversample", 10), lr.get("seed", 0))
        else:
            s.set_precond(precond, p, eps_rel)
        s.set_rhs(np.ascontiguousarray(b, dtype=np.float64))
        done, status = s.iterate(maxit)
        tr, sk = s.get_residual_norms()
        info = s.get_info()
        x = s.get_x()
    finally:
        s.close()
    return dict(x=x, status=status, k=info["k_x"], true_res=tr, sketch_res=sk, info=info)
