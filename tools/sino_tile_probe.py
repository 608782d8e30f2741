"""Probe: Aᵀ w gather locality with a tiled sinogram layout of w (config 3).

The transposed Siddon operator's rows (pixels) gather w at ray indices a*nb + j: consecutive
entries are consecutive angles, one 128 B line each.  Storing w in (TA angles x TB bins) tiles
puts TA consecutive angles of nearby bins into one line.  Times T w for several tile shapes."""
import os
import sys
import json

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp

from gen import make_problem
from paper_2605_22281_b200 import SFLSQR

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = make_problem(cfg)
na, nb = p.geometry["n_angles"], p.geometry["nb"]
A = sp.csr_matrix((p.A.val, p.A.col, p.A.rowptr), shape=(p.m, p.n))
At = A.T.tocsr()
At.sort_indices()
rng = np.random.default_rng(0)
w = rng.standard_normal(p.m)


def tiled_perm(TA, TB):
    a, j = np.divmod(np.arange(p.m), nb)
    nbt = (nb + TB - 1) // TB
    tile = (a // TA) * nbt + (j // TB)
    within = (a % TA) * TB + (j % TB)
    key = tile * (TA * TB) + within
    return np.argsort(np.argsort(key, kind="stable"), kind="stable").astype(np.int64)  # rank of each ray


for TA, TB in [(1, 1), (4, 4), (8, 2), (2, 8), (16, 1), (8, 4)]:
    perm = tiled_perm(TA, TB)                         # ray i -> position perm[i]
    col = perm[At.indices].astype(np.int32)
    # keep entries of each row sorted by new position (summation order may change: compare to 1e-13)
    T = sp.csr_matrix((At.data.copy(), col, At.indptr.copy()), shape=At.shape)
    T.sort_indices()
    wp = np.empty(p.m)
    wp[perm] = w
    s = SFLSQR(maxit=4)
    s.set_operator(p.m, p.n, p.A.rowptr, p.A.col, p.A.val, t=(T.indptr.astype(np.int64), T.indices.astype(np.int32), T.data))
    s.set_profiling(True)
    y = s.debug_apply(1, wp)
    s.reset_profile()
    for _ in range(5):
        y = s.debug_apply(1, wp)
    pr = s.get_profile()["spmv_T"]
    ref = At @ w
    err = np.abs(y - ref).max() / np.abs(ref).max()
    print(json.dumps(dict(TA=TA, TB=TB, T_ms=round(pr["ms"] / pr["launches"], 4), err=float(err))), flush=True)
    s.close()
