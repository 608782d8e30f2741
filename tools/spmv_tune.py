"""SpMV variant timing on the config-4 operators (device time via the library's CUDA events)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from gen import make_problem
from paper_2605_22281_b200 import SFLSQR

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
if len(sys.argv) > 2:
    from gen.problems import CONFIGS
    CONFIGS[cfg] = dict(CONFIGS[cfg], tile=int(sys.argv[2]))
p = make_problem(cfg)
print("tile", p.geometry.get("tile"))
s = SFLSQR(maxit=4)
if p.t_mode == "given":
    s.set_operator(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, p.A.val, t=(p.T.rowptr, p.T.col, p.T.val))
else:
    s.set_operator(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, p.A.val)
info = s.get_info()
nnzA, nnzT = info["nnz_a"], info["nnz_t"]
rng = np.random.default_rng(0)
x, w = rng.standard_normal(p.n), rng.standard_normal(p.m)
ref = None
variants = [(m, 16) for m in (14, 3, 8, 10, 11, 12, 13, 15)]
for mode, sh in variants:
    s.debug_set_tuning(mode, sh)
    s.set_profiling(True)
    ya = s.debug_apply(0, x); yt = s.debug_apply(1, w)   # warm
    s.reset_profile()
    for _ in range(5):
        ya = s.debug_apply(0, x); yt = s.debug_apply(1, w)
    pr = s.get_profile()
    s.set_profiling(False)
    a, t = pr["spmv_A"], pr["spmv_T"]
    msa, mst = a["ms"] / a["launches"], t["ms"] / t["launches"]
    ba, bt = a["bytes"] / a["launches"], t["bytes"] / t["launches"]
    if ref is None:
        ref = (ya, yt)
    da = np.max(np.abs(ya - ref[0])) / np.max(np.abs(ref[0]))
    dt = np.max(np.abs(yt - ref[1])) / np.max(np.abs(ref[1]))
    print(json.dumps(dict(mode=mode, shift=sh, A_ms=round(msa, 4), A_GBs=round(ba / msa / 1e6, 1),
                          T_ms=round(mst, 4), T_GBs=round(bt / mst / 1e6, 1), dA=float(da), dT=float(dt))), flush=True)
s.close()
