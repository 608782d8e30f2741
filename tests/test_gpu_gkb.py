"""GPU parity of textbook LSQR / LSMR (methods 4 / 5; PAPER.md
L277-319) through the C ABI against the fp64 oracle (oracle/gkb.py, pinned in
tests/test_oracle_gkb.py).

Bar: the recurrence residual histories (and LSMR's ||T r||) within 1e-9 relative over the
iterations where the oracle itself is forward-stable (a 1e-15 perturbation of b moves its
residuals by < 1e-11; short recurrences lose orthogonality, reading R17), x within
1e-6 there, identical status and stop index.
"""
import numpy as np
import pytest

from gen import make_problem
from oracle.operators import operator_from_problem
from oracle.sflsqr import solve_problem

from horizons import horizon

pytestmark = pytest.mark.gpu

RES_TOL = 1e-9
X_TOL = 1e-6


@pytest.fixture(scope="session", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_22281_b200._build import build_library
    build_library()


def _gpu_run(prob, spec, maxit, method, eta=0.0, use_graph=True, spmv_mode=None, knobs=()):
    from paper_2605_22281_b200 import solver_for_problem
    s = solver_for_problem(prob, spec, maxit=maxit, eta=eta, method=method, use_graph=use_graph,
                           knobs=(["keep_csr"] if spmv_mode is not None else []) + list(knobs))
    if spmv_mode is not None:
        s.debug_set_tuning(spmv_mode)
    s.set_rhs(prob.b)
    done, status = s.iterate(maxit)
    res, nres = s.get_residual_norms()
    x = s.get_x()
    info = s.get_info()
    s.close()
    return dict(done=done, status=status, res=res, nres=nres, x=x, info=info)


def _compare(g, r, method):
    kk = len(r.est_res)
    assert g["info"]["k_done"] == kk and g["status"] == r.status and g["info"]["k_x"] == r.k
    rr = np.abs(g["res"][:kk] - np.array(r.est_res)) / np.array(r.est_res)
    assert rr.max() < RES_TOL, ("residual", rr.max(), int(rr.argmax()) + 1)
    if method == "lsmr":
        # ||T r_k|| decays by orders of magnitude on ill-conditioned problems; its recurrence
        # carries absolute rounding ~ u * ||T b|| (its first value), so the bar is relative with
        # that absolute floor: 1e-9 |.| + 1e-12 ||T r_0||
        ref = np.array(r.est_nres)
        rn = np.abs(g["nres"][:kk] - ref) / (ref + 1e-3 * ref[0])
        assert rn.max() < RES_TOL, ("||T r||", rn.max(), int(rn.argmax()) + 1)
    ex = np.linalg.norm(g["x"] - r.x) / np.linalg.norm(r.x)
    assert ex < X_TOL, ("x", ex)


@pytest.mark.parametrize("method", ["lsqr", "lsmr"])
@pytest.mark.parametrize("cfg,kw,tag", [
    (1, {}, "c1"),                                        # dense, sigma_min 1e-6
    (2, {}, "c2"),                                        # matrix-free blur (separate epilogue pass)
    (3, dict(N=128, n_angles=90, nb=183), "c3r128"),      # Siddon, matched A^T
    (4, dict(N=160, n_angles=113, nb=227), "c4r160"),     # unmatched B ("LSQR ignoring A# != A^T")
])
def test_gkb_parity(method, cfg, kw, tag):
    p = make_problem(cfg, **kw)
    spec = p.solvers[0]
    kstar, _ = horizon(f"gkb/{tag}/{method}", p)
    r = solve_problem(p, spec, maxit=kstar, eta=0.0, method=method)
    g = _gpu_run(p, spec, kstar, method)
    _compare(g, r, method)


@pytest.mark.parametrize("method", ["lsqr", "lsmr"])
def test_gkb_discrepancy_stop_and_forced_formats(method):
    p = make_problem(3, N=96, n_angles=70, nb=137)
    spec = p.solvers[0]
    full = solve_problem(p, spec, maxit=30, eta=0.0, method=method)
    ratio = np.array(full.est_res) / p.delta_e
    k0 = min(11, int(np.flatnonzero(ratio > 1.001)[-1]))   # a level > 1 the run reaches mid-way
    eta = float(ratio[k0]) * (1 + 1e-7)
    r = solve_problem(p, spec, maxit=30, eta=eta, method=method)
    assert r.status == 3
    for mode in (None, 14, 16):                            # default format / fused CSR / fused pair-CSR epilogue
        g = _gpu_run(p, spec, 30, method, eta=eta, spmv_mode=mode)
        _compare(g, r, method)


def test_gkb_graph_and_eager_agree_bitwise():
    p = make_problem(1)
    spec = p.solvers[0]
    g1 = _gpu_run(p, spec, 25, "lsmr", use_graph=False)
    g2 = _gpu_run(p, spec, 25, "lsmr", use_graph=True)
    assert np.array_equal(g1["x"], g2["x"]) and np.array_equal(g1["res"], g2["res"])


def test_gkb_rejects_flexible_preconditioner():
    from paper_2605_22281_b200 import SFLSQR, SflsqrError
    from paper_2605_22281_b200 import sflsqr as B
    p = make_problem(1)
    s = SFLSQR(method="lsqr", maxit=5)
    s.set_operator(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, p.A.val)
    s.set_precond("irn", 1.0, 1e-3)
    with pytest.raises(SflsqrError) as e:
        s.set_rhs(p.b)
    assert e.value.code == B.E_INVALID
    s.close()


@pytest.mark.parametrize("cfg,maxit", [(3, 8), (4, 3)])
@pytest.mark.parametrize("method", ["lsqr", "lsmr"])
def test_gkb_full_size_first_iterations(cfg, maxit, method):
    p = make_problem(cfg)
    spec = p.solvers[0]
    r = solve_problem(p, spec, maxit=maxit, eta=0.0, method=method, record=False)
    g = _gpu_run(p, spec, maxit, method)
    _compare(g, r, method)
