"""GPU: the deferred stop test (sflsqr.cu defer_stop) against the inline order.

On one rank the W-path residual and the stop tests of iteration k run on the side stream during
iteration k + 1, beside its z side and A z_{k+1}; the main stream waits for the decision before
anything a stop at k must not see.  Only the order of independent work changes, so every result --
x, both residual histories, status, stop index, the iterate held in y -- must be bitwise that of
SFLSQR_KNOB_STOP_INLINE (the residual and stop at the end of iteration k), including runs that stop
by the discrepancy principle, by the sketched-residual tolerance, by maxit, by a breakdown, and
runs driven by several iterate() calls (the last iteration's tests run after each call's final
launch and again, identically, at the start of the next call).
"""
import dataclasses

import numpy as np
import pytest

from gen import make_problem
from gen.problems import CSR, Problem, SolverSpec
from oracle.sflsqr import solve_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_22281_b200._build import build_library
    build_library()


def _run(p, spec, knobs, maxit, eta=None, chunks=None, use_graph=True):
    from paper_2605_22281_b200 import solver_for_problem
    s = solver_for_problem(p, spec, maxit=maxit, eta=eta, knobs=knobs, use_graph=use_graph)
    s.set_rhs(p.b)
    for c in (chunks or [maxit]):
        done, status = s.iterate(c)
    tr, sk = s.get_residual_norms()
    out = dict(x=s.get_x(), tr=tr, sk=sk, status=status, done=done, info=s.get_info())
    s.close()
    return out


def _same(a, b):
    assert a["status"] == b["status"] and a["done"] == b["done"]
    for key in ("k_done", "k_x"):
        assert a["info"][key] == b["info"][key], key
    for key in ("x", "tr", "sk"):
        assert np.array_equal(a[key], b[key]), key


CASES = {
    "c3r_sflsqr": (lambda: make_problem(3, N=128, n_angles=90, nb=183), "sflsqr", 14),   # NONNEG: x update on the side
    "c3r_sflsmr": (lambda: make_problem(3, N=128, n_angles=90, nb=183), "sflsmr", 14),
    "c4r_sflsqr": (lambda: make_problem(4, N=96, n_angles=61, nb=137), "sflsqr", 14),    # identity tau, unmatched B
    "c1_sflsmr": (lambda: make_problem(1), "sflsmr", 20),                                 # IRN, dense
    "c2_sflsqr": (lambda: make_problem(2), "sflsqr", 12),                                 # matrix-free blur
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_deferred_stop_bitwise_equal_to_inline(case):
    mk, method, K = CASES[case]
    p = mk()
    spec = dataclasses.replace([s for s in p.solvers if s.method == method][0] if any(
        s.method == method for s in p.solvers) else p.solvers[0], method=method)
    a = _run(p, spec, [], K, eta=0.0)
    b = _run(p, spec, ["stop_inline"], K, eta=0.0)
    assert a["status"] == 1 and a["info"]["k_done"] == K
    _same(a, b)
    # several iterate() calls (the tail re-evaluated at the next call) and eager launches
    _same(a, _run(p, spec, [], K, eta=0.0, chunks=[1, 4, 2, K]))
    _same(a, _run(p, spec, [], K, eta=0.0, use_graph=False))


@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_deferred_discrepancy_and_tol_stops(method):
    p = make_problem(1)
    spec = [s for s in p.solvers if s.method == method][0]
    full = solve_problem(p, spec, eta=0.0)
    eta = float(full.true_res[14] / p.delta_e) * (1 + 1e-7)
    a = _run(p, spec, [], 40, eta=eta)
    assert a["status"] == 3 and a["info"]["k_done"] == 15
    _same(a, _run(p, spec, ["stop_inline"], 40, eta=eta))
    _same(a, _run(p, spec, [], 40, eta=eta, chunks=[15, 5]))   # stops in the tail of the first call
    _same(a, _run(p, spec, [], 40, eta=eta, chunks=[16, 5]))   # stops inside the second call's first graph
    # sketched-residual tolerance (L498 / L798): stop when ||rhs - M_k y_k|| < tol ||rhs||, mid-run
    tol = float(full.sketch_res[11] / np.linalg.norm(full.rhs)) * (1 + 1e-7)
    spec_t = dataclasses.replace(spec, tol=tol)
    r = solve_problem(p, spec_t, eta=0.0)
    assert r.status == 2
    a = _run(p, spec_t, [], 40, eta=0.0)
    assert a["status"] == 2 and a["info"]["k_done"] == r.k
    _same(a, _run(p, spec_t, ["stop_inline"], 40, eta=0.0))


def test_deferred_breakdown():
    A = np.diag([1.0, 2.0, 3.0, 4.0])
    b = np.array([1.0, 1.0, 0.0, 0.0])
    p = Problem(name="bd", config_index=0, m=4, n=4, A=CSR.from_dense(A), T=None, t_mode="build", blur=None,
                x_true=np.zeros(4), b=b, e=np.zeros(4), delta=0, delta_e=0.0, sketch_seed=5)
    spec = SolverSpec(method="sflsqr", maxit=4, window=4, d=4, s_nz=1, precond="identity")
    a = _run(p, spec, [], 4)
    assert a["status"] == 4
    _same(a, _run(p, spec, ["stop_inline"], 4))
    _same(a, _run(p, spec, [], 4, chunks=[1, 1, 1, 1]))
