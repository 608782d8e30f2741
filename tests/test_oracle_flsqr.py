"""Pins for the oracle's unsketched full-orthogonalisation methods FLSQR / FLSMR
(PAPER.md §"Flexible Golub-Kahan factorization, FLSQR and
FLSMR", L321-373).

Each test fixes the oracle against something other than itself:
  * tau = id: FGK = GKB (L342-344), so FLSQR / FLSMR iterates are SciPy's textbook
    LSQR / LSMR iterates (eqs. xlsqr / xlsmr, L292-313);
  * any tau (IRN, NONNEG), matched or unmatched: the DEFINITIONS of eq. (FLSQR)
    (x_k = Z_k argmin ||b - A Z_k y||) and of FLSMR L361-367 (argmin ||A^T (b - A Z_k y)||,
    with the transpose-side operator in place of A^T when unmatched), solved by dense
    brute force (numpy.linalg.lstsq) on the run's own Z_k;
  * FLSQR == sFLSQR with the identity sketch and a full window (L532 footnote);
  * the FLSQR projected residual equals ||b - A x_k|| (orthonormal W_{k+1}, L357);
  * eq. (flsqr-relations) L335-345 with full orthogonalisation: A^T W_k = P_k T_k,
    A Z_k = W_{k+1} H_{k+1,k}, P and W orthonormal, T upper triangular.
"""
import numpy as np
import pytest
from scipy.sparse.linalg import lsmr, lsqr

from oracle.operators import DenseOperator
from oracle.sflsqr import MAXIT, solve
from oracle.sketch import IdentitySketch


def _dense_problem(m, n, cond, seed, noise=0.05):
    rng = np.random.default_rng(seed)
    U = np.linalg.qr(rng.standard_normal((m, n)))[0]
    V = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = (U * np.logspace(0, -np.log10(cond), n)) @ V.T
    x = np.abs(rng.standard_normal(n))
    b = A @ x
    e = rng.standard_normal(m)
    b = b + e * (noise * np.linalg.norm(b) / np.linalg.norm(e))
    return A, b, rng


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("method,ref", [("flsqr", "lsqr"), ("flsmr", "lsmr")])
def test_identity_tau_equals_scipy(method, ref):
    A, b, _ = _dense_problem(60, 40, 1e2, 21)
    K = 14
    r = solve(DenseOperator(A), b, method, maxit=K, precond="identity")
    assert r.status == MAXIT
    for k in range(1, K + 1):
        if ref == "lsqr":
            xk = lsqr(A, b, atol=0, btol=0, conlim=0, iter_lim=k)[0]
        else:
            xk = lsmr(A, b, atol=0, btol=0, conlim=0, maxiter=k)[0]
        assert _rel(r.xs[k - 1], xk) < 1e-8, k


@pytest.mark.parametrize("precond", ["irn", "nonneg"])
@pytest.mark.parametrize("matched", [True, False])
def test_definitions_by_brute_force(precond, matched):
    A, b, rng = _dense_problem(70, 50, 1e3, 22)
    B = A.T if matched else A.T + 0.03 * rng.standard_normal((50, 70)) / np.sqrt(70)
    op = DenseOperator(A, None if matched else B)
    K = 15
    rq = solve(op, b, "flsqr", maxit=K, precond=precond)
    rm = solve(op, b, "flsmr", maxit=K, precond=precond)
    for k in range(1, K + 1):
        AZ = A @ rq.Z[:, :k]
        yq = np.linalg.lstsq(AZ, b, rcond=None)[0]                       # eq. (FLSQR)
        assert _rel(rq.xs[k - 1], rq.Z[:, :k] @ yq) < 1e-8, k
        AZm = A @ rm.Z[:, :k]
        ym = np.linalg.lstsq(B @ AZm, B @ b, rcond=None)[0]              # FLSMR L361-363 (T for A^T)
        assert _rel(rm.xs[k - 1], rm.Z[:, :k] @ ym) < 1e-8, k


def test_flsqr_equals_sflsqr_with_identity_sketch_full_window():
    A, b, _ = _dense_problem(64, 48, 1e2, 23)
    K = 12
    r1 = solve(DenseOperator(A), b, "flsqr", maxit=K, precond="irn")
    r2 = solve(DenseOperator(A), b, "sflsqr", maxit=K, window=K + 1, sketch=IdentitySketch(64), precond="irn")
    for k in range(K):
        assert _rel(r1.xs[k], r2.xs[k]) < 1e-9, k
        assert abs(r1.sketch_res[k] - r2.sketch_res[k]) <= 1e-9 * r2.sketch_res[k], k


@pytest.mark.parametrize("precond", ["identity", "irn"])
def test_flsqr_projected_residual_is_true_residual(precond):
    A, b, _ = _dense_problem(80, 60, 1e4, 24, noise=0.1)
    r = solve(DenseOperator(A), b, "flsqr", maxit=20, precond=precond)
    np.testing.assert_allclose(r.sketch_res, r.true_res, rtol=1e-9)
    assert np.all(np.diff(r.true_res) <= 1e-12 * r.true_res[0])          # nested spaces: monotone


@pytest.mark.parametrize("method", ["flsqr", "flsmr"])
@pytest.mark.parametrize("matched", [True, False])
def test_full_fgk_relations(method, matched):
    A, b, rng = _dense_problem(70, 50, 1e3, 25)
    B = None if matched else A.T + 0.03 * rng.standard_normal((50, 70)) / np.sqrt(70)
    op = DenseOperator(A, B)
    K = 18
    r = solve(op, b, method, maxit=K, precond="irn")
    Z, W, H, P, Tm = r.Z, r.W, r.H, r.P, r.T
    assert np.linalg.norm(A @ Z - W @ H) <= 1e-12 * np.linalg.norm(A @ Z)
    TW = op.Td @ W[:, :K]
    assert np.linalg.norm(TW - P @ Tm) <= 1e-12 * np.linalg.norm(TW)
    assert np.all(np.tril(Tm, -1) == 0) and np.all(np.tril(H, -2) == 0)
    np.testing.assert_allclose(W.T @ W, np.eye(K + 1), atol=1e-12)
    np.testing.assert_allclose(P.T @ P, np.eye(K), atol=1e-12)


def test_flsmr_objective_is_normal_equation_residual():
    # L361-367: || T_{k+1}(beta e1 - H y) || = || A^T (b - A x_k) || (P_{k+1} orthonormal)
    A, b, _ = _dense_problem(60, 45, 1e3, 26)
    r = solve(DenseOperator(A), b, "flsmr", maxit=16, precond="irn")
    for k in range(16):
        ne = np.linalg.norm(A.T @ (b - A @ r.xs[k]))
        assert abs(r.sketch_res[k] - ne) <= 1e-9 * ne, k
