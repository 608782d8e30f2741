"""Pins for the oracle's textbook LSQR / LSMR (oracle/gkb.py; SURVEY.md §8(f) NEXT-4;
PAPER.md L277-319).

  * iterates and residual norms equal SciPy's lsqr / lsmr (library routines; with an
    unmatched transpose-side operator through a LinearOperator whose rmatvec is B);
  * the definitions eq. (xlsqr) L292-300 / eq. (xlsmr) L304-313 by brute force (explicit
    Krylov basis + dense least squares) on a well-conditioned problem;
  * the GKB bidiagonal B_{k+1,k} (alphas / betas) equals the FLSQR H with tau = id (L342-344);
  * the recurrence residual equals the explicit ||b - A x_k|| while GKB stays orthogonal.
"""
import numpy as np
import pytest
from scipy.sparse.linalg import LinearOperator, lsmr, lsqr

from oracle import gkb
from oracle.operators import DenseOperator
from oracle.sflsqr import solve


def _problem(m, n, cond, seed, noise=0.05):
    rng = np.random.default_rng(seed)
    U = np.linalg.qr(rng.standard_normal((m, n)))[0]
    V = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = (U * np.logspace(0, -np.log10(cond), n)) @ V.T
    b = A @ rng.standard_normal(n)
    e = rng.standard_normal(m)
    return A, b + e * (noise * np.linalg.norm(b) / np.linalg.norm(e)), rng


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("matched", [True, False])
def test_lsqr_equals_scipy(matched):
    # a well-separated spectrum: short-recurrence GKB stays forward-stable over K steps, so two
    # implementations agree to rounding (clustered spectra amplify 1-ulp differences, reading R17)
    A, b, rng = _problem(300, 200, 10, 31)
    B = A.T if matched else A.T + 0.02 * rng.standard_normal(A.T.shape) / np.sqrt(300)
    op = DenseOperator(A, None if matched else B)
    lo = LinearOperator(A.shape, matvec=lambda v: A @ v, rmatvec=lambda u: B @ u, dtype=np.float64)
    K = 25
    r = gkb.lsqr(op, b, maxit=K)
    for k in range(1, K + 1):
        out = lsqr(lo, b, atol=0, btol=0, conlim=0, iter_lim=k)
        assert _rel(r.xs[k - 1], out[0]) < 1e-9, k
        assert abs(r.est_res[k - 1] - out[3]) <= 1e-9 * out[3], k       # r1norm = |phibar|


@pytest.mark.parametrize("matched", [True, False])
def test_lsmr_equals_scipy(matched):
    A, b, rng = _problem(300, 200, 10, 32)
    B = A.T if matched else A.T + 0.02 * rng.standard_normal(A.T.shape) / np.sqrt(300)
    op = DenseOperator(A, None if matched else B)
    lo = LinearOperator(A.shape, matvec=lambda v: A @ v, rmatvec=lambda u: B @ u, dtype=np.float64)
    K = 25
    r = gkb.lsmr(op, b, maxit=K)
    for k in range(1, K + 1):
        out = lsmr(lo, b, atol=0, btol=0, conlim=0, maxiter=k)
        assert _rel(r.xs[k - 1], out[0]) < 1e-9, k
        assert abs(r.est_res[k - 1] - out[3]) <= 1e-9 * out[3], k       # normr
        assert abs(r.est_nres[k - 1] - out[4]) <= 1e-9 * out[4], k      # normar


def test_definitions_by_brute_force():
    A, b, _ = _problem(60, 40, 1e2, 33)
    K = 12
    rq, rm = gkb.lsqr(DenseOperator(A), b, maxit=K), gkb.lsmr(DenseOperator(A), b, maxit=K)
    for k in range(1, K + 1):
        Q = (A.T @ b)[:, None] / np.linalg.norm(A.T @ b)      # orthonormal basis of K_k(A^T A, A^T b)
        for _ in range(k - 1):
            q = A.T @ (A @ Q[:, -1])
            for _ in range(2):
                q = q - Q @ (Q.T @ q)
            Q = np.column_stack([Q, q / np.linalg.norm(q)])
        xq = Q @ np.linalg.lstsq(A @ Q, b, rcond=None)[0]                # eq. (xlsqr)
        xm = Q @ np.linalg.lstsq(A.T @ A @ Q, A.T @ b, rcond=None)[0]    # eq. (xlsmr)
        assert _rel(rq.xs[k - 1], xq) < 1e-9 and _rel(rm.xs[k - 1], xm) < 1e-9, k


def test_bidiagonal_is_flsqr_H_with_identity_tau():
    A, b, _ = _problem(50, 35, 1e2, 34)
    K = 10
    r = gkb.lsqr(DenseOperator(A), b, maxit=K)
    f = solve(DenseOperator(A), b, "flsqr", maxit=K, precond="identity")
    H = f.H
    np.testing.assert_allclose(np.diag(H[:K, :K]), r.alphas[:K], rtol=1e-10)
    np.testing.assert_allclose(np.diag(H[1:K + 1, :K]), r.betas[1:K + 1], rtol=1e-10)
    for k in range(K):
        assert _rel(r.xs[k], f.xs[k]) < 1e-9


@pytest.mark.parametrize("fn", [gkb.lsqr, gkb.lsmr])
def test_recurrence_residual_is_true_residual(fn):
    A, b, _ = _problem(80, 50, 1e2, 35)
    r = fn(DenseOperator(A), b, maxit=15)
    np.testing.assert_allclose(r.est_res, r.true_res, rtol=1e-9)


def test_discrepancy_stop_on_recurrence_residual():
    A, b, _ = _problem(90, 60, 1e4, 36, noise=0.1)
    full = gkb.lsqr(DenseOperator(A), b, maxit=30)
    level = full.est_res[9] * (1 + 1e-9)
    hit = next(k + 1 for k, v in enumerate(full.est_res) if v <= level)
    r = gkb.lsqr(DenseOperator(A), b, maxit=30, eta=1.5, delta_e=level / 1.5)
    assert r.status == gkb.DISCREPANCY and r.k == hit
