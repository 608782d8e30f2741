"""Pin P3: the oracle's small Householder least-squares solve (Alg. 1,
Alg. 2) against numpy.linalg.lstsq (LAPACK SVD) and LS optimality."""
import numpy as np
import pytest

from oracle.lsq import householder_qr_solve, lstsq


@pytest.mark.parametrize("d,k", [(80, 1), (80, 17), (80, 40), (300, 150), (5, 5)])
def test_householder_matches_lapack(d, k):
    rng = np.random.default_rng(d * 1000 + k)
    U = np.linalg.qr(rng.standard_normal((d, k)))[0]
    V = np.linalg.qr(rng.standard_normal((k, k)))[0]
    M = (U * np.logspace(0, -3, k)) @ V.T           # cond 1e3
    rhs = rng.standard_normal(d)
    y, res = lstsq(M, rhs)
    y_ref = np.linalg.lstsq(M, rhs, rcond=None)[0]
    np.testing.assert_allclose(y, y_ref, rtol=1e-10 * 1e3, atol=0)
    r_ref = np.linalg.norm(rhs - M @ y_ref)
    assert abs(res - r_ref) <= 1e-12 * max(1.0, r_ref) + 1e-13 * np.linalg.norm(rhs)
    # normal-equation optimality: M^T (M y - rhs) ~ 0
    assert np.linalg.norm(M.T @ (M @ y - rhs)) <= 1e-9 * np.linalg.norm(M) * np.linalg.norm(rhs)


def test_qtb_tail_is_residual():
    rng = np.random.default_rng(5)
    M = rng.standard_normal((50, 12))
    rhs = rng.standard_normal(50)
    y, qtb, ratio = householder_qr_solve(M, rhs)
    assert abs(np.linalg.norm(qtb[12:]) - np.linalg.norm(rhs - M @ y)) < 1e-12
    assert 0 < ratio <= 1


def test_exact_system_and_scale_invariance():
    rng = np.random.default_rng(6)
    M = rng.standard_normal((30, 10))
    ytrue = rng.standard_normal(10)
    y, res = lstsq(M, M @ ytrue)
    np.testing.assert_allclose(y, ytrue, rtol=1e-12, atol=1e-12)
    assert res < 1e-12
    # argmin is invariant under scaling both M and rhs by c > 0 (SPEC "sketch" invariants)
    rhs = rng.standard_normal(30)
    y1, _ = lstsq(M, rhs)
    y2, _ = lstsq(3.7 * M, 3.7 * rhs)
    np.testing.assert_allclose(y1, y2, rtol=1e-12)


def test_rank_deficiency_flag():
    rng = np.random.default_rng(7)
    M = rng.standard_normal((20, 4))
    M[:, 3] = M[:, 0] + M[:, 1]
    _, _, ratio = householder_qr_solve(M, rng.standard_normal(20))
    assert ratio < 1e-14
