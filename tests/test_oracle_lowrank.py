"""Pins for the oracle's low-rank truncation tau_r (oracle/lowrank.py; PAPER.md eq.
def:lowr-trc L77-81; randomized variant L1619-1623, reading R22).

  * Eckart-Young: ||C - C_r||_F^2 = sum_{i > r} sigma_i^2 and rank(C_r) = r;
  * tau_r is the identity on matrices of rank <= r and idempotent;
  * the randomized variant equals the exact truncation when the range finder sees the whole
    space (l = N), and when rank(C) <= r;
  * the HMT expectation bound E||C - Q Q^T C|| <= (1 + ...) holds on average over draws;
  * sFLSQR with tau_r keeps the FGK relations (A Z = W H, T W = P T) - tau only shapes Z.
"""
import numpy as np
import pytest

from oracle.lowrank import rnd_omega, tau_lowrank_exact, tau_lowrank_rnd
from oracle.operators import DenseOperator
from oracle.sflsqr import solve
from oracle.sketch import SparseSignSketch


def _decaying(N, seed, decay=0.7):
    rng = np.random.default_rng(seed)
    U = np.linalg.qr(rng.standard_normal((N, N)))[0]
    V = np.linalg.qr(rng.standard_normal((N, N)))[0]
    s = decay ** np.arange(N)
    return (U * s) @ V.T, s


def test_eckart_young_and_rank():
    N, r = 40, 7
    C, s = _decaying(N, 1)
    Cr = tau_lowrank_exact(C.reshape(-1), N, r).reshape(N, N)
    assert abs(np.linalg.norm(C - Cr) ** 2 - np.sum(s[r:] ** 2)) <= 1e-12 * np.sum(s ** 2)
    sv = np.linalg.svd(Cr, compute_uv=False)
    assert sv[r - 1] > 1e-3 and sv[r] < 1e-12


def test_identity_on_low_rank_and_idempotent():
    rng = np.random.default_rng(2)
    N, r = 30, 5
    C = rng.standard_normal((N, 3)) @ rng.standard_normal((3, N))          # rank 3 <= r
    c = C.reshape(-1)
    np.testing.assert_allclose(tau_lowrank_exact(c, N, r), c, atol=1e-12 * np.abs(c).max())
    om = rnd_omega(5, N, r)
    np.testing.assert_allclose(tau_lowrank_rnd(c, N, r, om), c, atol=1e-12 * np.abs(c).max())
    D, _ = _decaying(N, 3)
    t1 = tau_lowrank_exact(D.reshape(-1), N, r)
    np.testing.assert_allclose(tau_lowrank_exact(t1, N, r), t1, atol=1e-13)


def test_rnd_equals_exact_when_range_finder_is_complete():
    N, r = 24, 6
    C, _ = _decaying(N, 4, decay=0.8)
    om = rnd_omega(9, N, r, oversample=N)          # l = N: Y spans R^N
    np.testing.assert_allclose(tau_lowrank_rnd(C.reshape(-1), N, r, om), tau_lowrank_exact(C.reshape(-1), N, r),
                               atol=1e-12)


def test_hmt_expected_error_bound():
    # HMT Thm 10.5: E||C - Q Q^T C||_F <= (1 + r/(o-1))^{1/2} (sum_{i>r} s_i^2)^{1/2}  (o = oversampling)
    N, r, o = 60, 8, 10
    C, s = _decaying(N, 5, decay=0.85)
    tail = np.sqrt(np.sum(s[r:] ** 2))
    errs = []
    for seed in range(40):
        om = rnd_omega(100 + seed, N, r, oversample=o)
        Q = np.linalg.qr(C @ om)[0]
        errs.append(np.linalg.norm(C - Q @ (Q.T @ C)))
    assert np.mean(errs) <= np.sqrt(1 + r / (o - 1)) * tail


@pytest.mark.parametrize("kind", ["lowrank", "lowrank_rnd"])
def test_fgk_relations_with_lowrank_tau(kind):
    rng = np.random.default_rng(6)
    N = 12
    n, m = N * N, 200
    A = rng.standard_normal((m, n)) / np.sqrt(m)
    b = A @ tau_lowrank_exact(rng.standard_normal(n), N, 3) + 0.01 * rng.standard_normal(m)
    lr = dict(N=N, r=4, omega=rnd_omega(11, N, 4))
    K = 12
    r = solve(DenseOperator(A), b, "sflsqr", maxit=K, window=3, sketch=SparseSignSketch(1, 40, 4, m),
              precond=kind, fixed_diag=lr)
    assert np.linalg.norm(A @ r.Z - r.W @ r.H) <= 1e-12 * np.linalg.norm(A @ r.Z)
    TW = A.T @ r.W[:, :K]
    assert np.linalg.norm(TW - r.P @ r.T) <= 1e-12 * np.linalg.norm(TW)
    for j in range(K):                            # every basis vector is a rank-4 image
        assert np.linalg.svd(r.Z[:, j].reshape(N, N), compute_uv=False)[4] < 1e-12
