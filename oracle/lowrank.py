"""Low-rank truncation tau_r of PAPER.md eq. (def:lowr-trc) L77-81, exact and randomised.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  tau_r(c) = vec(C_r),  C = vec^{-1}(c) the N x N image of the basis vector (row-major, reading
  R16), C_r its rank-r truncated SVD (L77-81; FLSQR with r = 30, L109, L1612).
  sFLSQR-RND / sFLSMR-RND (L1619-1623) replace the truncated SVD by the randomized SVD of
  Halko, Martinsson & Tropp (the paper's [hmt]): Y = C Omega (range finder, Omega N x l Gaussian,
  l = r + oversampling), Q = orth(Y), B = Q^T C, the top-r left singular subspace U_r of B,
  C_r = Q U_r U_r^T B.  Reading R22: the paper states neither the oversampling nor
  the power iterations nor whether Omega is redrawn; here oversampling o = 10, no power
  iterations, one Omega per solve drawn by the Gaussian generator of reading R21
  (Omega = G^T sqrt(l), G = gaussian_table(seed, l, 0, N)), U_r from the symmetric
  eigendecomposition of B B^T (LAPACK here, Jacobi on the GPU; U_r U_r^T is unique when
  lambda_r > lambda_{r+1}).
Pins: tests/test_oracle_lowrank.py (Eckart-Young, rank <= r identity, idempotence, RND == exact
when l = N, the HMT expectation bound).
"""
import numpy as np

from .sketch import gaussian_table


def tau_lowrank_exact(p, N, r, W=None):
    """vec(C_r) with C_r the rank-r truncated SVD of C = p.reshape(N, W) (eq. def:lowr-trc; W = N)."""
    C = np.asarray(p, dtype=np.float64).reshape(N, W or N)
    U, s, Vt = np.linalg.svd(C)
    return ((U[:, :r] * s[:r]) @ Vt[:r]).reshape(-1)


def rnd_omega(seed, N, r, oversample=10, W=None):
    """The range-finder test matrix Omega (W x l), l = min(r + oversample, N, W) (reading R22)."""
    W = W or N
    ell = min(r + oversample, N, W)
    return gaussian_table(seed, ell, 0, W).T * np.sqrt(ell)


def tau_lowrank_rnd(p, N, r, omega):
    """Randomised rank-r truncation (HMT range finder + SVD of the projected matrix); C is
    N x W with W = omega.shape[0]."""
    C = np.asarray(p, dtype=np.float64).reshape(N, omega.shape[0])
    Y = C @ omega
    Q, _ = np.linalg.qr(Y)                     # orthonormal basis of range(Y)
    B = Q.T @ C
    lam, V = np.linalg.eigh(B @ B.T)           # ascending
    Ur = V[:, ::-1][:, :r]                     # top-r left singular vectors of B
    return (Q @ (Ur @ (Ur.T @ B))).reshape(-1)
