"""Small dense least squares  y = argmin_y || rhs - M y ||_2  for the oracle.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Used for the projected sketched problems of Alg. 1 L488-496 / eq. sFLSQR
 and Alg. 2 L790-797 / eq. sFLSMR (L730-739).  Plain
unpivoted Householder QR, recomputed from scratch on every call (reading R14):
for j = 1..k the reflector H_j = I - tau_j v_j v_j^T (v_j[j] = 1) zeroes column j
below the diagonal of the partially reduced matrix; then R y = (Q^T rhs)[1:k] by
back substitution.  Pinned against numpy.linalg.lstsq (tests/test_oracle_lsq.py).
"""
import math

import numpy as np


def householder_qr_solve(M, rhs):
    """Return (y, qtb, Rdiag_min_ratio): y the LS solution, qtb = Q^T rhs, and
    min|R_jj| / max|R_jj| (rank-deficiency indicator, reading R14)."""
    R = np.array(M, dtype=np.float64, copy=True)
    q = np.array(rhs, dtype=np.float64, copy=True)
    d, k = R.shape
    if k > d:
        raise ValueError("need k <= d")
    for j in range(k):
        x = R[j:, j]
        alpha = x[0]
        xnorm = float(np.linalg.norm(x[1:])) if x.size > 1 else 0.0
        if xnorm == 0.0:
            continue  # tau = 0: H_j = I
        beta = -math.copysign(math.hypot(alpha, xnorm), alpha)
        tau = (beta - alpha) / beta
        v = x / (alpha - beta)
        v[0] = 1.0
        # apply H_j to the trailing columns (including column j) and to rhs
        R[j:, j:] -= tau * np.outer(v, v @ R[j:, j:])
        q[j:] -= tau * v * (v @ q[j:])
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        y[i] = (q[i] - R[i, i + 1:k] @ y[i + 1:k]) / R[i, i]
    diag = np.abs(np.diag(R[:k, :k]))
    ratio = float(diag.min() / diag.max()) if k > 0 and diag.max() > 0 else 0.0
    return y, q, ratio


def lstsq(M, rhs):
    """(y, ||rhs - M y||) with the residual evaluated by its definition."""
    y, _, _ = householder_qr_solve(M, rhs)
    res = float(np.linalg.norm(np.asarray(rhs) - np.asarray(M) @ y))
    return y, res
