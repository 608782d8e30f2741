"""Textbook LSQR and LSMR on the Golub-Kahan bidiagonalization (GKB), plain fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §"Golub-Kahan bidiagonalization, LSQR and LSMR" (L277-319): GKB eq. (GKB)
L279-285 with u_1 = b / ||b||; LSQR eq. (xlsqr), x_k = V_k argmin || ||b|| e_1 -
B_{k+1,k} y ||; LSMR eq. (xlsmr), x_k = V_k argmin || B_{k+1}^T (||b|| e_1 - B_{k+1,k} y) ||;
"computing x_k efficiently (using smart QR factorization updates for B_{k+1,k} and
B_{k+1}) only requires the storage of 2 vectors of length m and 3 or 4 vectors of length n"
(L316-319).  The short recurrences are the published ones: Paige & Saunders (1982) for
LSQR (one Givens rotation per step on B_{k+1,k}), Fong & Saunders (2011) for LSMR (two
rotations: QR of B_k, then of R_k^T), each restated here in the order of the papers.
With an unmatched transpose-side operator T ~ A^T the same recurrences run with T in
place of A^T ("LSQR ignoring A# != A^T").

Histories (reading R19):
  est_res[k-1]  = the recurrence's ||b - A x_k|| (LSQR: |phibar_{k+1}|; LSMR: Fong-Saunders'
                  ||r_k|| estimate) -- what a GKB solver monitors and what its stop rules use;
  true_res[k-1] = ||b - A x_k|| by an explicit product (the definition, eq. discrP);
  est_nres[k-1] = LSMR's ||T (b - A x_k)|| = |zetabar_{k+1}|.
Pins: tests/test_oracle_gkb.py (SciPy lsqr / lsmr iterates and residual norms, brute-force
Krylov least squares, the FLSQR / FLSMR reduction with tau = id).
"""
import math
from dataclasses import dataclass, field

import numpy as np

RUNNING, MAXIT, TOL, DISCREPANCY, BREAKDOWN = 0, 1, 2, 3, 4


@dataclass
class GKBResult:
    x: np.ndarray
    k: int
    status: int
    true_res: list = field(default_factory=list)
    est_res: list = field(default_factory=list)
    est_nres: list = field(default_factory=list)
    xs: list = field(default_factory=list)
    alphas: list = field(default_factory=list)     # alpha_1, alpha_2, ... (diagonal of B)
    betas: list = field(default_factory=list)      # beta_1, beta_2, ... (subdiagonal of B)


def _rot(a, b):
    """Givens rotation [c s; -s c] with c a + s b = r >= 0 ... (r = hypot(a, b), c = a/r, s = b/r)."""
    r = math.hypot(a, b)
    if r == 0.0:
        return 1.0, 0.0, 0.0
    return a / r, b / r, r


def _gkb_start(op, b):
    """eq. (GKB): beta_1 u_1 = b, alpha_1 v_1 = A^T u_1."""
    b = np.asarray(b, dtype=np.float64)
    beta = float(np.linalg.norm(b))
    if beta == 0.0:
        raise ValueError("||b|| = 0")
    u = b / beta
    v = op.tmatvec(u)
    alpha = float(np.linalg.norm(v))
    if alpha > 0.0:
        v = v / alpha
    return b, u, v, alpha, beta


def _gkb_step(op, u, v, alpha):
    """One GKB step: beta u' = A v - alpha u, alpha' v' = A^T u' - beta v."""
    u = op.matvec(v) - alpha * u
    beta = float(np.linalg.norm(u))
    if beta > 0.0:
        u = u / beta
    v = op.tmatvec(u) - beta * v
    alpha = float(np.linalg.norm(v))
    if alpha > 0.0:
        v = v / alpha
    return u, v, alpha, beta


def lsqr(op, b, maxit=10, eta=0.0, delta_e=0.0, record=True):
    """LSQR (Paige & Saunders): QR of B_{k+1,k} by one rotation per step, x by a short recurrence.
    Stops at maxit, on the discrepancy principle with the recurrence residual
    (|phibar| <= eta delta_e, reading R19), or on breakdown (alpha or beta = 0)."""
    b, u, v, alpha, beta = _gkb_start(op, b)
    n = op.n
    x = np.zeros(n)
    w = v.copy()
    phibar, rhobar = beta, alpha
    res = GKBResult(x=x, k=0, status=RUNNING)
    res.alphas.append(alpha)
    res.betas.append(beta)
    for k in range(1, maxit + 1):
        u, v, alpha, beta = _gkb_step(op, u, v, alpha)      # beta_{k+1}, alpha_{k+1}
        res.alphas.append(alpha)
        res.betas.append(beta)
        c, s, rho = _rot(rhobar, beta)                      # rotation eliminating beta_{k+1}
        theta = s * alpha
        rhobar = -c * alpha
        phi = c * phibar
        phibar = s * phibar
        if rho > 0.0:                                       # rho = 0 only at an exact breakdown
            x = x + (phi / rho) * w
            w = v - (theta / rho) * w
        res.x, res.k = x, k
        res.est_res.append(abs(phibar))
        res.true_res.append(float(np.linalg.norm(b - op.matvec(x))))
        if record:
            res.xs.append(x)
        if alpha == 0.0 or beta == 0.0:
            res.status = BREAKDOWN
            return res
        if eta > 0.0 and abs(phibar) <= eta * delta_e:
            res.status = DISCREPANCY
            return res
    res.status = MAXIT
    return res


def lsmr(op, b, maxit=10, eta=0.0, delta_e=0.0, record=True):
    """LSMR (Fong & Saunders), undamped: rotation Q_k turns B_k into R_k, rotation Qbar_k
    turns R_k^T into Rbar_k; x by the h / hbar recurrences; ||r_k|| by the paper's
    estimate (rotations Qhat (identity when undamped), Q, Qtilde)."""
    b, u, v, alpha, beta = _gkb_start(op, b)
    n = op.n
    x = np.zeros(n)
    h = v.copy()
    hbar = np.zeros(n)
    zetabar, alphabar = alpha * beta, alpha
    rho, rhobar, cbar, sbar = 1.0, 1.0, 1.0, 0.0
    # ||r|| estimate
    betadd, betad, rhodold, tautildeold, thetatilde, zeta, dsum = beta, 0.0, 1.0, 0.0, 0.0, 0.0, 0.0
    res = GKBResult(x=x, k=0, status=RUNNING)
    res.alphas.append(alpha)
    res.betas.append(beta)
    for k in range(1, maxit + 1):
        u, v, alpha, beta = _gkb_step(op, u, v, alpha)      # beta_{k+1}, alpha_{k+1}
        res.alphas.append(alpha)
        res.betas.append(beta)
        # Q_k on [alphabar_k; beta_{k+1}]  (damping 0: alphahat = alphabar)
        rhoold = rho
        c, s, rho = _rot(alphabar, beta)
        thetanew = s * alpha
        alphabar = c * alpha
        # Qbar_k on [cbar_{k-1} rho_k; theta_{k+1}]
        rhobarold, zetaold = rhobar, zeta
        thetabar = sbar * rho
        cbar, sbar, rhobar = _rot(cbar * rho, thetanew)
        zeta = cbar * zetabar
        zetabar = -sbar * zetabar
        # h, hbar, x
        hbar = h - (thetabar * rho / (rhoold * rhobarold)) * hbar
        x = x + (zeta / (rho * rhobar)) * hbar
        h = v - (thetanew / rho) * h
        # ||r_k|| estimate: Qhat = I (undamped), then Q_k, then Qtilde_{k-1}
        betaacute = betadd
        betahat = c * betaacute
        betadd = -s * betaacute
        thetatildeold = thetatilde
        ctildeold, stildeold, rhotildeold = _rot(rhodold, thetabar)
        thetatilde = stildeold * rhobar
        rhodold = ctildeold * rhobar
        betad = -stildeold * betad + ctildeold * betahat
        tautildeold = (zetaold - thetatildeold * tautildeold) / rhotildeold
        taud = (zeta - thetatilde * tautildeold) / rhodold
        normr = math.sqrt(dsum + (betad - taud) ** 2 + betadd * betadd)
        res.x, res.k = x, k
        res.est_res.append(normr)
        res.est_nres.append(abs(zetabar))
        res.true_res.append(float(np.linalg.norm(b - op.matvec(x))))
        if record:
            res.xs.append(x)
        if alpha == 0.0 or beta == 0.0:
            res.status = BREAKDOWN
            return res
        if eta > 0.0 and normr <= eta * delta_e:
            res.status = DISCREPANCY
            return res
    res.status = MAXIT
    return res
