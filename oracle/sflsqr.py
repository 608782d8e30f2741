"""sFLSQR (Algorithm 1) and sFLSMR (Algorithm 2), plain fp64, followed line by line.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Sources:
  * Alg. 1 sFLSQR, L450-508; eq. sFLSQR; eq. FGK (partial flexible
    Golub-Kahan with window ell) L400-406; cost L444-448.
  * Alg. 2 sFLSMR, L752-808; eq. sFLSMR L730-749 ("compute the columns of
    S A^T W ... then right-multiply by H ... implemented in our code").
  * Discrepancy principle eq. discrP, L50-53.
  * Flexible preconditioning as tau, L59-64, L322-345.
Readings of paper-silent / ambiguous points (R1-R14):
  R1  orth_mode "P" orthogonalises the new direction against the last ell
      normalised pre-tau directions p_j (eq. FGK: A^T W = P T); "Z" is the
      literal Alg. 1 L466 form (against z_j = tau(p_j)).  Identical when tau = id.
  R2  loop bounds of Alg. 1/2 are followed verbatim.
  R3  the sFLSMR tol test uses the residual of the L796 problem.
  R4  sFLSQR sketches m-vectors, sFLSMR sketches n-vectors.
  R7  IRN-l_p: tau_k(v) = D_k v, D_k = diag((x_{k-1}^2 + eps^2)^((2-p)/4)),
      eps = eps_rel * max|x_{k-1}|; D_1 = I (x_0 = 0; also D = I if x_{k-1} = 0).
  R8  NONNEG: D_k = diag(max(x_{k-1}, 0) + eps_rel * max(x_{k-1})_+); D_1 = I
      (also D = I if max(x_{k-1})_+ = 0).
  R11 breakdown: if ||z|| <= 1e-14 ||T w_k|| (before orthogonalisation) z_k
      cannot be formed: status BREAKDOWN, return x_{k-1}.  If
      ||w|| <= 1e-14 ||A z_k|| after the w-orthogonalisation (A z_k in span W_k):
      H_{k+1,k} := 0, w_{k+1} := 0, z := 0, the step-k LS is still solved and x_k
      is returned with status BREAKDOWN.
  R12 discrepancy uses the true residual ||b - A x_k|| (explicit product here).
  R13 z = T w_{k+1} is formed before the stop test (Alg. 1 L486 precedes L498).
  R14 the projected problem is solved by Householder QR from scratch (oracle/lsq.py).
"""
from dataclasses import dataclass, field

import numpy as np

from .lsq import householder_qr_solve
from .sketch import SparseSignSketch

RUNNING, MAXIT, TOL, DISCREPANCY, BREAKDOWN = 0, 1, 2, 3, 4


@dataclass
class OracleResult:
    x: np.ndarray
    k: int                      # iterate index returned (x = x_k)
    status: int
    true_res: list = field(default_factory=list)     # ||b - A x_k||, k = 1..
    sketch_res: list = field(default_factory=list)   # ||rhs - M_k y_k||
    ys: list = field(default_factory=list)
    xs: list = field(default_factory=list)
    H: np.ndarray = None
    T: np.ndarray = None
    Z: np.ndarray = None
    P: np.ndarray = None
    W: np.ndarray = None
    sketch_cols: np.ndarray = None   # M_k columns (sFLSQR) / [S_TW, S z] (sFLSMR)
    rhs: np.ndarray = None
    rank_ratio: list = field(default_factory=list)


def tau_apply(kind, p_k, x_prev, k, p_exp=1.0, eps_rel=1e-3, fixed=None):
    """z_k = tau_k(p_k) (Alg. 1 L470 / Alg. 2; readings R7, R8)."""
    if kind == "identity":
        return p_k.copy()
    if kind == "diag":                     # fixed SPD diagonal (pin P4b)
        return fixed * p_k
    if k == 1:
        return p_k.copy()                  # D_1 = I (x_0 = 0)
    if kind == "irn":
        xm = float(np.max(np.abs(x_prev)))
        if xm == 0.0:
            return p_k.copy()
        eps = eps_rel * xm
        v = x_prev * x_prev + eps * eps
        if p_exp == 1.0:
            D = np.sqrt(np.sqrt(v))        # (.)^(1/4)
        else:
            D = np.power(v, (2.0 - p_exp) / 4.0)
        return D * p_k
    if kind == "nonneg":
        xp = np.maximum(x_prev, 0.0)
        mx = float(np.max(xp))
        if mx == 0.0:
            return p_k.copy()
        return (xp + eps_rel * mx) * p_k
    raise ValueError(kind)


def solve(op, b, method="sflsqr", maxit=10, window=2, sketch=None, sketch_seed=0, d=None, s_nz=1,
          precond="identity", p_exp=1.0, eps_rel=1e-3, fixed_diag=None, tol=0.0, eta=0.0, delta_e=0.0,
          orth_mode="P", record=True):
    """Run sFLSQR / sFLSMR for at most maxit iterations.

    op: object with m, n, matvec(z) = A z, tmatvec(w) = T w.
    sketch: an object with .apply(v) (oracle.sketch.*); default: the sparse-sign
    sketch (sketch_seed, d, s_nz) on R^m (sFLSQR) or R^n (sFLSMR) - reading R4.
    """
    m, n = op.m, op.n
    b = np.asarray(b, dtype=np.float64)
    ell = int(window)
    if sketch is None:
        sketch = SparseSignSketch(sketch_seed, d, s_nz, m if method == "sflsqr" else n)
    S = sketch.apply

    # Alg. 1 L457-460 / Alg. 2
    beta = float(np.linalg.norm(b))
    if beta == 0.0:
        raise ValueError("||b|| = 0")
    W = [b / beta]
    z = op.tmatvec(W[0])
    if method == "sflsqr":
        rhs = S(b)                          # s_b = S b
        SAZ = []
    elif method == "sflsmr":
        Sz = S(z)
        rhs = beta * Sz                     # s_{A^T b} = beta S z
        STW = [rhs / beta]                  # S_{A^T W} = [s_{A^T b} / beta]
    else:
        raise ValueError(method)
    Z, P = [], []
    H = np.zeros((maxit + 1, maxit))
    Tm = np.zeros((maxit, maxit))
    res = OracleResult(x=np.zeros(n), k=0, status=RUNNING, rhs=rhs)
    x_prev = np.zeros(n)
    k_done = 0
    for k in range(1, maxit + 1):
        # L464-469: z-side windowed MGS + normalisation
        z_in = float(np.linalg.norm(z))
        for j in range(max(1, k - ell), k):
            qj = P[j - 1] if orth_mode == "P" else Z[j - 1]
            c = float(np.dot(qj, z))
            z = z - c * qj
            Tm[j - 1, k - 1] = c
        t = float(np.linalg.norm(z))
        if t == 0.0 or t <= 1e-14 * z_in:
            res.status = BREAKDOWN
            break
        Tm[k - 1, k - 1] = t
        p_k = z / t
        P.append(p_k)
        # L470-471: flexible preconditioner, Z = [Z, z_k]
        z_k = tau_apply(precond, p_k, x_prev, k, p_exp, eps_rel, fixed_diag)
        Z.append(z_k)
        # L473-474: w = A z_k; S_AZ = [S_AZ, S w]
        w = op.matvec(z_k)
        w_in = float(np.linalg.norm(w))
        if method == "sflsqr":
            SAZ.append(S(w))
        # L476-484: w-side windowed MGS
        for j in range(max(1, k - ell), k + 1):
            h = float(np.dot(W[j - 1], w))
            H[j - 1, k - 1] = h
            w = w - h * W[j - 1]
        hn = float(np.linalg.norm(w))
        w_breakdown = hn == 0.0 or hn <= 1e-14 * w_in
        if w_breakdown:
            # A z_k in span(W_k): H_{k+1,k} = 0, w_{k+1} := 0; y_k is still defined (R11)
            W.append(np.zeros(m))
            z = np.zeros(n)
        else:
            H[k, k - 1] = hn
            W.append(w / hn)
            # L486: z = A^T w_{k+1}
            z = op.tmatvec(W[k])
        # L488-490 / L790-797: projected sketched LS
        if method == "sflsqr":
            M = np.column_stack(SAZ)
        else:
            Sz = S(z)
            M = np.column_stack(STW + [Sz]) @ H[:k + 1, :k]
        y, _, ratio = householder_qr_solve(M, rhs)
        sres = float(np.linalg.norm(rhs - M @ y))
        Zk = np.column_stack(Z)
        x = Zk @ y                                   # L504 / L804: x_k = Z y_k
        k_done = k
        res.x, res.k = x, k
        res.sketch_res.append(sres)
        res.rank_ratio.append(ratio)
        r = float(np.linalg.norm(b - op.matvec(x)))  # eq. discrP residual
        res.true_res.append(r)
        if record:
            res.ys.append(y)
            res.xs.append(x)
        if w_breakdown:
            res.status = BREAKDOWN
            break
        # L498 / L798 (R3): tol test; eq. discrP (R12)
        if tol > 0.0 and sres < tol * float(np.linalg.norm(rhs)):
            res.status = TOL
            break
        if eta > 0.0 and r <= eta * delta_e:
            res.status = DISCREPANCY
            break
        if method == "sflsmr":
            STW.append(Sz)                           # L801
        x_prev = x
    else:
        res.status = MAXIT
    kk = len(Z)
    res.H = H[:k_done + 1, :k_done]
    res.T = Tm[:kk, :kk]
    res.Z = np.column_stack(Z) if Z else np.zeros((n, 0))
    res.P = np.column_stack(P) if P else np.zeros((n, 0))
    res.W = np.column_stack(W)
    if method == "sflsqr":
        res.sketch_cols = np.column_stack(SAZ) if SAZ else None
    else:
        res.sketch_cols = np.column_stack(STW)
    return res


def solve_problem(prob, spec, op=None, maxit=None, record=True, **over):
    """Convenience: run the oracle on a gen.Problem with a gen.SolverSpec."""
    from .operators import operator_from_problem
    if op is None:
        op = operator_from_problem(prob)
    kw = dict(method=spec.method, maxit=maxit or spec.maxit, window=spec.window, sketch_seed=prob.sketch_seed,
              d=spec.d, s_nz=spec.s_nz, precond=spec.precond, p_exp=spec.p, eps_rel=spec.eps_rel,
              tol=spec.tol, eta=spec.eta, delta_e=prob.delta_e, orth_mode=spec.orth_mode, record=record)
    kw.update(over)
    return solve(op, prob.b, **kw)
