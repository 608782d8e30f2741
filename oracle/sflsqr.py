"""sFLSQR (Algorithm 1) and sFLSMR (Algorithm 2), plain fp64, followed line by line;
and their unsketched full-orthogonalisation parents FLSQR / FLSMR (SURVEY.md §8(f)
NEXT-1), which share the same flexible Golub-Kahan step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Sources:
  * Alg. 1 sFLSQR, L450-508; eq. sFLSQR; eq. FGK (partial flexible
    Golub-Kahan with window ell) L400-406; cost L444-448.
  * Alg. 2 sFLSMR, L752-808; eq. sFLSMR L730-749 ("compute the columns of
    S A^T W ... then right-multiply by H ... implemented in our code").
  * FLSQR eq. (FLSQR): x_k = Z_k y_k, y_k = argmin || ||b|| e_1 - H_{k+1,k} y ||,
    on the FGK factorisation eq. (flsqr-relations) L335-345 with FULL
    orthogonalisation (P_k, W_{k+1} orthonormal; T_k, H_{k+1,k} fill up, L344-345).
  * FLSMR L359-368: y_k = argmin || T_{k+1} ( ||b|| e_1 - H_{k+1,k} y ) ||, where
    T_{k+1} is the (k+1) x (k+1) upper-triangular factor of A^T W_{k+1} = P_{k+1} T_{k+1}:
    its last column is the orthogonalisation of z = A^T w_{k+1} against p_1..p_k,
    i.e. the first half of FGK step k+1 (Alg. 1 L464-469 with k -> k+1), computed here
    at the end of step k by the same code that step k+1 then repeats.
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
      Pinned (tests/test_oracle_precond.py): sum (x/D)^2 -> ||x||_p^p as eps -> 0, and
      x / D^2 = the gradient of (1/p) sum (x^2 + eps^2)^{p/2} (the IRLS weights, L59-64).
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
    method: str = ""                 # bookkeeping: which algorithm produced the run


def tau_apply(kind, p_k, x_prev, k, p_exp=1.0, eps_rel=1e-3, fixed=None):
    """z_k = tau_k(p_k) (Alg. 1 L470 / Alg. 2; readings R7, R8, R22).
    fixed: the diagonal of kind "diag", or the dict (N, r, omega) of the low-rank kinds."""
    if kind == "identity":
        return p_k.copy()
    if kind == "diag":                     # fixed SPD diagonal (pin P4b)
        return fixed * p_k
    if kind == "lowrank":                  # eq. def:lowr-trc L77-81, truncated SVD
        from .lowrank import tau_lowrank_exact
        return tau_lowrank_exact(p_k, fixed["N"], fixed["r"])
    if kind == "lowrank_rnd":              # randomized SVD (L1619-1623, reading R22)
        from .lowrank import tau_lowrank_rnd
        return tau_lowrank_rnd(p_k, fixed["N"], fixed["r"], fixed["omega"])
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


class FGKState:
    """Everything Alg. 1 / Alg. 2 carry from one iteration to the next."""

    def __init__(self, m, n, maxit, method, rhs, beta, b):
        self.m, self.n, self.method = m, n, method
        self.W, self.Z, self.P = [], [], []            # w_1.., z_1.., p_1..
        self.z = None                                  # current T w_k (before the z-orthogonalisation)
        self.x_prev = np.zeros(n)                      # x_{k-1} (tau needs it)
        self.H = np.zeros((maxit + 1, maxit))
        self.Tm = np.zeros((maxit, maxit))
        self.SAZ = []                                  # sFLSQR: columns S A z_j
        self.STW = []                                  # sFLSMR: columns S T w_j
        self.rhs, self.beta, self.b = rhs, beta, b


def init_state(op, b, method, maxit, S):
    """Alg. 1 L457-460 / Alg. 2 L759-763."""
    b = np.asarray(b, dtype=np.float64)
    beta = float(np.linalg.norm(b))
    if beta == 0.0:
        raise ValueError("||b|| = 0")
    w1 = b / beta
    z = op.tmatvec(w1)
    if method == "sflsqr":
        rhs = S(b)                          # s_b = S b
    elif method == "sflsmr":
        Sz = S(z)
        rhs = beta * Sz                     # s_{A^T b} = beta S z
    elif method == "flsqr":
        rhs = np.zeros(maxit + 1)           # ||b|| e_1 (eq. FLSQR)
        rhs[0] = beta
    elif method == "flsmr":
        rhs = None                          # ||b|| T_{k+1} e_1 = ||b|| T_11 e_1, T_11 known after step 1's L469
    else:
        raise ValueError(method)
    st = FGKState(op.m, op.n, maxit, method, rhs, beta, b)
    st.W.append(w1)
    st.z = z
    if method == "sflsmr":
        st.STW.append(rhs / beta)           # S_{A^T W} = [s_{A^T b} / beta]
    return st


def z_orthogonalise(st, k, ell, orth_mode, z):
    """Alg. 1 L464-469 / Alg. 2 L767-772 for step k: windowed MGS of z = T w_k against
    q_j (j = max(1, k-ell) .. k-1) and its norm.  Returns (coefficients {j: c}, t, z_perp)."""
    coeffs = {}
    for j in range(max(1, k - ell), k):
        qj = st.P[j - 1] if orth_mode == "P" else st.Z[j - 1]
        c = float(np.dot(qj, z))
        z = z - c * qj
        coeffs[j] = c
    return coeffs, float(np.linalg.norm(z)), z


def fgk_step(op, st, k, ell, S, precond="identity", p_exp=1.0, eps_rel=1e-3, fixed_diag=None, orth_mode="P"):
    """Iteration k of Alg. 1 (L462-496) / Alg. 2 (L765-797), updating st in place.

    Returns a dict of the step's outputs, or {"breakdown": "z"} when z_k cannot be formed (R11).
    """
    m, n = st.m, st.n
    out = {}
    # L464-469: z-side windowed MGS + normalisation
    z_in = float(np.linalg.norm(st.z))
    coeffs, t, z = z_orthogonalise(st, k, ell, orth_mode, st.z)
    for j, c in coeffs.items():
        st.Tm[j - 1, k - 1] = c
    if t == 0.0 or t <= 1e-14 * z_in:
        return {"breakdown": "z"}
    st.Tm[k - 1, k - 1] = t
    p_k = z / t
    st.P.append(p_k)
    # L470-471: flexible preconditioner, Z = [Z, z_k]
    z_k = tau_apply(precond, p_k, st.x_prev, k, p_exp, eps_rel, fixed_diag)
    st.Z.append(z_k)
    # L473-474: w = A z_k; S_AZ = [S_AZ, S w]
    w = op.matvec(z_k)
    w_in = float(np.linalg.norm(w))
    if st.method == "sflsqr":
        st.SAZ.append(S(w))
    # L476-484: w-side windowed MGS
    for j in range(max(1, k - ell), k + 1):
        h = float(np.dot(st.W[j - 1], w))
        st.H[j - 1, k - 1] = h
        w = w - h * st.W[j - 1]
    hn = float(np.linalg.norm(w))
    w_breakdown = hn == 0.0 or hn <= 1e-14 * w_in
    if w_breakdown:
        # A z_k in span(W_k): H_{k+1,k} = 0, w_{k+1} := 0; y_k is still defined (R11)
        st.W.append(np.zeros(m))
        st.z = np.zeros(n)
    else:
        st.H[k, k - 1] = hn
        st.W.append(w / hn)
        # L486: z = A^T w_{k+1}
        st.z = op.tmatvec(st.W[k])
    # L488-490 / L790-797: projected sketched LS
    if st.method == "sflsqr":
        M = np.column_stack(st.SAZ)
    elif st.method == "sflsmr":
        Sz = S(st.z)
        M = np.column_stack(st.STW + [Sz]) @ st.H[:k + 1, :k]
        out["Sz"] = Sz
    elif st.method == "flsqr":
        M = st.H[:k + 1, :k]                                  # eq. FLSQR
        st.rhs_k = st.rhs[:k + 1]
    else:                                                     # FLSMR L361-367
        if k == 1:
            st.rhs = np.zeros(st.H.shape[0])
            st.rhs[0] = st.beta * st.Tm[0, 0]                 # ||b|| T_{k+1} e_1 (T upper triangular)
        Tk1 = np.zeros((k + 1, k + 1))
        Tk1[:k, :k] = st.Tm[:k, :k]
        coeffs, t1, _ = z_orthogonalise(st, k + 1, ell, orth_mode, st.z)  # column k+1 of T (step k+1's L464-469)
        for j, c in coeffs.items():
            Tk1[j - 1, k] = c
        Tk1[k, k] = t1
        M = Tk1 @ st.H[:k + 1, :k]
        st.rhs_k = st.rhs[:k + 1]
    rhs_k = st.rhs_k if st.method in ("flsqr", "flsmr") else st.rhs
    y, _, ratio = householder_qr_solve(M, rhs_k)
    sres = float(np.linalg.norm(rhs_k - M @ y))
    x = np.column_stack(st.Z) @ y                 # L504 / L804: x_k = Z y_k
    r = float(np.linalg.norm(st.b - op.matvec(x)))  # eq. discrP residual (R12)
    out.update(p=p_k, z=z_k, w_next=st.W[k], Tcol=st.Tm[:k, k - 1].copy(), Hcol=st.H[:k + 1, k - 1].copy(),
               Mcol=M[:, -1].copy(), M=M, y=y, sres=sres, x=x, r=r, ratio=ratio, w_breakdown=w_breakdown)
    return out


def solve(op, b, method="sflsqr", maxit=10, window=2, sketch=None, sketch_seed=0, d=None, s_nz=1,
          precond="identity", p_exp=1.0, eps_rel=1e-3, fixed_diag=None, tol=0.0, eta=0.0, delta_e=0.0,
          orth_mode="P", record=True):
    """Run sFLSQR / sFLSMR (sketched, window ell) or FLSQR / FLSMR (full orthogonalisation,
    no sketch; `window`, `sketch*` ignored) for at most maxit iterations.

    op: object with m, n, matvec(z) = A z, tmatvec(w) = T w.
    sketch: an object with .apply(v) (oracle.sketch.*); default: the sparse-sign
    sketch (sketch_seed, d, s_nz) on R^m (sFLSQR) or R^n (sFLSMR) - reading R4.
    """
    m, n = op.m, op.n
    ell = int(window)
    if method in ("flsqr", "flsmr"):
        ell = max(ell, maxit + 1)             # full orthogonalisation (L344-345); no sketch
        S = None
    else:
        if sketch is None:
            sketch = SparseSignSketch(sketch_seed, d, s_nz, m if method == "sflsqr" else n)
        S = sketch.apply
    st = init_state(op, b, method, maxit, S)
    res = OracleResult(x=np.zeros(n), k=0, status=RUNNING, rhs=st.rhs, method=method)
    k_done = 0
    for k in range(1, maxit + 1):
        out = fgk_step(op, st, k, ell, S, precond, p_exp, eps_rel, fixed_diag, orth_mode)
        if out.get("breakdown") == "z":
            res.status = BREAKDOWN
            break
        x, sres, r = out["x"], out["sres"], out["r"]
        k_done = k
        res.x, res.k = x, k
        res.sketch_res.append(sres)
        res.rank_ratio.append(out["ratio"])
        res.true_res.append(r)
        if record:
            res.ys.append(out["y"])
            res.xs.append(x)
        if out["w_breakdown"]:
            res.status = BREAKDOWN
            break
        # L498 / L798 (R3): tol test; eq. discrP (R12)
        if tol > 0.0 and sres < tol * float(np.linalg.norm(st.rhs)):
            res.status = TOL
            break
        if eta > 0.0 and r <= eta * delta_e:
            res.status = DISCREPANCY
            break
        if method == "sflsmr":
            st.STW.append(out["Sz"])                 # L801
        st.x_prev = x
    else:
        res.status = MAXIT
    kk = len(st.Z)
    res.H = st.H[:k_done + 1, :k_done]
    res.T = st.Tm[:kk, :kk]
    res.Z = np.column_stack(st.Z) if st.Z else np.zeros((n, 0))
    res.P = np.column_stack(st.P) if st.P else np.zeros((n, 0))
    res.W = np.column_stack(st.W)
    if method == "sflsqr":
        res.sketch_cols = np.column_stack(st.SAZ) if st.SAZ else None
    elif method == "sflsmr":
        res.sketch_cols = np.column_stack(st.STW)
    res.rhs = st.rhs
    return res


def step_from_state(op, b, method, k, window, sketch, Z_prev, P_window, W_prev, z, x_prev, H_prev, sketch_prev,
                    rhs, precond="identity", p_exp=1.0, eps_rel=1e-3, orth_mode="P"):
    """State injection: run iteration k of Alg. 1/2 from an externally supplied state.

    Z_prev: n x (k-1) (z_1..z_{k-1}); P_window: {j: p_j} for the last ell j < k;
    W_prev: m x k (w_1..w_k); z = T w_k; x_prev = x_{k-1}; H_prev: k x (k-1);
    sketch_prev: d x (k-1) (S A z_j, sFLSQR) or d x k (S T w_j, sFLSMR); rhs: s_b / s_{A^T b}.
    """
    maxit = k
    st = FGKState(op.m, op.n, maxit, method, np.asarray(rhs, dtype=np.float64), float(np.linalg.norm(b)),
                  np.asarray(b, dtype=np.float64))
    col = lambda M, j: np.ascontiguousarray(M[:, j], dtype=np.float64)  # noqa: E731
    st.Z = [col(Z_prev, j) for j in range(Z_prev.shape[1])]
    st.P = [None if P_window.get(j + 1) is None else np.ascontiguousarray(P_window[j + 1], dtype=np.float64)
            for j in range(k - 1)]                             # only the window entries are used
    st.W = [col(W_prev, j) for j in range(W_prev.shape[1])]
    st.z = np.asarray(z, dtype=np.float64)
    st.x_prev = np.asarray(x_prev, dtype=np.float64)
    st.H[:k, :k - 1] = H_prev
    if method == "sflsqr":
        st.SAZ = [col(sketch_prev, j) for j in range(sketch_prev.shape[1])]
    else:
        st.STW = [col(sketch_prev, j) for j in range(sketch_prev.shape[1])]
    return fgk_step(op, st, k, int(window), sketch.apply, precond, p_exp, eps_rel, None, orth_mode)


def solve_problem(prob, spec, op=None, maxit=None, record=True, **over):
    """Convenience: run the oracle on a gen.Problem with a gen.SolverSpec."""
    from .operators import operator_from_problem
    if op is None:
        op = operator_from_problem(prob)
    method = over.pop("method", spec.method)
    if method in ("lsqr", "lsmr"):                      # textbook GKB baselines (oracle/gkb.py)
        from . import gkb
        eta = over.pop("eta", spec.eta)
        fn = gkb.lsqr if method == "lsqr" else gkb.lsmr
        return fn(op, prob.b, maxit=maxit or spec.maxit, eta=eta, delta_e=prob.delta_e,
                  record=over.pop("record", record))
    over["method"] = method
    if getattr(spec, "sketch", "sparse") == "gaussian" and method in ("sflsqr", "sflsmr") and "sketch" not in over:
        from .sketch import GaussianSketch                 # reading R21
        over["sketch"] = GaussianSketch(prob.sketch_seed, spec.d, prob.m if method == "sflsqr" else prob.n)
    if spec.precond in ("lowrank", "lowrank_rnd") and "fixed_diag" not in over:
        from .lowrank import rnd_omega                     # reading R22
        lr = spec.lowrank
        over["fixed_diag"] = dict(N=lr["N"], r=lr["r"], omega=rnd_omega(lr["seed"], lr["N"], lr["r"], lr["oversample"]))
    kw = dict(method=spec.method, maxit=maxit or spec.maxit, window=spec.window, sketch_seed=prob.sketch_seed,
              d=spec.d, s_nz=spec.s_nz, precond=spec.precond, p_exp=spec.p, eps_rel=spec.eps_rel,
              tol=spec.tol, eta=spec.eta, delta_e=prob.delta_e, orth_mode=spec.orth_mode, record=record)
    kw.update(over)
    return solve(op, prob.b, **kw)
