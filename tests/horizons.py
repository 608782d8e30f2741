"""The oracle's forward-stable horizons (reading R17), committed per parity case.

Some runs are not forward-stable in the oracle itself: a rounding-level perturbation moves its
residual history by more than the 1e-9 bar after some iteration k*, so no independent
implementation can be held to 1e-9 beyond k*.  The parity tests hold the GPU to the strict bar
up to k* and check later iterations by state injection.

k* = the last k at which the oracle's true residuals (the recurrence residuals for LSQR/LSMR)
move by < 1e-11 relative under
  * "b":        a 1e-15 relative perturbation of b (seeded), or
  * "products": a 2^-53 relative perturbation of every operator product (short recurrences).

The numbers in tests/golden/horizons.json were written by tools/compute_horizons.py, which calls
only gen/ and oracle/.  Each test recomputes k* on the box, asserts it is not shorter than the
committed value by more than 3 (host-to-host rounding of NumPy's reductions) and holds the GPU to
the strict bar over min(k*, committed) iterations, so a change that shrinks a strict window shows
up as a failure, not as a silently shorter window.
"""
import json
import os

import numpy as np

from gen import make_problem
from gen.problems import CSR, Problem, SolverSpec
from oracle.operators import operator_from_problem
from oracle.sflsqr import solve_problem

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "horizons.json")
THRESH = 1e-11


def dense_prob(m, n, seed=0, cond=1e3):
    """Seeded dense test problem U diag(logspace) V^T with 2 % exact-norm noise."""
    rng = np.random.default_rng(seed)
    U = np.linalg.qr(rng.standard_normal((m, min(m, n))))[0]
    V = np.linalg.qr(rng.standard_normal((n, min(m, n))))[0]
    A = (U * np.logspace(0, -np.log10(cond), min(m, n))) @ V.T
    x = rng.standard_normal(n)
    e = rng.standard_normal(m)
    b = A @ x
    e *= 0.02 * np.linalg.norm(b) / np.linalg.norm(e)
    return Problem(name="dense", config_index=0, m=m, n=n, A=CSR.from_dense(A), T=None, t_mode="build", blur=None,
                   x_true=x, b=b + e, e=e, delta=0.02, delta_e=float(np.linalg.norm(e)), sketch_seed=1234 + seed)


EDGE_CASES = [  # (m, n, method, window, precond, orth, s_nz, d): test_gpu_parity.test_edge_configurations
    (37, 29, "sflsqr", 1, "irn", "P", 1, 25),
    (64, 40, "sflsmr", 50, "identity", "P", 3, 30),
    (90, 70, "sflsqr", 3, "nonneg", "Z", 8, 41),
    (90, 70, "sflsmr", 2, "irn", "Z", 4, 21),
    (300, 1000, "sflsqr", 2, "irn", "P", 8, 21),
    (1025, 513, "sflsmr", 4, "nonneg", "P", 2, 20),
]
MAXSIZE_CASES = [("sflsqr", 1500, 30, 3), ("sflsmr", 2048, 24, 2), ("sflsqr", 700, 600, 5)]

C5R = dict(N=256, n_angles=180, nb=363)      # config 5's recipe at 1/8 of its grid side (reduced C5)


def _registry():
    """key -> (problem factory, spec or solver method name, maxit, oracle method override, perturbation)."""
    import dataclasses
    reg = {}
    for i, (m, n, method, window, precond, orth, s_nz, d) in enumerate(EDGE_CASES):
        spec = SolverSpec(method=method, maxit=20, window=window, d=d, s_nz=s_nz, precond=precond, orth_mode=orth)
        reg[f"edge/{i}"] = ((lambda m=m, n=n: dense_prob(m, n, seed=m + n)), spec, 20, None, "b")
    for i, (method, d, maxit, window) in enumerate(MAXSIZE_CASES):
        spec = SolverSpec(method=method, maxit=maxit, window=window, d=d, s_nz=8, precond="irn")
        reg[f"maxsize/{i}"] = ((lambda d=d, maxit=maxit: dense_prob(1600, 900, seed=d + maxit, cond=1e2)), spec,
                               min(maxit, 40), None, "b")
    c3r128 = lambda: make_problem(3, N=128, n_angles=90, nb=183)           # noqa: E731
    c4r160 = lambda: make_problem(4, N=160, n_angles=113, nb=227)          # noqa: E731
    c8r128 = lambda: make_problem(8, N=128)                                # noqa: E731
    reg.update({
        # sFLSQR / sFLSMR (test_gpu_parity.py)
        "c2/sflsqr": (lambda: make_problem(2), "sflsqr", 100, None, "b"),
        "c3full/sflsqr": (lambda: make_problem(3), "sflsqr", 30, None, "b"),
        "c3full/sflsmr": (lambda: make_problem(3), "sflsmr", 30, None, "b"),
        "c4r192/sflsqr": (lambda: make_problem(4, N=192, n_angles=135, nb=273), "sflsqr", 60, None, "b"),
        "c4full/sflsqr": (lambda: make_problem(4), "sflsqr", 25, None, "b"),
        "c5r/sflsqr": (lambda: make_problem(5, **C5R), "sflsqr", 150, None, "b"),
        "c5r/sflsmr": (lambda: make_problem(5, **C5R), "sflsmr", 150, None, "b"),
        # FLSQR / FLSMR (test_gpu_flsqr.py: the spec of solvers[0], oracle method overridden)
        "flsqr/c1/flsqr": (lambda: make_problem(1), "sflsqr", 40, "flsqr", "b"),
        "flsqr/c1/flsmr": (lambda: make_problem(1), "sflsqr", 40, "flsmr", "b"),
        "flsqr/c3r128/flsqr": (c3r128, "sflsqr", 60, "flsqr", "b"),
        "flsqr/c3r128/flsmr": (c3r128, "sflsqr", 60, "flsmr", "b"),
        "flsqr/c4r160/flsqr": (c4r160, "sflsqr", 50, "flsqr", "b"),
        "flsqr/c4r160/flsmr": (c4r160, "sflsqr", 50, "flsmr", "b"),
        "flsqr/c2/flsqr": (lambda: make_problem(2), "sflsqr", 40, "flsqr", "b"),
        "flsqr/c2/flsmr": (lambda: make_problem(2), "sflsqr", 40, "flsmr", "b"),
        # Gaussian sketch (test_gpu_gaussian.py)
        "gauss/c6/sflsqr": (lambda: make_problem(6), "sflsqr", 50, None, "b"),
        "gauss/c6/sflsmr": (lambda: make_problem(6), "sflsmr", 50, None, "b"),
        "gauss/c7/sflsqr": (lambda: make_problem(7), "sflsqr", 50, None, "b"),
        "gauss/c7/sflsmr": (lambda: make_problem(7), "sflsmr", 50, None, "b"),
        "gauss/ct": ((lambda: make_problem(3, N=96, n_angles=70, nb=137)),
                     (lambda p: dataclasses.replace(p.solvers[0], sketch="gaussian", maxit=40, d=81)), 40, None, "b"),
        # tau_r by randomized SVD (test_gpu_lowrank.py)
        "lowrank/c8r128/sflsqr": (c8r128, "sflsqr", 50, None, "b"),
        "lowrank/c8r128/sflsmr": (c8r128, "sflsmr", 50, None, "b"),
        "lowrank/c8/sflsqr": (lambda: make_problem(8), "sflsqr", 30, None, "b"),
        "lowrank/c8/sflsmr": (lambda: make_problem(8), "sflsmr", 30, None, "b"),
        "lowrank/c8r128/flsqr": (c8r128, (lambda p: dataclasses.replace(p.solvers[0], maxit=30)), 30, "flsqr", "b"),
    })
    # textbook LSQR / LSMR (test_gpu_gkb.py): every product perturbed
    for tag, mk, maxit in (("c1", lambda: make_problem(1), 40), ("c2", lambda: make_problem(2), 60),
                           ("c3r128", c3r128, 80), ("c4r160", c4r160, 80)):
        for meth in ("lsqr", "lsmr"):
            reg[f"gkb/{tag}/{meth}"] = (mk, "sflsqr", maxit, meth, "products")
    return reg


def all_keys():
    return list(_registry())


def _resolve(key, p):
    mk, sp, maxit, meth, mode = _registry()[key]
    if p is None:
        p = mk()
    if isinstance(sp, str):
        spec = [s for s in p.solvers if s.method == sp][0]
    elif callable(sp):
        spec = sp(p)
    else:
        spec = sp
    return p, spec, maxit, meth, mode


class _Noisy:
    """The oracle's operator with a 2^-53-scale relative perturbation of every product result
    (models another implementation's summation order)."""

    def __init__(self, op, seed=0):
        self.op, self.m, self.n = op, op.m, op.n
        self.rng = np.random.default_rng(seed)

    def matvec(self, v):
        y = self.op.matvec(v)
        return y * (1 + 2.0 ** -53 * self.rng.standard_normal(y.size))

    def tmatvec(self, w):
        y = self.op.tmatvec(w)
        return y * (1 + 2.0 ** -53 * self.rng.standard_normal(y.size))


def stable_horizon(p, spec, maxit, method=None, mode="b", thresh=THRESH, op=None):
    """(k*, the unperturbed oracle run to maxit).  Pure oracle: gen/ inputs, oracle/ arithmetic."""
    op = op or operator_from_problem(p)
    kw = {} if method is None else dict(method=method)
    r0 = solve_problem(p, spec, op=op, maxit=maxit, eta=0.0, **kw)
    if mode == "products":
        r1 = solve_problem(p, spec, op=_Noisy(op), maxit=maxit, eta=0.0, **kw)
        dev = np.abs(np.array(r1.est_res) - np.array(r0.est_res)) / np.array(r0.est_res)
        if method == "lsmr":                              # ||T r|| is the more sensitive history
            dev = np.maximum(dev, np.abs(np.array(r1.est_nres) - np.array(r0.est_nres)) / np.array(r0.est_nres))
    else:
        b0 = p.b
        p.b = b0 * (1 + 1e-15 * np.random.default_rng(0).standard_normal(b0.size))
        try:
            r1 = solve_problem(p, spec, op=op, maxit=maxit, eta=0.0, **kw)
        finally:
            p.b = b0
        dev = np.abs(np.array(r1.true_res) - np.array(r0.true_res)) / np.array(r0.true_res)
    bad = np.flatnonzero(dev > thresh)
    return (int(bad[0]) if bad.size else len(dev)), r0


def committed(key):
    with open(GOLDEN) as f:
        return int(json.load(f)["horizons"][key])


def case(key):
    """(problem, spec, maxit, oracle method) of a committed case."""
    p, spec, maxit, meth, _ = _resolve(key, None)
    return p, spec, maxit, meth


def truncate(r, k):
    """The oracle run r (recorded, unstopped through k) as if it had been run with maxit = k."""
    import dataclasses
    from oracle.sflsqr import MAXIT
    if len(r.true_res) == k:
        return r
    assert len(r.true_res) > k and r.xs, (len(r.true_res), k)
    ncols = k + 1 if r.method == "sflsmr" else k
    return dataclasses.replace(
        r, x=r.xs[k - 1], k=k, status=MAXIT, true_res=r.true_res[:k], sketch_res=r.sketch_res[:k], ys=r.ys[:k],
        xs=r.xs[:k], rank_ratio=r.rank_ratio[:k], H=None if r.H is None else r.H[:k + 1, :k],
        sketch_cols=None if r.sketch_cols is None else r.sketch_cols[:, :ncols])


def horizon(key, p=None, op=None, slack=3):
    """Recompute k* for a committed case on this host and check it against the committed value.

    The oracle runs to min(case maxit, committed + 1).  Its arithmetic is host-independent up to
    NumPy's CPU-dispatched SIMD reductions (OpenBLAS is pinned in conftest.py), which move k* by up
    to 3 iterations between this container and the GPU box (measured: config 5 reduced 96 / 99,
    config 8 reduced 19 / 22).  The check is one-sided -- k* >= committed - slack: a change that
    shortens the oracle's stable window fails, a host on which it is longer passes.  The strict
    window is min(k*, committed).  Returns (window, the unperturbed oracle run truncated to it)."""
    p, spec, maxit, meth, mode = _resolve(key, p)
    want = committed(key)
    run_to = min(maxit, want + 1)
    kstar, r0 = stable_horizon(p, spec, run_to, meth, mode, op=op)
    print(f"horizon {key}: k* = {kstar} (committed {want}, run to {run_to})")
    assert kstar >= want - slack, (key, kstar, want)
    window = min(kstar, want)
    from oracle.sflsqr import OracleResult
    return window, (truncate(r0, window) if isinstance(r0, OracleResult) else r0)
