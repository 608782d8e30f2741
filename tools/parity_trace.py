"""Per-iteration GPU-vs-oracle divergence trace (debug tool; test infrastructure)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from gen import make_problem
from oracle.sflsqr import solve_problem
from paper_2605_22281_b200 import solver_for_problem

def trace(p, spec, maxit=None, label=""):
    r = solve_problem(p, spec, maxit=maxit, eta=0.0)
    s = solver_for_problem(p, spec, maxit=maxit, eta=0.0)
    s.set_rhs(p.b)
    xs = []
    K = len(r.true_res)
    for k in range(1, K + 1):
        s.iterate(1)
        xs.append(s.get_x())
    tr, sk = s.get_residual_norms()
    s.close()
    rt = np.abs(tr - np.array(r.true_res)) / np.array(r.true_res)
    rs = np.abs(sk - np.array(r.sketch_res)) / np.array(r.sketch_res)
    ex = [np.linalg.norm(xs[k] - r.xs[k]) / np.linalg.norm(r.xs[k]) for k in range(K)]
    for k in list(range(0, K, max(1, K // 30))) + [K - 1]:
        print(f"{label} {spec.method} k={k+1:4d} true {rt[k]:.2e} sketch {rs[k]:.2e} x {ex[k]:.2e}")

which = sys.argv[1] if len(sys.argv) > 1 else "c3r"
if which == "c3r":
    p = make_problem(3, N=128, n_angles=90, nb=183)
    for spec in p.solvers:
        trace(p, spec, label="c3r")
elif which == "c4r":
    p = make_problem(4, N=192, n_angles=135, nb=273)
    trace(p, p.solvers[0], label="c4r")
elif which == "c1":
    p = make_problem(1)
    for spec in p.solvers:
        trace(p, spec, label="c1")

if which == "c3r_batch":
    p = make_problem(3, N=128, n_angles=90, nb=183)
    spec = p.solvers[0]
    r = solve_problem(p, spec, eta=0.0)
    import torch
    print("torch stream", torch.cuda.current_stream().cuda_stream)
    for use_graph in (True, False):
        for chunk in (150, 1, 7):
            s = solver_for_problem(p, spec, eta=0.0, use_graph=use_graph)
            s.set_rhs(p.b)
            for _ in range(0, 150, chunk):
                s.iterate(chunk)
            tr, sk = s.get_residual_norms()
            x = s.get_x()
            s.close()
            rt = np.abs(tr - np.array(r.true_res)) / np.array(r.true_res)
            bad = np.flatnonzero(rt > 1e-9)
            print(f"graph={use_graph} chunk={chunk}: max true-res err {rt.max():.2e} first>1e-9 at k={bad[0]+1 if bad.size else None}"
                  f" x err {np.linalg.norm(x - r.x)/np.linalg.norm(r.x):.2e}")

if which == "determinism":
    p = make_problem(3, N=128, n_angles=90, nb=183)
    spec = p.solvers[0]
    r = solve_problem(p, spec, eta=0.0)
    outs = []
    for rep in range(4):
        for use_graph, chunk in ((True, 150), (False, 7), (False, 150), (False, 1)):
            s = solver_for_problem(p, spec, eta=0.0, use_graph=use_graph)
            s.set_rhs(p.b)
            for _ in range(0, 150, chunk):
                s.iterate(chunk)
            tr, sk = s.get_residual_norms()
            x = s.get_x()
            s.close()
            rt = np.abs(tr - np.array(r.true_res)) / np.array(r.true_res)
            bad = np.flatnonzero(~(rt <= 1e-9))
            print(f"rep {rep} graph={use_graph} chunk={chunk}: nan={np.isnan(tr).any()} max err {np.nanmax(rt):.2e} "
                  f"first bad k={bad[0]+1 if bad.size else None} x err {np.linalg.norm(x - r.x)/np.linalg.norm(r.x):.2e}", flush=True)
            outs.append(tr)
    ref = outs[0]
    print("bitwise identical across runs:", [bool(np.array_equal(ref, o)) for o in outs])
