"""Small eager + graph runs for compute-sanitizer (debug tool): every method, the pair formats
(rows >= 64 nonzeros), the low-rank tau_r, the Gaussian sketch."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from gen import make_problem
from paper_2605_22281_b200 import solver_for_problem


def run(p, spec, maxit, method=None, graph=True, tune=None):
    s = solver_for_problem(p, spec, maxit=maxit, eta=0.0, use_graph=graph, knobs=["keep_csr"] if tune else [],
                           **({} if method is None else dict(method=method)))
    if tune is not None:
        s.debug_set_tuning(tune)
    s.set_rhs(p.b)
    s.iterate(maxit // 2); s.iterate(maxit - maxit // 2)
    x = s.get_x(); tr, sk = s.get_residual_norms()
    inf = s.get_info()
    s.close()
    print(spec.method if method is None else method, graph, tune, inf["a_fmt"], inf["t_fmt"], tr[-1], np.linalg.norm(x), flush=True)


p = make_problem(4, N=64, n_angles=45, nb=91)          # rows >= 64 nnz: pair formats
spec = p.solvers[0]
for m in ("sflsqr", "sflsmr", "flsqr", "flsmr", "lsqr", "lsmr"):
    for g in (False, True):
        run(p, spec, 10, method=m, graph=g)
for t in (14, 16, 17):
    run(p, spec, 8, tune=t)
p3 = make_problem(3, N=48, n_angles=30, nb=69)
for spec in p3.solvers:
    run(p3, spec, 12)
p8 = make_problem(8, N=64)
run(p8, p8.solvers[0], 10)
p6 = make_problem(6)
run(p6, p6.solvers[0], 8)
