"""Small eager + graph run for compute-sanitizer (debug tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from gen import make_problem
from paper_2605_22281_b200 import solver_for_problem
p = make_problem(3, N=48, n_angles=30, nb=69)
for spec in p.solvers:
    for g in (False, True):
        s = solver_for_problem(p, spec, maxit=12, eta=0.0, use_graph=g)
        s.set_rhs(p.b)
        s.iterate(5); s.iterate(7)
        x = s.get_x(); tr, sk = s.get_residual_norms()
        s.close()
        print(spec.method, g, tr[-1], np.linalg.norm(x))
