import os, sys, numpy as np
sys.path.insert(0, '.')
from gen import make_problem
from oracle.sflsqr import solve_problem
from paper_2605_22281_b200 import solver_for_problem
from paper_2605_22281_b200._build import build_library
build_library()
p = make_problem(8, N=128)
spec = [s for s in p.solvers if s.method == 'sflsqr'][0]
r = solve_problem(p, spec, maxit=25, eta=0.0)
s = solver_for_problem(p, spec, maxit=25, eta=0.0)
s.set_rhs(p.b); s.iterate(25)
tr, sk = s.get_residual_norms(); s.close()
rt = np.abs(tr - np.array(r.true_res)) / np.array(r.true_res)
print(os.environ.get('SFLSQR_LR_QR', 'chol'), ' '.join('%.0e' % v for v in rt))
