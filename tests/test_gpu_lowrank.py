"""GPU parity of the low-rank truncation tau_r by randomized SVD (reading R22; SURVEY.md §8(f)
NEXT-2; PAPER.md eq. def:lowr-trc L77-81, sFLSQR-RND / sFLSMR-RND L1619-1623) on the
deblurring + inpainting workload (config 8), through the C ABI against the
fp64 oracle (oracle/lowrank.py, pinned in tests/test_oracle_lowrank.py).
"""
import dataclasses

import numpy as np
import pytest

from gen import make_problem
from oracle.lowrank import rnd_omega, tau_lowrank_rnd
from oracle.operators import operator_from_problem
from oracle.sflsqr import solve_problem

from horizons import horizon

pytestmark = pytest.mark.gpu

RES_TOL = 1e-9
X_TOL = 1e-6


@pytest.fixture(scope="session", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_22281_b200._build import build_library
    build_library()


def _gpu(prob, spec, maxit, method=None):
    from paper_2605_22281_b200 import solver_for_problem
    s = solver_for_problem(prob, spec, maxit=maxit, eta=0.0, method=method)
    s.set_rhs(prob.b)
    s.iterate(maxit)
    tr, sk = s.get_residual_norms()
    out = dict(true_res=tr, sketch_res=sk, x=s.get_x(), info=s.get_info(), basis=s.debug_basis())
    s.close()
    return out


def test_first_basis_vector_is_rnd_truncation():
    p = make_problem(8, N=128)
    spec = p.solvers[0]
    g = _gpu(p, spec, 1)
    lr = spec.lowrank
    op = operator_from_problem(p)
    z = op.tmatvec(p.b / np.linalg.norm(p.b))
    ref = tau_lowrank_rnd(z / np.linalg.norm(z), lr["N"], lr["r"], rnd_omega(lr["seed"], lr["N"], lr["r"], lr["oversample"]))
    got = g["basis"]["Z"][:, 0]
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.linalg.svd(got.reshape(lr["N"], lr["N"]), compute_uv=False)[lr["r"]] < 1e-12 * np.linalg.norm(got)


@pytest.mark.parametrize("N", [128, 512])
@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_deblur_inpaint_rnd(N, method):
    p = make_problem(8, N=N)
    spec = [s for s in p.solvers if s.method == method][0]
    kstar, _ = horizon(f"lowrank/{'c8' if N == 512 else 'c8r128'}/{method}", p)
    r = solve_problem(p, spec, maxit=kstar, eta=0.0)
    g = _gpu(p, spec, kstar)
    rt = np.abs(g["true_res"] - np.array(r.true_res)) / np.array(r.true_res)
    rs = np.abs(g["sketch_res"] - np.array(r.sketch_res)) / np.array(r.sketch_res)
    assert rt.max() < RES_TOL and rs.max() < RES_TOL, (kstar, rt.max(), rs.max())
    assert np.linalg.norm(g["x"] - r.x) / np.linalg.norm(r.x) < X_TOL


def test_flsqr_rnd():
    p = make_problem(8, N=128)
    spec = dataclasses.replace(p.solvers[0], maxit=30)
    kstar, _ = horizon("lowrank/c8r128/flsqr", p)
    r = solve_problem(p, spec, maxit=kstar, eta=0.0, method="flsqr")
    g = _gpu(p, spec, kstar, method="flsqr")
    rt = np.abs(g["true_res"] - np.array(r.true_res)) / np.array(r.true_res)
    assert rt.max() < RES_TOL, (kstar, rt.max())
