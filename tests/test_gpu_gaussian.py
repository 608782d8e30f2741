"""GPU parity with the dense Gaussian sketch (reading R21): the
paper's synthetic rho-decay family (configs 6 / 7: PAPER.md L533-556, L1144-1152) and a
Gaussian-sketched CT run, through the C ABI against the fp64 oracle (oracle/sketch.py
GaussianSketch, pinned in tests/test_oracle_sketch.py).

The Gaussian entries come from log / sin / cos on both sides, so they agree to a few ulps,
not bitwise (the bit-exact bar of north_star is for the sparse-sign indices and signs);
iterates are held to the usual 1e-9 (residuals, within the oracle's stable horizon) and
1e-6 (x).
"""
import numpy as np
import pytest

from gen import make_problem
from oracle.operators import operator_from_problem
from oracle.sflsqr import solve_problem
from oracle.sketch import gaussian_table

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


@pytest.mark.parametrize("seed,d,col0,ncols", [(0x5F1A63, 101, 0, 1024), (7, 13, (1 << 33) + 5, 3000),
                                               (1 << 40, 400, 1043280 - 2000, 2000)])
def test_gaussian_entries_match_oracle(seed, d, col0, ncols):
    from paper_2605_22281_b200 import SFLSQR
    s = SFLSQR(maxit=1)
    s.set_sketch_gaussian(seed, d)
    got = s.debug_sketch_dense(col0, ncols)
    ref = gaussian_table(seed, d, col0, ncols)
    s.close()
    # log / cos / sin: a few ulps of the entry (scaled by the largest entry for entries near 0)
    err = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-3 * np.abs(ref).max())
    assert err.max() < 1e-14, err.max()


def _gpu_run(prob, spec, maxit):
    from paper_2605_22281_b200 import solver_for_problem
    s = solver_for_problem(prob, spec, maxit=maxit, eta=0.0)
    s.set_rhs(prob.b)
    done, status = s.iterate(maxit)
    tr, sk = s.get_residual_norms()
    x = s.get_x()
    info = s.get_info()
    s.close()
    return dict(status=status, true_res=tr, sketch_res=sk, x=x, info=info)


@pytest.mark.parametrize("cfg", [6, 7])
@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_decay_family(cfg, method):
    p = make_problem(cfg)
    spec = [s for s in p.solvers if s.method == method][0]
    kstar, _ = horizon(f"gauss/c{cfg}/{method}", p)
    r = solve_problem(p, spec, maxit=kstar, eta=0.0)
    g = _gpu_run(p, spec, kstar)
    assert g["info"]["k_done"] == len(r.true_res) and g["status"] == r.status
    rt = np.abs(g["true_res"] - np.array(r.true_res)) / np.array(r.true_res)
    rs = np.abs(g["sketch_res"] - np.array(r.sketch_res)) / np.array(r.sketch_res)
    assert rt.max() < RES_TOL and rs.max() < RES_TOL, (rt.max(), rs.max())
    assert np.linalg.norm(g["x"] - r.x) / np.linalg.norm(r.x) < X_TOL


def test_gaussian_sketch_on_ct():
    import dataclasses
    p = make_problem(3, N=96, n_angles=70, nb=137)
    spec = dataclasses.replace(p.solvers[0], sketch="gaussian", maxit=40, d=81)
    kstar, _ = horizon("gauss/ct", p)
    r = solve_problem(p, spec, maxit=kstar, eta=0.0)
    g = _gpu_run(p, spec, kstar)
    rt = np.abs(g["true_res"] - np.array(r.true_res)) / np.array(r.true_res)
    assert rt.max() < RES_TOL, rt.max()
    assert np.linalg.norm(g["x"] - r.x) / np.linalg.norm(r.x) < X_TOL
