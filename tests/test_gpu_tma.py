"""GPU: the TMA-staged aligned pair-CSR product (SFLSQR_KNOB_TMA, k_spmv_tma).

Its streams reach shared memory by cp.async.bulk behind mbarriers, and the lanes sum each row in
the order of the full-warp register kernel: products and whole solves are bitwise equal to that
kernel, and within rounding of the half-warp kernel and of the oracle's products.  Edge cases:
empty rows, rows of only pairs or only singletons, ragged chunk tails, stream ranges starting at
every residue mod 4 (the copy ranges widened to 16-byte boundaries), more rows than warps.
"""
import numpy as np
import pytest

from gen import make_problem
from oracle.operators import OracleCSR
from oracle.sflsqr import solve_problem

from horizons import C5R
from test_gpu_parity import _compare, _gpu_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_22281_b200._build import build_library
    build_library()


def _product(M, z, knobs, tuning=None):
    from paper_2605_22281_b200 import SFLSQR
    s = SFLSQR(maxit=4, knobs=knobs)
    s.set_operator(M.nrows, M.ncols, M.rowptr, M.col, M.val)
    if tuning is not None:
        s.debug_set_tuning(spmv_mode=tuning)
    info = s.get_info()
    y = s.debug_apply(0, z)
    s.close()
    return y, info


def _ragged_runs(m, n, seed):
    """Rows of runs of consecutive columns (pairs and singletons), lengths 0 .. ~700, some empty,
    some with one long run only (pairs only), some with isolated columns only (singletons only)."""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(m):
        kind = (i + 1) % 7  # row 0: pairs only (the format has pairs even at m = 1)
        if kind == 0:
            rows.append(np.zeros(0, dtype=np.int64))
            continue
        if kind == 1:  # one even-aligned run: pairs only
            c0 = 2 * int(rng.integers(0, n // 2 - 400))
            rows.append(np.arange(c0, c0 + 2 * int(rng.integers(1, 200))))
            continue
        if kind == 2:  # isolated columns, every other column: singletons only
            k = int(rng.integers(1, 300))
            c = np.sort(rng.choice(n // 2, size=k, replace=False)) * 2
            rows.append(c)
            continue
        cols = set()
        for _ in range(int(rng.integers(1, 60))):
            c0 = int(rng.integers(0, n - 16))
            cols.update(range(c0, c0 + int(rng.integers(1, 14))))
        rows.append(np.array(sorted(cols)))
    rowptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    col = np.concatenate(rows).astype(np.int32)
    val = rng.standard_normal(col.size)
    return OracleCSR(m, n, rowptr, col, val)


@pytest.mark.parametrize("m", [1, 8, 4099])
def test_tma_product_ragged_rows(m):
    # aligned pair-CSR forced on a matrix of ragged run-structured rows: the TMA product is bitwise
    # equal to the full-warp register kernel... which the default rule does not pick here (rows of
    # mixed lengths), so compare with the oracle's product and with the half-warp kernel instead
    M = _ragged_runs(m, 5000, seed=m)
    z = np.random.default_rng(m + 1).standard_normal(M.ncols)
    ref = M.matvec(z)
    absref = OracleCSR(M.nrows, M.ncols, M.rowptr, M.col, np.abs(M.val)).matvec(np.abs(z))
    y_tma, inf = _product(M, z, ["tma", "keep_csr"], tuning=17)
    y_reg, _ = _product(M, z, ["keep_csr"], tuning=17)
    assert inf["a_fmt"] == 2
    assert np.all(np.abs(y_tma - ref) <= 1e-14 * absref + 1e-300)
    assert np.all(np.abs(y_tma - y_reg) <= 1e-14 * absref + 1e-300)
    empty = np.diff(M.rowptr) == 0
    assert np.all(y_tma[empty] == 0.0)


@pytest.mark.parametrize("cfg", [3, 5])
def test_tma_bitwise_equals_full_warp_kernel(cfg):
    # config 3's and config 5-reduced's Siddon A run a full warp per row by default: the TMA-staged
    # product sums every row in the same order, so the products agree bit for bit; the solve (whose
    # transpose also runs TMA-staged, a full warp per row instead of half a warp) holds the oracle's bar
    kw = dict(N=128, n_angles=90, nb=183) if cfg == 3 else C5R
    p = make_problem(cfg, **kw)
    z = np.random.default_rng(7).standard_normal(p.n)
    y_tma, inf = _product(p.A, z, ["tma"])
    y_reg, inf_reg = _product(p.A, z, [])
    assert inf["a_fmt"] == 2 and inf_reg["a_fmt"] == 2
    assert np.array_equal(y_tma, y_reg)
    spec = p.solvers[0]
    K = 12
    r = solve_problem(p, spec, maxit=K, eta=0.0)
    _compare(_gpu_run(p, spec, maxit=K, eta=0.0, knobs=["tma"]), r, n_res=K)


def test_tma_config4_reduced_against_oracle():
    # config 4's A (long rays: half a warp per row by default) on the TMA path: a full warp per row,
    # another summation order; the solve holds the oracle's bar
    p = make_problem(4, N=96, n_angles=61, nb=137)
    spec = p.solvers[0]
    K = 12
    r = solve_problem(p, spec, maxit=K, eta=0.0)
    g = _gpu_run(p, spec, maxit=K, eta=0.0, knobs=["tma"])
    assert g["info"]["a_fmt"] == 2
    _compare(g, r, n_res=K)


@pytest.mark.parametrize("cfg,method", [(3, "sflsqr"), (3, "sflsmr"), (4, "sflsqr"), (1, "sflsmr")])
def test_wnorm_fused_into_transpose_product(cfg, method):
    # one rank: the w normalisation (k_finish_w) runs inside the transpose product (SpmvEpi kind 5:
    # gathers of the unnormalised w', row sums scaled by 1/||w'||, W[:, k] and H_{k+1,k} stored by
    # the product's threads); SFLSQR_KNOB_WNORM_SEP keeps the separate kernel.  Both solves hold the
    # oracle's bar, and the bases agree to rounding
    import dataclasses
    kw = {3: dict(N=128, n_angles=90, nb=183), 4: dict(N=96, n_angles=61, nb=137), 1: {}}[cfg]
    p = make_problem(cfg, **kw)
    spec = dataclasses.replace(p.solvers[0], method=method)
    K = 12
    r = solve_problem(p, spec, maxit=K, eta=0.0)
    runs = {}
    for kn in ([], ["wnorm_sep"]):
        g = _gpu_run(p, spec, maxit=K, eta=0.0, knobs=kn)
        _compare(g, r, n_res=K)
        runs[bool(kn)] = g
    a, b = runs[False], runs[True]
    assert np.max(np.abs(a["x"] - b["x"])) <= 1e-8 * np.max(np.abs(b["x"]))
