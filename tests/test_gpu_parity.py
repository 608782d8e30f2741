"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bar (BASELINE.json north_star): sketch tables bit-exact; per-iteration true and
sketched residual norms within 1e-9 relative for iterations 1..30; final x
within 1e-6 relative (2-norm); the same stopping iteration and status.
"""
import numpy as np
import pytest

from gen import make_problem
from gen.problems import SolverSpec
from oracle.operators import BlurOperator, OracleCSR, operator_from_problem
from oracle.sflsqr import solve, solve_problem
from oracle.sketch import sparse_sign_table

from horizons import C5R, EDGE_CASES, MAXSIZE_CASES, dense_prob, horizon

pytestmark = pytest.mark.gpu

RES_TOL = 1e-9
X_TOL = 1e-6
N_RES = 30


@pytest.fixture(scope="session", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_22281_b200._build import build_library
    build_library()


def _gpu_run(prob, spec, maxit=None, eta=None, use_graph=True, **kw):
    from paper_2605_22281_b200 import solver_for_problem
    s = solver_for_problem(prob, spec, maxit=maxit, eta=eta, use_graph=use_graph, **kw)
    s.set_rhs(prob.b)
    done, status = s.iterate(maxit or spec.maxit)
    tr, sk = s.get_residual_norms()
    x = s.get_x()
    info = s.get_info()
    s.close()
    return dict(done=done, status=status, true_res=tr, sketch_res=sk, x=x, info=info)


def sketch_floor(r, k):
    """Rounding floor of the step-k sketched residual rho_k = ||rhs - M_k y_k|| (reading R24).

    rho_k is the residual norm of a least-squares problem, and r_k = rhs - M_k y_k is orthogonal to
    range(M_k): to first order a backward perturbation dM of M_k moves it by |r_k^T dM y_k| / rho_k
    <= ||dM|| ||y_k||.  Both sides solve backward stably, so the floor is 100 u ||M_k||_2 ||y_k||,
    with M_k the step-k matrix (sFLSQR: S A Z_k; sFLSMR: [S_TW, S z]_{k+1} H_{k+1,k}) and y_k the
    oracle's solution at step k, not the final one."""
    if r.method != "sflsmr":                                         # sFLSQR: M_k = S A Z_k
        M = r.sketch_cols[:, :k]
    elif r.sketch_cols.shape[1] >= k + 1:                            # sFLSMR: [S_TW, S z]_{k+1} H_{k+1,k}
        M = r.sketch_cols[:, :k + 1] @ r.H[:k + 1, :k]
    else:                                                            # stopped at k: S z_{k+1} not kept
        M = r.sketch_cols[:, :k] @ r.H[:k, :k]
    return 100 * 2.0 ** -53 * np.linalg.norm(M, 2) * np.linalg.norm(r.ys[k - 1])


def _compare(g, r, n_res=N_RES, res_tol=RES_TOL, x_tol=X_TOL, eff_bound=None, eff_k=N_RES):
    """Strict parity: true residuals within res_tol relative, sketched residuals within res_tol
    relative plus the per-k floor of sketch_floor (its effective relative tolerance is printed and,
    with eff_bound, asserted for k <= eff_k: north_star's window), x within x_tol, the same status
    and stop index."""
    kk = len(r.true_res)
    assert g["info"]["k_done"] == kk, (g["info"], kk)
    assert g["status"] == r.status and g["info"]["k_x"] == r.k
    n = min(n_res, kk)
    rt = np.abs(g["true_res"][:n] - np.array(r.true_res[:n])) / np.array(r.true_res[:n])
    ref_sk = np.array(r.sketch_res[:n])
    tol_k = res_tol * ref_sk + np.array([sketch_floor(r, k) for k in range(1, n + 1)])
    eff = tol_k / ref_sk                                              # effective relative tolerance per k
    rs = np.abs(g["sketch_res"][:n] - ref_sk) / tol_k                 # must be < 1
    ex = np.linalg.norm(g["x"] - r.x) / max(np.linalg.norm(r.x), 1e-300)
    print(f"parity k<={n}: true-res {rt.max():.2e}, sketch-res {np.max(np.abs(g['sketch_res'][:n] - ref_sk) / ref_sk):.2e} "
          f"(effective tol max {eff.max():.2e} at k={int(eff.argmax()) + 1}), x {ex:.2e}")
    assert rt.max() < res_tol, ("true residual", rt.max(), int(rt.argmax()) + 1)
    assert rs.max() < 1.0, ("sketched residual", rs.max(), int(rs.argmax()) + 1)
    if eff_bound is not None:
        e30 = eff[:eff_k]
        assert e30.max() <= eff_bound, ("effective sketched-residual tolerance", e30.max(), int(e30.argmax()) + 1)
    assert ex < x_tol, ("x", ex)
    return rt.max(), rs.max(), ex


# ------------------------------------------------------------------ P1: sketch table bit-exact
@pytest.mark.parametrize("seed,d,s,dim", [(0x5F1A5E, 80, 4, 256), (0x5F1A5F, 200, 8, 65536), (0x5F1A60, 300, 8, 262144),
                                          (0x5F1A61, 400, 8, 1043280), (7, 13, 13, 5000), (1 << 40, 31, 1, 9999),
                                          (12345, 64, 32, 3000), (99, 50, 5, 7777)])
def test_sketch_table_bit_exact(seed, d, s, dim):
    from paper_2605_22281_b200 import SFLSQR
    sol = SFLSQR(maxit=1)
    sol.set_sketch(seed, d, s)
    if dim > 300000:
        for c0 in (0, dim // 2 - 1000, dim - 50000):
            nc = min(50000, dim - c0)
            rg, sg = sol.debug_sketch_table(c0, nc, s)
            ro, so = sparse_sign_table(seed, d, s, c0, nc)
            assert np.array_equal(rg, ro) and np.array_equal(sg, so)
    else:
        rg, sg = sol.debug_sketch_table(0, dim, s)
        ro, so = sparse_sign_table(seed, d, s, 0, dim)
        assert np.array_equal(rg, ro) and np.array_equal(sg, so)
    sol.close()


# ------------------------------------------------------------------ operators
def test_spmv_matches_oracle_ct_ragged():
    from paper_2605_22281_b200 import SFLSQR
    p = make_problem(4, N=96, n_angles=61, nb=137)   # ragged rows, empty corner rays, unmatched B
    s = SFLSQR(maxit=4)
    s.set_operator(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, p.A.val, t=(p.T.rowptr, p.T.col, p.T.val))
    A = OracleCSR(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, p.A.val)
    B = OracleCSR(p.T.nrows, p.T.ncols, p.T.rowptr, p.T.col, p.T.val)
    rng = np.random.default_rng(0)
    x, w = rng.standard_normal(p.n), rng.standard_normal(p.m)
    for got, ref in ((s.debug_apply(0, x), A.matvec(x)), (s.debug_apply(1, w), B.matvec(w))):
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    s.close()


def test_built_transpose_matches_oracle():
    from paper_2605_22281_b200 import SFLSQR
    p = make_problem(3, N=80, n_angles=50, nb=115)
    s = SFLSQR(maxit=4)
    s.set_operator(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, p.A.val)
    At = OracleCSR(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, p.A.val).transpose()
    w = np.random.default_rng(1).standard_normal(p.m)
    got, ref = s.debug_apply(1, w), At.matvec(w)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    s.close()


def test_built_transpose_device_arrays_and_determinism():
    # T_BUILD from device arrays (torch CUDA tensors, copied or borrowed) forms A^T on the device like
    # the host-array path: the same bits, and the oracle's transpose to rounding
    import torch
    from paper_2605_22281_b200 import SFLSQR
    p = make_problem(3, N=80, n_angles=50, nb=115)
    w = np.random.default_rng(11).standard_normal(p.m)
    outs = []
    for kind in ("host", "device", "borrow"):
        s = SFLSQR(maxit=4)
        if kind == "host":
            s.set_operator(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, p.A.val)
        else:
            arrs = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (p.A.rowptr, p.A.col, p.A.val)]
            s.set_operator(p.A.nrows, p.A.ncols, *arrs, borrow=(kind == "borrow"))
        outs.append(s.debug_apply(1, w))
        s.close()
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    ref = OracleCSR(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, p.A.val).transpose().matvec(w)
    assert np.max(np.abs(outs[0] - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_built_transpose_long_columns_and_duplicates():
    # columns with more than 4096 entries (the shared-memory row sort's limit) take the segmented-sort
    # fallback; duplicate (row, column) entries are kept as separate entries (ordered by value bits)
    from paper_2605_22281_b200 import SFLSQR
    rng = np.random.default_rng(12)
    m, n = 5000, 24
    D = rng.standard_normal((m, n))
    D[rng.random((m, n)) < 0.2] = 0.0
    rows, cols, vals = [], [], []
    for i in range(m):
        c = np.flatnonzero(D[i])
        v = D[i, c]
        if i % 97 == 0 and c.size:                       # a duplicate entry of this row's first column
            c, v = np.append(c, c[0]), np.append(v, 0.5)
        rows.append(c), vals.append(v)
    rowptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    col, val = np.concatenate(rows).astype(np.int32), np.concatenate(vals)
    A = OracleCSR(m, n, rowptr, col, val)
    w = rng.standard_normal(m)
    got = []
    for _ in range(2):
        s = SFLSQR(maxit=4)
        s.set_operator(m, n, rowptr, col, val)
        got.append(s.debug_apply(1, w))
        s.close()
    assert np.array_equal(got[0], got[1])
    absref = OracleCSR(m, n, rowptr, col, np.abs(val)).transpose().matvec(np.abs(w))
    assert np.all(np.abs(got[0] - A.transpose().matvec(w)) <= 1e-13 * absref)


def test_blur_matches_oracle():
    from paper_2605_22281_b200 import SFLSQR
    for H, W in ((256, 256), (37, 53)):
        s = SFLSQR(maxit=4)
        s.set_operator_blur(H, W, 2.5, 7)
        op = BlurOperator(H, W, 2.5, 7)
        x = np.random.default_rng(2).standard_normal(H * W)
        got, ref = s.debug_apply(0, x), op.matvec(x)
        assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
        s.close()


# ------------------------------------------------------------------ end to end, config 1 (dense, sigma_min 1e-6)
@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_config1_full(method):
    p = make_problem(1)
    spec = [s for s in p.solvers if s.method == method][0]
    r = solve_problem(p, spec)
    g = _gpu_run(p, spec)
    _compare(g, r, eff_bound=2e-9)


@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_config1_discrepancy_stop(method):
    # a safety factor the run reaches mid-way, so the discrepancy rule fires (eq. discrP)
    p = make_problem(1)
    spec = [s for s in p.solvers if s.method == method][0]
    full = solve_problem(p, spec, eta=0.0)
    eta = float(full.true_res[14] / p.delta_e) * (1 + 1e-7)
    r = solve_problem(p, spec, eta=eta)
    assert r.status == 3
    g = _gpu_run(p, spec, eta=eta)
    _compare(g, r)


@pytest.mark.parametrize("use_graph", [True, False])
def test_graph_and_eager_agree_bitwise(use_graph):
    p = make_problem(1)
    spec = p.solvers[0]
    g1 = _gpu_run(p, spec, maxit=15, use_graph=use_graph)
    g2 = _gpu_run(p, spec, maxit=15, use_graph=True)
    assert g1["info"]["graph"] == int(use_graph) and g2["info"]["graph"] == 1
    assert np.array_equal(g1["x"], g2["x"])              # deterministic reductions
    assert np.array_equal(g1["true_res"], g2["true_res"])


# ------------------------------------------------------------------ config 2 (blur, IRN)
def test_config2_blur():
    # all 100 iterations of BASELINE's config 2 are inside the oracle's stable horizon
    p = make_problem(2)
    spec = p.solvers[0]
    kstar, r = horizon("c2/sflsqr", p)
    g = _gpu_run(p, spec, maxit=kstar)
    if kstar < spec.maxit:
        r = solve_problem(p, spec, maxit=kstar)
    _compare(g, r, n_res=kstar)


# ------------------------------------------------------------------ config 3 reduced (Siddon, NONNEG), full 150 its
@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_config3_reduced(method):
    p = make_problem(3, N=128, n_angles=90, nb=183)
    spec = [s for s in p.solvers if s.method == method][0]
    r = solve_problem(p, spec)
    g = _gpu_run(p, spec)
    _compare(g, r, eff_bound=2e-9)


# ------------------------------------------------------------------ config 4 reduced (unmatched B, identity tau)
def test_config4_reduced_within_oracle_stable_horizon():
    # The unmatched-B, identity-tau run loses forward stability in the oracle itself after ~15
    # iterations (S A Z_k becomes ill-conditioned); strict parity is required up to that horizon,
    # later iterations are checked by state injection below.
    p = make_problem(4, N=192, n_angles=135, nb=273)
    spec = p.solvers[0]
    kstar, _ = horizon("c4r192/sflsqr", p)
    r = solve_problem(p, spec, maxit=kstar, eta=0.0)
    g = _gpu_run(p, spec, maxit=kstar)
    _compare(g, r, n_res=kstar)


# ------------------------------------------------------------------ state injection (one oracle step from GPU state)
def _inject(p, spec, ks, maxit, tol_vec=1e-12, tol_res=1e-9):
    from oracle.sflsqr import step_from_state
    from oracle.sketch import SparseSignSketch
    from paper_2605_22281_b200 import solver_for_problem
    op = operator_from_problem(p)
    dim = p.m if spec.method == "sflsqr" else p.n
    sk = SparseSignSketch(p.sketch_seed, spec.d, spec.s_nz, dim)
    ell = min(spec.window, maxit)
    s = solver_for_problem(p, spec, maxit=maxit, eta=0.0)
    s.set_rhs(p.b)
    done = 0
    rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)  # noqa: E731
    report = []
    for k in ks:
        s.iterate(k - 1 - done)
        done = k - 1
        B = s.debug_basis()
        V = s.debug_state(ell, spec.d, spec.method)
        use_ring = spec.orth_mode == "P" and spec.precond != "identity"
        if use_ring:
            Pw = {j: V["p_ring"][(j - 1) % ell] for j in range(max(1, k - ell), k)}
        else:
            Pw = {j: B["Z"][:, j - 1] for j in range(max(1, k - ell), k)}
        out = step_from_state(op, p.b, spec.method, k, ell, sk, B["Z"], Pw, B["W"], V["z"], V["x"],
                              B["H"], V["sketch_cols"], V["rhs"], precond=spec.precond, p_exp=spec.p,
                              eps_rel=spec.eps_rel, orth_mode=spec.orth_mode)
        s.iterate(1)
        done = k
        B2 = s.debug_basis()
        V2 = s.debug_state(ell, spec.d, spec.method)
        tr, sk_res = s.get_residual_norms()
        newcol = V2["sketch_cols"][:, -1]
        ocol = out["Mcol"] if spec.method == "sflsqr" else out["Sz"]
        # The projected LS is backward stable on both sides; its outputs can differ by
        # ~u * cond(M) (normwise), which near rank deficiency exceeds 1e-9.
        kappa = float(np.linalg.cond(out["M"]))
        ls_tol = max(tol_res, 100 * 2.0 ** -53 * kappa)
        nrhs, nb = np.linalg.norm(V["rhs"]), np.linalg.norm(p.b)
        errs = dict(T=rel(B2["T"][:k, k - 1], out["Tcol"]), z=rel(B2["Z"][:, k - 1], out["z"]),
                    H=rel(B2["H"][:k + 1, k - 1], out["Hcol"]), w=rel(B2["W"][:, k], out["w_next"]),
                    sk=rel(newcol, ocol),
                    sres=abs(sk_res[k - 1] - out["sres"]) / max(out["sres"], ls_tol * nrhs / tol_res),
                    r=abs(tr[k - 1] - out["r"]) / max(out["r"], ls_tol * nb / tol_res),
                    My=np.linalg.norm(out["M"] @ (B2["y"] - out["y"])) / nrhs / (ls_tol / tol_res))
        report.append((k, kappa, errs))
        print(f"inject k={k} cond(M)={kappa:.2e} " + " ".join(f"{a}={b:.1e}" for a, b in errs.items()))
        for key in ("T", "z", "H", "w", "sk"):
            assert errs[key] < tol_vec, (k, key, errs)
        for key in ("sres", "r", "My"):
            assert errs[key] < tol_res, (k, key, kappa, errs)
    s.close()
    return report


def test_config4_reduced_state_injection():
    p = make_problem(4, N=192, n_angles=135, nb=273)
    _inject(p, p.solvers[0], ks=[2, 17, 60, 140, 200], maxit=200)


@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_config3_reduced_state_injection(method):
    p = make_problem(3, N=128, n_angles=90, nb=183)
    spec = [s for s in p.solvers if s.method == method][0]
    _inject(p, spec, ks=[1, 4, 90, 150], maxit=150)


def test_config1_state_injection_both_orth_modes():
    p = make_problem(1)
    for spec in p.solvers:
        _inject(p, spec, ks=[3, 20, 40], maxit=40)
        spec_z = SolverSpec(**{**spec.__dict__, "orth_mode": "Z"})
        _inject(p, spec_z, ks=[3, 40], maxit=40)


# ------------------------------------------------------------------ full BASELINE sizes (oracle to its horizon)
@pytest.fixture(scope="module")
def c3_full():
    return make_problem(3)


@pytest.fixture(scope="module")
def c4_full():
    return make_problem(4)


@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_config3_full_size_first_30_iterations(c3_full, method):
    # north_star's window: iterations 1..30 at 1e-9 on BASELINE's full config 3 (inside the horizon)
    p = c3_full
    spec = [s for s in p.solvers if s.method == method][0]
    kstar, r = horizon(f"c3full/{method}", p)
    g = _gpu_run(p, spec, maxit=kstar)
    _compare(g, r, n_res=kstar, eff_bound=2e-9)


def test_config4_full_size_to_horizon(c4_full):
    # full BASELINE config 4 (the bench workload) at the strict bar up to the oracle's own horizon
    p = c4_full
    spec = p.solvers[0]
    kstar, r = horizon("c4full/sflsqr", p)
    g = _gpu_run(p, spec, maxit=kstar)
    _compare(g, r, n_res=kstar)


def test_config4_full_size_state_injection(c4_full):
    # full BASELINE size, the launch configuration bench.py times: one oracle step from the GPU state
    _inject(c4_full, c4_full.solvers[0], ks=[101, 200], maxit=200)


def test_config3_full_size_state_injection_sflsmr(c3_full):
    _inject(c3_full, c3_full.solvers[1], ks=[150], maxit=150)


# ------------------------------------------------------------------ config 5 (BASELINE configs[4]) at reduced size
# Siddon CT with A^T built by the library, IRN-l1 tau, window 5, d = 600, s = 8, both methods, 300
# iterations: BASELINE's recipe on a 256^2 grid (180 angles, 363 bins) instead of 2048^2 (the full
# operators, 185 GB, need >= 2 GPUs).  Sharded runs: tests/test_gpu_sharded.py.
@pytest.fixture(scope="module")
def c5_reduced():
    return make_problem(5, **C5R)


@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_config5_reduced_to_horizon(c5_reduced, method):
    p = c5_reduced
    spec = [s for s in p.solvers if s.method == method][0]
    assert (spec.window, spec.d, spec.s_nz, spec.precond, spec.maxit) == (5, 600, 8, "irn", 300)
    kstar, r = horizon(f"c5r/{method}", p)
    g = _gpu_run(p, spec, maxit=kstar)
    _compare(g, r, n_res=kstar, eff_bound=2e-9)


@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_config5_reduced_full_run_state_injection(c5_reduced, method):
    # all 300 iterations on the GPU; one oracle step from the GPU state at early, middle and late k
    p = c5_reduced
    spec = [s for s in p.solvers if s.method == method][0]
    _inject(p, spec, ks=[1, 6, 160, 300], maxit=300)


@pytest.fixture(scope="module")
def c5_full_row_block():
    """BASELINE configs[4] at full size (2048^2, 1440 angles x 2897 bins, 7.7e9 Siddon nonzeros) does
    not fit one GPU.  Rank 0's block of an 8-way nnz-balanced row split -- the rows one of 8 ranks
    holds, ~9.6e8 nonzeros -- from the sharded generator (gen.problems.make_ct_shard), posed as a
    least-squares problem of its own: min ||A_0 x - b_0|| with T = A_0^T built by the library."""
    from gen.problems import Problem, ct_row_nnz, make_ct_shard
    from paper_2605_22281_b200.shard import balanced_row_blocks
    a_cnt, _ = ct_row_nnz(5)
    blocks = balanced_row_blocks(np.concatenate([[0], np.cumsum(a_cnt)]), 8)
    sp = make_ct_shard(5, blocks[0], None, lambda v: v)   # ||A x_true|| over this block only
    A = sp.A_loc
    assert A.ncols == 2048 * 2048 and A.nnz > 9e8 and A.rowptr.dtype == np.int64
    return Problem(name="c5_row_block0_of8", config_index=5, m=A.nrows, n=A.ncols, A=A, T=None, t_mode="build",
                   blur=None, x_true=np.zeros(A.ncols), b=sp.b_loc, e=np.zeros(A.nrows), delta=0.01,
                   delta_e=sp.delta_e, sketch_seed=sp.sketch_seed, solvers=sp.solvers)


@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_config5_full_size_row_block_first_iterations(c5_full_row_block, method):
    p = c5_full_row_block
    spec = [s for s in p.solvers if s.method == method][0]
    K = 4
    r = solve_problem(p, spec, maxit=K, eta=0.0)
    g = _gpu_run(p, spec, maxit=K)
    _compare(g, r, n_res=K)


# ------------------------------------------------------------------ edge cases
_dense_prob = dense_prob


# CountSketch + window 1 + ragged sizes; window >= maxit (full orthogonalisation); literal Alg. 1
# orthogonalisation (two cases); underdetermined with d = maxit + 1; d = maxit
@pytest.mark.parametrize("case", range(len(EDGE_CASES)))
def test_edge_configurations(case):
    # strict parity over the iterations where the oracle itself is forward-stable
    m, n, method, window, precond, orth, s_nz, d = EDGE_CASES[case]
    p = _dense_prob(m, n, seed=m + n)
    spec = SolverSpec(method=method, maxit=20, window=window, d=d, s_nz=s_nz, precond=precond, orth_mode=orth)
    kstar, _ = horizon(f"edge/{case}", p)
    r = solve_problem(p, spec, maxit=kstar)
    g = _gpu_run(p, spec, maxit=kstar)
    _compare(g, r, n_res=kstar)


def test_breakdown_matches_oracle():
    from gen.problems import CSR, Problem
    A = np.diag([1.0, 2.0, 3.0, 4.0])
    b = np.array([1.0, 1.0, 0.0, 0.0])
    p = Problem(name="bd", config_index=0, m=4, n=4, A=CSR.from_dense(A), T=None, t_mode="build", blur=None,
                x_true=np.zeros(4), b=b, e=np.zeros(4), delta=0, delta_e=0.0, sketch_seed=5)
    spec = SolverSpec(method="sflsqr", maxit=4, window=4, d=4, s_nz=1, precond="identity")
    r = solve_problem(p, spec)
    g = _gpu_run(p, spec)
    assert r.status == 4 and g["status"] == 4 and g["info"]["k_x"] == r.k
    np.testing.assert_allclose(g["x"], r.x, rtol=1e-10, atol=1e-12)


def test_k1_and_restart():
    from paper_2605_22281_b200 import solver_for_problem
    p = make_problem(1)
    spec = p.solvers[0]
    s = solver_for_problem(p, spec, maxit=5, eta=0.0)
    s.set_rhs(p.b)
    s.iterate(1)
    r1 = solve_problem(p, spec, maxit=1, eta=0.0)
    assert np.linalg.norm(s.get_x() - r1.x) <= 1e-12 * np.linalg.norm(r1.x)
    done, st = s.iterate(100)
    assert done and st == 1 and s.get_info()["k_done"] == 5
    s.set_rhs(p.b)                       # restart reproduces the first solve
    s.iterate(5)
    r5 = solve_problem(p, spec, maxit=5, eta=0.0)
    assert np.linalg.norm(s.get_x() - r5.x) <= 1e-10 * np.linalg.norm(r5.x)
    s.close()


def test_error_codes():
    from paper_2605_22281_b200 import SFLSQR, SflsqrError
    from paper_2605_22281_b200 import sflsqr as B
    s = SFLSQR(maxit=10)
    with pytest.raises(SflsqrError) as e:
        s.set_rhs(np.ones(4))                        # no operator yet
    assert e.value.code == B.E_STATE
    rp = np.array([0, 1, 2], dtype=np.int64)
    with pytest.raises(SflsqrError) as e:
        s.set_operator(2, 2, rp, np.array([0, 5], dtype=np.int32), np.ones(2))
    assert e.value.code == B.E_DIM
    with pytest.raises(SflsqrError) as e:
        s.set_operator(2, 2, rp, np.array([0, 1], dtype=np.int32), np.array([1.0, np.nan]))
    assert e.value.code == B.E_NONFINITE
    s.set_operator(2, 2, rp, np.array([0, 1], dtype=np.int32), np.ones(2))
    with pytest.raises(SflsqrError) as e:
        s.set_sketch(1, 5, 1)                        # d < maxit
    assert e.value.code == B.E_INVALID
    s.set_sketch(1, 10, 1)
    with pytest.raises(SflsqrError) as e:
        s.set_rhs(np.zeros(2))
    assert e.value.code == B.E_ZERO_RHS
    with pytest.raises(SflsqrError) as e:
        s.set_rhs(np.ones(3))
    assert e.value.code == B.E_DIM
    with pytest.raises(SflsqrError) as e:
        s.set_precond("irn", p=3.0)
    assert e.value.code == B.E_INVALID
    s.close()


# ------------------------------------------------------------------ pair-CSR (SpMV mode 16)
def _runs_csr(seed, m, n):
    """Rows made of runs of consecutive columns (lengths 1..9, odd and even, some rows empty,
    some longer than 32 entries so runs straddle the kernel's 32-entry steps)."""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(m):
        cols, c = [], int(rng.integers(0, 5))
        target = 0 if i % 17 == 0 else int(rng.integers(1, 120))
        while len(cols) < target and c < n - 10:
            L = int(rng.integers(1, 10))
            cols.extend(range(c, min(c + L, n)))
            c += L + int(rng.integers(1, 4))
        rows.append(np.array(cols[:target], dtype=np.int64))
    rowptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    col = np.concatenate(rows).astype(np.int32) if rowptr[-1] else np.zeros(0, np.int32)
    return rowptr, col, rng.standard_normal(col.size)


@pytest.mark.parametrize("mode", [16, 17])   # 17: pairs only at even columns, 16-byte gathers
@pytest.mark.parametrize("seed", [0, 1])
def test_pair_csr_matches_oracle_matvec(seed, mode):
    from paper_2605_22281_b200 import SFLSQR
    m, n = 700, 2000
    rp, col, val = _runs_csr(seed, m, n)
    A = OracleCSR(m, n, rp, col, val)
    At = A.transpose()
    s = SFLSQR(maxit=4, knobs=["keep_csr"])
    s.set_operator(m, n, rp, col, val)                       # T = A^T built by the library
    rng = np.random.default_rng(10 + seed)
    x, w = rng.standard_normal(n), rng.standard_normal(m)
    s.debug_set_tuning(mode)
    ya, yt = s.debug_apply(0, x), s.debug_apply(1, w)
    ra, rt = A.matvec(x), At.matvec(w)
    absa = OracleCSR(m, n, rp, col, np.abs(val))
    # each entry within a few ulp of the row's absolute sum (summation order differs)
    assert np.all(np.abs(ya - ra) <= 1e-14 * absa.matvec(np.abs(x)) + 1e-300)
    assert np.all(np.abs(yt - rt) <= 1e-14 * absa.transpose().matvec(np.abs(w)) + 1e-300)
    s.close()


@pytest.mark.parametrize("mode", [16, 17])
def test_pair_csr_solver_parity_unmatched_ct(mode):
    # sFLSQR on a reduced config-4 problem (pixel-driven B: all pairs; Siddon A: mixed) with
    # SpMV mode 16 / 17 against the oracle, same bar as the mode-14 runs
    from paper_2605_22281_b200 import solver_for_problem
    p = make_problem(4, N=96, n_angles=61, nb=137)
    spec = p.solvers[0]
    r = solve_problem(p, spec, maxit=12, eta=0.0)
    s = solver_for_problem(p, spec, maxit=12, eta=0.0, knobs=["keep_csr"])
    s.debug_set_tuning(mode)
    s.set_rhs(p.b)
    s.iterate(12)
    tr, sk = s.get_residual_norms()
    x = s.get_x()
    s.close()
    assert np.max(np.abs(tr - np.array(r.true_res)) / np.array(r.true_res)) < 1e-9
    assert np.max(np.abs(sk - np.array(r.sketch_res)) / np.array(r.sketch_res)) < 1e-9
    assert np.linalg.norm(x - r.x) / np.linalg.norm(r.x) < 1e-6


def test_default_spmv_format_rule():
    # >= 75 % adjacent pairs -> pair-CSR (the pixel-driven B), else >= 20 % even-column
    # pairs -> aligned pair-CSR (Siddon), else CSR; the same for the GKB methods (fused epilogues)
    from paper_2605_22281_b200 import SflsqrError, solver_for_problem
    from paper_2605_22281_b200 import sflsqr as B
    p = make_problem(4, N=96, n_angles=61, nb=137)
    spec = p.solvers[0]
    s = solver_for_problem(p, spec, maxit=3, eta=0.0)
    inf = s.get_info()
    s.close()
    assert inf["t_fmt"] == 4 and inf["t_pairs"] >= 0.375 * p.T.nnz    # B: interpolation pairs (1 - f, f), sliced ELL
    assert inf["a_fmt"] == 2 and inf["a_pairs"] >= 0.2 * p.A.nnz
    s = solver_for_problem(p, spec, maxit=3, eta=0.0, method="lsqr")
    inf = s.get_info()
    s.close()
    assert inf["a_fmt"] == 2 and inf["t_fmt"] == 4
    assert inf["csr_kept"] == 0                            # both copies serve: the uploaded CSR is released
    s = solver_for_problem(p, spec, maxit=3, eta=0.0)
    with pytest.raises(SflsqrError) as e:                  # forcing a format needs the CSR
        s.debug_set_tuning(14)
    assert e.value.code == B.E_STATE
    s.close()
    s = solver_for_problem(p, spec, maxit=3, eta=0.0, knobs=["keep_csr"])
    assert s.get_info()["csr_kept"] == 3
    s.debug_set_tuning(14)                                 # forced plain CSR
    inf = s.get_info()
    s.close()
    assert inf["a_fmt"] == 0 and inf["t_fmt"] == 0 and inf["a_pairs"] == 0 and inf["t_pairs"] == 0


def test_interpolation_pairs_bitwise_equal_to_pair_csr():
    # config 4's pixel-driven B: every pair is (1 - f, f) bitwise, so only f is stored (12 instead
    # of 20 bytes per pair); the reconstructed values and the summation order are those of the
    # pair-CSR kernel, so the products agree bit for bit
    from paper_2605_22281_b200 import SFLSQR
    p = make_problem(4, N=96, n_angles=61, nb=137)
    rng = np.random.default_rng(5)
    w, x = rng.standard_normal(p.m), rng.standard_normal(p.n)
    out = {}
    for interp, sell in (("0", "0"), ("1", "0"), ("1", "1")):
        knobs = (["no_interp"] if interp == "0" else []) + (["no_sell"] if sell == "0" else [])
        s = SFLSQR(maxit=4, knobs=knobs)
        s.set_operator(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, p.A.val, t=(p.T.rowptr, p.T.col, p.T.val))
        out[interp + sell] = (s.get_info()["t_fmt"], s.debug_apply(1, w), s.debug_apply(0, x))
        s.close()
    assert out["00"][0] == 1 and out["10"][0] == 3 and out["11"][0] == 4
    assert np.array_equal(out["00"][1], out["10"][1]) and np.array_equal(out["00"][2], out["10"][2])
    B = OracleCSR(p.T.nrows, p.T.ncols, p.T.rowptr, p.T.col, p.T.val)
    ref = B.matvec(w)
    absref = OracleCSR(p.T.nrows, p.T.ncols, p.T.rowptr, p.T.col, np.abs(p.T.val)).matvec(np.abs(w))
    for key in ("10", "11"):   # the sliced-ELL copy sums each row in its own (k) order
        assert np.all(np.abs(out[key][1] - ref) <= 1e-14 * absref + 1e-300)
    # an operator whose pairs are not interpolation weights keeps the full pair values
    m, n = 700, 2000
    rp, col, val = _runs_csr(3, m, n)
    s = SFLSQR(maxit=4)
    s.set_operator(m, n, rp, col, val, t=(rp, col, val) if m == n else None)
    assert s.get_info()["a_fmt"] in (0, 1, 2)
    s.close()


def _interp_csr(seed, nrows, ncols, singles=True):
    """Rows of (1 - f, f) pairs at adjacent columns (the interpolation structure), ragged lengths
    (64..200 pairs, some rows far shorter than their slice's longest), optional singleton tails."""
    rng = np.random.default_rng(seed)
    rows_c, rows_v = [], []
    for i in range(nrows):
        npair = int(rng.integers(140, 161)) if i % 97 else int(rng.integers(0, 5))
        base = np.sort(rng.choice(np.arange(0, ncols - 4, 3), size=npair, replace=False))
        f = rng.uniform(0.0, 1.0, npair)
        c = np.empty(2 * npair, np.int64)
        v = np.empty(2 * npair)
        c[0::2], c[1::2] = base, base + 1
        v[0::2], v[1::2] = 1.0 - f, f
        if singles and i % 5 == 0 and npair > 0:     # a singleton after the last pair
            c = np.concatenate([c, [base[-1] + 3]])      # not adjacent to base[-1] + 1
            v = np.concatenate([v, [rng.standard_normal()]])
        rows_c.append(c)
        rows_v.append(v)
    rowptr = np.concatenate([[0], np.cumsum([len(c) for c in rows_c])]).astype(np.int64)
    return rowptr, np.concatenate(rows_c).astype(np.int32), np.concatenate(rows_v)


@pytest.mark.parametrize("singles", [False, True])
def test_sliced_ell_interpolation_pairs_ragged(singles):
    # T given as a ragged interpolation operator (n rows not a multiple of the 32-row slices, rows of
    # very different lengths in one slice, optional singletons): the sliced-ELL kernel, the
    # interpolation pair-CSR kernel and plain CSR all match the oracle product
    from paper_2605_22281_b200 import SFLSQR
    m, n = 1500, 1000 + 13
    trp, tcol, tval = _interp_csr(7, n, m, singles)
    T = OracleCSR(n, m, trp, tcol, tval)
    A = T.transpose()                                    # any A with the right shape
    rng = np.random.default_rng(8)
    w = rng.standard_normal(m)
    ref = T.matvec(w)
    absref = OracleCSR(n, m, trp, tcol, np.abs(tval)).matvec(np.abs(w))
    fmts = set()
    for tune in (-1, 14):
        s = SFLSQR(maxit=4, knobs=["keep_csr"] if tune == 14 else [])
        s.set_operator(m, n, A.rowptr, A.col, A.val, t=(trp, tcol, tval))
        if tune == 14:
            s.debug_set_tuning(14)
        fmts.add(s.get_info()["t_fmt"])
        got = s.debug_apply(1, w)
        s.close()
        assert np.all(np.abs(got - ref) <= 1e-14 * absref + 1e-300), tune
    # the sliced-ELL copy is kept when its padding is <= 10 % (here about 8 %): format 4
    npairs = np.array([(np.diff(trp)[r] // 2) for r in range(n)])
    slices = [npairs[i:i + 32] for i in range(0, n, 32)]
    pad = sum(len(sl) * sl.max() for sl in slices) / npairs.sum() - 1.0
    assert pad <= 0.10 and fmts == {4, 0}, (pad, fmts)


def test_pair_formats_odd_dimensions():
    # odd n (97^2 pixels, row-major order) and odd m: the columns of Z / W are 16-byte aligned only
    # for every other k, so the aligned pair kernel alternates with its two-load fallback; the
    # sliced-ELL backprojector does not depend on alignment.  Same bar as the other solver runs.
    from paper_2605_22281_b200 import solver_for_problem
    p = make_problem(4, N=97, n_angles=61, nb=139)
    assert p.n % 2 == 1 and p.m % 2 == 1
    spec = p.solvers[0]
    r = solve_problem(p, spec, maxit=10, eta=0.0)
    s = solver_for_problem(p, spec, maxit=10, eta=0.0)
    inf = s.get_info()
    s.set_rhs(p.b)
    s.iterate(10)
    tr, sk = s.get_residual_norms()
    x = s.get_x()
    s.close()
    assert inf["a_fmt"] == 2 and inf["t_fmt"] == 4, (inf["a_fmt"], inf["t_fmt"])
    assert np.max(np.abs(tr - np.array(r.true_res)) / np.array(r.true_res)) < 1e-9
    assert np.max(np.abs(sk - np.array(r.sketch_res)) / np.array(r.sketch_res)) < 1e-9
    assert np.linalg.norm(x - r.x) / np.linalg.norm(r.x) < 1e-6


@pytest.mark.parametrize("knob", ["no_pdl", "sketch_main", "full_spmv_grid", "res_main", "res_side", "keep_csr",
                                  "debug_poison"])
def test_scheduling_knobs_bitwise_neutral(knob):
    # launch scheduling (programmatic dependent launch, the sketch and the W-path residual on the side
    # or main stream, the SpMV grid size), keeping the uploaded CSR and NaN-poisoned solve buffers
    # (a read before write would show) change no arithmetic: the same solve bit for bit
    from paper_2605_22281_b200 import solver_for_problem
    p = make_problem(4, N=96, n_angles=61, nb=137)
    spec = p.solvers[0]
    out = []
    for kn in ([knob], []):
        s = solver_for_problem(p, spec, maxit=12, eta=0.0, knobs=kn)
        s.set_rhs(p.b)
        s.iterate(12)
        tr, sk = s.get_residual_norms()
        out.append((s.get_x(), tr, sk))
        s.close()
    # (full_spmv_grid changes which CTA takes which rows, not any row's summation order)
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("cfg", [3, 5])
def test_full_warp_rows_match_half_warp(cfg):
    # short ray-like rows (config 3's and config 5-reduced's Siddon A) run a full warp
    # per row; another summation order than the half-warp kernel (SFLSQR_KNOB_HALF_WARP_ROWS): the
    # products agree to rounding and both solves hold the oracle's bar
    from paper_2605_22281_b200 import SFLSQR
    kw = dict(N=128, n_angles=90, nb=183) if cfg == 3 else C5R
    p = make_problem(cfg, **kw)
    spec = p.solvers[0]
    z = np.random.default_rng(31).standard_normal(p.n)
    prods = []
    for kn in ([], ["half_warp_rows"]):
        s = SFLSQR(maxit=4, knobs=kn)
        s.set_operator(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, p.A.val)
        prods.append(s.debug_apply(0, z))
        s.close()
    absref = OracleCSR(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.col, np.abs(p.A.val)).matvec(np.abs(z))
    assert np.all(np.abs(prods[0] - prods[1]) <= 1e-14 * absref + 1e-300)
    K = 12
    r = solve_problem(p, spec, maxit=K, eta=0.0)
    for kn in ([], ["half_warp_rows"]):
        _compare(_gpu_run(p, spec, maxit=K, eta=0.0, knobs=kn), r, n_res=K)


def test_wide_column_range_rows_match_oracle():
    # short rows whose columns span 200 000 columns (random, sorted): plain CSR, built transpose
    from paper_2605_22281_b200 import SFLSQR
    rng = np.random.default_rng(4)
    m, n = 300, 200000
    rows = []
    for i in range(m):
        k = 1 + (i * 7) % 40
        rows.append(np.sort(rng.choice(n, size=k, replace=False)))
    rowptr = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    col = np.concatenate(rows).astype(np.int32)
    val = rng.standard_normal(col.size)
    s = SFLSQR(maxit=4)
    s.set_operator(m, n, rowptr, col, val)
    A = OracleCSR(m, n, rowptr, col, val)
    x = rng.standard_normal(n)
    got = s.debug_apply(0, x)
    assert np.max(np.abs(got - A.matvec(x))) <= 1e-13 * np.max(np.abs(A.matvec(x)))
    w = rng.standard_normal(m)
    got_t = s.debug_apply(1, w)
    ref_t = A.transpose().matvec(w)
    assert np.max(np.abs(got_t - ref_t)) <= 1e-13 * np.max(np.abs(ref_t))
    s.close()


# ------------------------------------------------------------------ maximum sizes and tiny problems
# d > 1024 (the RPT = 4 projected-LS kernel); d = 2048, the largest sketch the one-CTA LS supports;
# 600 columns (blocked back substitution over 19 blocks, long W-path residual)
@pytest.mark.parametrize("case", range(len(MAXSIZE_CASES)))
def test_maximum_sketch_and_iteration_counts(case):
    method, d, maxit, window = MAXSIZE_CASES[case]
    p = _dense_prob(1600, 900, seed=d + maxit, cond=1e2)
    spec = SolverSpec(method=method, maxit=maxit, window=window, d=d, s_nz=8, precond="irn")
    kstar, _ = horizon(f"maxsize/{case}", p)
    r = solve_problem(p, spec, maxit=kstar)
    g = _gpu_run(p, spec, maxit=kstar)
    _compare(g, r, n_res=kstar)
    if maxit > 100:
        # the full 600-iteration run: same status and stop index, residual history within the oracle's own
        # forward-stability band beyond the horizon is not asserted (reading R17); x by state injection
        # is covered elsewhere — here the run must complete with finite, non-increasing sketched residuals
        g = _gpu_run(p, spec, maxit=maxit)
        assert g["info"]["k_done"] == maxit and np.all(np.isfinite(g["sketch_res"]))
        assert np.all(np.diff(g["sketch_res"]) <= 1e-12 * g["sketch_res"][0])


@pytest.mark.parametrize("m,n", [(3, 2), (2, 3), (1, 1), (5, 1)])
def test_tiny_problems(m, n):
    p = _dense_prob(m, n, seed=7 * m + n, cond=10)
    maxit = min(m, n) + 1
    spec = SolverSpec(method="sflsqr", maxit=maxit, window=2, d=max(maxit, 2), s_nz=1, precond="identity")
    r = solve_problem(p, spec)
    g = _gpu_run(p, spec)
    assert g["status"] == r.status and g["info"]["k_x"] == r.k, (g["status"], r.status, g["info"], r.k)
    np.testing.assert_allclose(g["x"], r.x, rtol=1e-10, atol=1e-12 * max(np.abs(r.x).max(), 1e-300))


def test_info_bytes_model_and_delta_e():
    # sflsqr_get_info: the SURVEY.md §8(d) byte model of the last iteration, written out here
    from paper_2605_22281_b200 import solver_for_problem
    p = make_problem(3, N=96, n_angles=70, nb=137)
    spec = p.solvers[0]                                   # NONNEG tau (x each step), history on
    s = solver_for_problem(p, spec, maxit=7, eta=0.0)
    s.set_rhs(p.b)
    s.iterate(7)
    info = s.get_info()
    s.close()
    m, n, ell, k = p.m, p.n, spec.window, 7
    nnz = p.A.nnz
    expect = (12.0 * 2 * nnz + 8.0 * (m + 1) + 8.0 * (n + 1) + 16.0 * (m + n) + 8.0 * m * (2 * ell + 5)
              + 8.0 * n * (2 * ell + 3) + 16.0 * n + 8.0 * n * (k - 1) + 8.0 * m * (k + 1))
    assert info["bytes_model"] == pytest.approx(expect, rel=1e-12)
    assert info["delta_e"] == p.delta_e


def test_one_call_solve_api_matches_handle_path():
    import scipy.sparse as sp
    from paper_2605_22281_b200 import solve
    p = make_problem(4, N=64, n_angles=45, nb=91)
    spec = p.solvers[0]
    A = sp.csr_matrix((p.A.val, p.A.col, p.A.rowptr), shape=(p.m, p.n))
    B = sp.csr_matrix((p.T.val, p.T.col, p.T.rowptr), shape=(p.n, p.m))
    out = solve(A, p.b, method="sflsqr", T=B, maxit=12, window=spec.window,
                sketch=("sparse", spec.d, spec.s_nz, p.sketch_seed), precond="identity")
    g = _gpu_run(p, spec, maxit=12)
    assert np.array_equal(out["x"], g["x"]) and np.array_equal(out["true_res"], g["true_res"])


@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_tol_stop_matches_oracle(method):
    import dataclasses
    p = make_problem(1)
    spec = [s for s in p.solvers if s.method == method][0]
    full = solve_problem(p, spec, eta=0.0)
    rel = np.array(full.sketch_res) / np.linalg.norm(full.rhs)
    spec_t = dataclasses.replace(spec, tol=float(rel[9]) * (1 + 1e-7))
    r = solve_problem(p, spec_t, eta=0.0)
    assert r.status == 2
    g = _gpu_run(p, spec_t, eta=0.0)
    _compare(g, r)
