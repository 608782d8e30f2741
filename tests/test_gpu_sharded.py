"""Sharded path on one GPU: world ranks as host threads of one
process (SFLSQR_COMM_LOCAL), each running the real sharded CUDA path (local A rows,
COLSHARD / ROWSHARD transpose side, all-gathers, reduce-scatters, allreduces),
against the fp64 oracle (pin P11: every world size matches the same oracle run)."""
import numpy as np
import pytest

from gen import make_problem
from oracle.sflsqr import solve_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_22281_b200._build import build_library
    build_library()


def _check_gathered(x, out):
    # sflsqr_get_x(..., SFLSQR_X_GATHERED): the whole x on every rank, bit for bit the slices' concatenation
    for o in out:
        assert np.array_equal(o[6], x)


def _check(x, tr, sk, r, n_res, res_tol=1e-9, x_tol=1e-6):
    n = min(n_res, len(r.true_res))
    rt = np.abs(tr[:n] - np.array(r.true_res[:n])) / np.array(r.true_res[:n])
    rs = np.abs(sk[:n] - np.array(r.sketch_res[:n])) / np.array(r.sketch_res[:n])
    assert rt.max() < res_tol, ("true residual", rt.max(), int(rt.argmax()) + 1)
    assert rs.max() < res_tol, ("sketched residual", rs.max(), int(rs.argmax()) + 1)
    ex = np.linalg.norm(x - r.x) / np.linalg.norm(r.x)
    assert ex < x_tol, ("x", ex)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_colshard_config3_reduced(world, method):
    from paper_2605_22281_b200.shard import run_local_group
    p = make_problem(3, N=128, n_angles=90, nb=183)
    spec = [s for s in p.solvers if s.method == method][0]
    r = solve_problem(p, spec, maxit=60, eta=0.0)
    x, tr, sk, infos, st, out = run_local_group(p, spec, world, maxit=60, eta=0.0)
    assert all(s == (True, 1) for s in st)
    assert all(i["graph"] == 0 for i in infos)         # in-process collectives are host rendezvous: eager
    assert sum(i["m_loc"] for i in infos) == p.m and sum(i["n_loc"] for i in infos) == p.n
    _check(x, tr, sk, r, 60)
    _check_gathered(x, out)


@pytest.fixture(scope="module")
def c5_reduced():
    from horizons import C5R
    return make_problem(5, **C5R)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("method", ["sflsqr", "sflsmr"])
def test_colshard_config5_reduced(c5_reduced, world, method):
    # BASELINE configs[4]'s recipe (Siddon, A^T column-sharded and built per rank, IRN-l1, ell = 5,
    # d = 600, s = 8) on a 256^2 grid, 40 iterations (inside the oracle's horizon, tests/horizons.py)
    from paper_2605_22281_b200.shard import run_local_group
    p = c5_reduced
    spec = [s for s in p.solvers if s.method == method][0]
    K = 40
    r = solve_problem(p, spec, maxit=K, eta=0.0)
    x, tr, sk, infos, st, out = run_local_group(p, spec, world, maxit=K, eta=0.0)
    assert all(s == (True, 1) for s in st)
    assert [i["n0"] for i in infos] == sorted(i["n0"] for i in infos)
    _check(x, tr, sk, r, K)
    _check_gathered(x, out)


@pytest.mark.parametrize("world", [2, 4])
def test_rowshard_config4_reduced(world):
    from paper_2605_22281_b200.shard import run_local_group
    p = make_problem(4, N=192, n_angles=135, nb=273)
    spec = p.solvers[0]
    K = 12   # inside the oracle's forward-stable horizon for this unmatched problem (test_gpu_parity)
    r = solve_problem(p, spec, maxit=K, eta=0.0)
    x, tr, sk, infos, st, out = run_local_group(p, spec, world, maxit=K, eta=0.0)
    _check(x, tr, sk, r, K)
    _check_gathered(x, out)


def test_dense_config1_world2_discrepancy_stop():
    from paper_2605_22281_b200.shard import run_local_group
    p = make_problem(1)
    spec = p.solvers[1]
    full = solve_problem(p, spec, eta=0.0)
    eta = float(full.true_res[14] / p.delta_e) * (1 + 1e-7)
    r = solve_problem(p, spec, eta=eta)
    x, tr, sk, infos, st, _ = run_local_group(p, spec, 2, eta=eta)
    assert all(s == (True, 3) for s in st) and infos[0]["k_x"] == r.k
    _check(x, tr, sk, r, len(r.true_res))


def test_world_size_invariance_close_to_single_rank():
    # P11: world sizes differ only by reduction order
    from paper_2605_22281_b200 import solver_for_problem
    from paper_2605_22281_b200.shard import run_local_group
    p = make_problem(3, N=96, n_angles=60, nb=137)
    spec = p.solvers[0]
    s = solver_for_problem(p, spec, maxit=40, eta=0.0)
    s.set_rhs(p.b)
    s.iterate(40)
    x1 = s.get_x()
    tr1, _ = s.get_residual_norms()
    s.close()
    for world in (2, 4):
        x, tr, sk, infos, st, _ = run_local_group(p, spec, world, maxit=40, eta=0.0)
        assert np.max(np.abs(tr - tr1) / tr1) < 1e-10
        assert np.linalg.norm(x - x1) / np.linalg.norm(x1) < 1e-8


def test_nccl_unique_id_available():
    from paper_2605_22281_b200.sflsqr import get_unique_id
    uid = get_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128 and any(uid)


@pytest.mark.parametrize("cfg,world", [(3, 3), (4, 2)])
def test_peer_memory_collectives_bitwise_equal_to_collectives(cfg, world):
    # peer memory (SFLSQR_KNOB_P2P_ON, the in-process default): all-gathers as direct stores into every rank's gathered buffer and the COLSHARD
    # reduce-scatter fused into the T product's epilogue (stores into the owner's receive slots),
    # each followed by a barrier; the sums run in rank order as in the in-process collectives,
    # so the two paths must agree bit for bit (config 3: COLSHARD, config 4: ROWSHARD)
    from paper_2605_22281_b200.shard import run_local_group
    kw = dict(N=96, n_angles=70, nb=137) if cfg == 3 else dict(N=128, n_angles=90, nb=183)
    p = make_problem(cfg, **kw)
    spec = p.solvers[0]
    out = {}
    for mode in ("0", "1"):
        x, tr, sk, infos, st, _ = run_local_group(p, spec, world, maxit=20, eta=0.0,
                                                  knobs=["p2p_off"] if mode == "0" else ["p2p_on"])
        out[mode] = (x, tr, sk)
    assert np.array_equal(out["0"][0], out["1"][0])
    assert np.array_equal(out["0"][1], out["1"][1]) and np.array_equal(out["0"][2], out["1"][2])
    # and the peer-memory path against the oracle
    r = solve_problem(p, spec, maxit=12, eta=0.0)
    x, tr, sk, _, _, _ = run_local_group(p, spec, world, maxit=12, eta=0.0)
    _check(x, tr, sk, r, 12)


def test_nccl_transport_one_rank_selftest():
    # the NCCL transport cannot run two ranks on one device; a ONE-rank communicator still drives
    # every entry the sharded path uses (dlopen'ed symbols and argument order, all-reduce sum / max,
    # all-gather, reduce-scatter, the setup byte all-gather, barrier, share_buffer) and the capture
    # of those calls into a CUDA graph replayed on changed inputs; results are compared with inputs
    from paper_2605_22281_b200.sflsqr import nccl_selftest
    nccl_selftest(0)
