"""N > 1 host logic on CPU (gloo, world_size 2): the partition plan and the
sharded data flow of SURVEY.md §8(e) reproduce the unsharded oracle."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2605_22281_b200.shard import balanced_row_blocks, csr_block, even_blocks


def test_balanced_row_blocks_tile_and_balance():
    rng = np.random.default_rng(0)
    cnt = rng.integers(0, 50, size=1000)
    rp = np.concatenate([[0], np.cumsum(cnt)])
    for world in (1, 2, 3, 8):
        bl = balanced_row_blocks(rp, world)
        assert bl[0][0] == 0 and bl[-1][1] == 1000
        assert all(bl[i][1] == bl[i + 1][0] for i in range(world - 1))
        loads = [rp[e] - rp[s] for s, e in bl]
        assert max(loads) - min(loads) <= 2 * cnt.max()
    assert balanced_row_blocks(np.zeros(5, dtype=np.int64), 2) == [(0, 2), (2, 4)]


def test_even_blocks_match_library_rule():
    assert even_blocks(10, 3) == [(0, 4), (4, 8), (8, 10)]
    assert even_blocks(4, 8)[-1] == (4, 4)


def test_csr_block_rebases():
    rp = np.array([0, 2, 5, 6], dtype=np.int64)
    col = np.arange(6, dtype=np.int32)
    val = np.arange(6.0)
    lrp, lc, lv = csr_block(rp, col, val, 1, 3)
    assert lrp.tolist() == [0, 3, 4] and lc.tolist() == [2, 3, 4, 5]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir, case):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        here = os.path.dirname(os.path.abspath(__file__))
        for pth in (here, os.path.dirname(here)):
            if pth not in sys.path:
                sys.path.insert(0, pth)
        from sharded_reference import sharded_solve
        from oracle.operators import DenseOperator
        from oracle.sflsqr import solve
        from oracle.sketch import SparseSignSketch
        method, colshard, precond = case
        rng = np.random.default_rng(42)
        m, n = 90, 70
        U = np.linalg.qr(rng.standard_normal((m, n)))[0]
        V = np.linalg.qr(rng.standard_normal((n, n)))[0]
        A = (U * np.logspace(0, -3, n)) @ V.T
        T = A.T.copy() if colshard else A.T + 0.02 * rng.standard_normal((n, m)) / np.sqrt(m)
        b = A @ rng.standard_normal(n)
        b += 0.02 * np.linalg.norm(b) * rng.standard_normal(m) / np.sqrt(m)
        rp = np.concatenate([[0], np.cumsum(np.full(m, n))])
        m_blocks = balanced_row_blocks(rp, world)
        n_blocks = even_blocks(n, world) if colshard else balanced_row_blocks(
            np.concatenate([[0], np.cumsum(np.full(n, m))]), world)
        # every rank computes the same plan
        plans = [None] * world
        dist.all_gather_object(plans, (m_blocks, n_blocks))
        assert all(p == plans[0] for p in plans)
        K, ell, d, s = 15, 3, 40, 4
        x_loc, tr, sk = sharded_solve(A, T, b, m_blocks, n_blocks, colshard, method, K, ell, 99, d, s, precond)
        xs = [None] * world
        dist.all_gather_object(xs, x_loc)
        x = np.concatenate(xs)
        dim = m if method == "sflsqr" else n
        r = solve(DenseOperator(A, T), b, method, maxit=K, window=ell, sketch=SparseSignSketch(99, d, s, dim),
                  precond=precond)
        rt = np.abs(np.array(tr) - np.array(r.true_res)) / np.array(r.true_res)
        rs = np.abs(np.array(sk) - np.array(r.sketch_res)) / np.array(r.sketch_res)
        ex = np.linalg.norm(x - r.x) / np.linalg.norm(r.x)
        if rank == 0:
            with open(os.path.join(outdir, "ok.txt"), "w") as f:
                f.write(f"{rt.max()} {rs.max()} {ex}\n")
        assert rt.max() < 1e-9 and rs.max() < 1e-9 and ex < 1e-6, (rt.max(), rs.max(), ex)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [("sflsqr", True, "nonneg"), ("sflsmr", True, "identity"),
                                  ("sflsqr", False, "identity"), ("sflsmr", False, "nonneg")])
def test_sharded_dataflow_gloo_world2(case):
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(2, _free_port(), td, case), nprocs=2, join=True)
        assert os.path.exists(os.path.join(td, "ok.txt"))
