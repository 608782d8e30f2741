"""NumPy emulation of the sharded data flow of SURVEY.md §8(e) over a real
torch.distributed process group (gloo on CPU).  TEST INFRASTRUCTURE: it mirrors,
step by step, what each rank of libsflsqr's sharded path holds and exchanges
(A row block, COLSHARD / ROWSHARD transpose side, n- and m-slices, the
collectives), and tests/test_sharding_cpu.py checks that the decomposition
reproduces the unsharded oracle.  It shares no code with the CUDA path.
"""
import numpy as np
import torch
import torch.distributed as dist

from oracle.lsq import householder_qr_solve
from oracle.sketch import sparse_sign_table


def _allreduce(v, op=dist.ReduceOp.SUM):
    t = torch.from_numpy(np.atleast_1d(np.asarray(v, dtype=np.float64)).copy())
    dist.all_reduce(t, op=op)
    return t.numpy()


def _allgather(v, blocks):
    """All-gather of uneven slices (padded to the largest block, like the CUDA path)."""
    mx = max(e - s for s, e in blocks)
    t = torch.zeros(mx, dtype=torch.float64)
    t[:len(v)] = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return np.concatenate([o.numpy()[:e - s] for o, (s, e) in zip(out, blocks)])


class LocalSketch:
    """Columns [c0, c1) of the global sparse-sign sketch (hash on global indices)."""

    def __init__(self, seed, d, s, c0, c1):
        self.rows, self.signs = sparse_sign_table(seed, d, s, c0, c1 - c0)
        self.d, self.scale = d, 1.0 / np.sqrt(s)

    def apply_partial(self, v):
        y = np.zeros(self.d)
        np.add.at(y, self.rows.reshape(-1), ((self.signs * self.scale) * v[:, None]).reshape(-1))
        return y


def sharded_solve(A, T, b, m_blocks, n_blocks, colshard, method, maxit, ell, seed, d, s_nz, precond, eps_rel=1e-3):
    """A (dense m x n), T (dense n x m); every rank holds the full arrays but only
    touches its blocks.  Returns (x slice, true residuals, sketched residuals)."""
    g, R = dist.get_rank(), dist.get_world_size()
    m0, m1 = m_blocks[g]
    n0, n1 = n_blocks[g]
    A_loc = A[m0:m1]                      # A row block (needs the full z)
    if colshard:
        T_loc = T[:, m0:m1]               # = (A block)^T: a partial n-vector per rank
    else:
        T_loc = T[n0:n1]                  # ROWSHARD: rows of T on the n-slice (needs the full w)
    b_loc = b[m0:m1]
    sk = LocalSketch(seed, d, s_nz, m0, m1) if method == "sflsqr" else LocalSketch(seed, d, s_nz, n0, n1)

    def dot(u, v):
        return float(_allreduce(np.dot(u, v))[0])

    def transpose_product(w_loc):
        if colshard:
            return _allreduce(T_loc @ w_loc)[n0:n1]   # emulates the reduce-scatter
        return T_loc @ _allgather(w_loc, m_blocks)

    beta = np.sqrt(dot(b_loc, b_loc))
    W = [b_loc / beta]
    z = transpose_product(W[0])
    if method == "sflsqr":
        rhs = _allreduce(sk.apply_partial(b_loc))
        SAZ = []
    else:
        Sz = _allreduce(sk.apply_partial(z))
        rhs = beta * Sz
        STW = [Sz]
    Z, P = [], []
    H = np.zeros((maxit + 1, maxit))
    x_prev = np.zeros(n1 - n0)
    true_res, sk_res = [], []
    for k in range(1, maxit + 1):
        for j in range(max(1, k - ell), k):
            c = dot(P[j - 1], z)
            z = z - c * P[j - 1]
        t = np.sqrt(dot(z, z))
        p = z / t
        P.append(p)
        if precond == "identity" or k == 1:
            zk = p.copy()
        else:   # NONNEG (R8) with a global max
            xp = np.maximum(x_prev, 0.0)
            mx = float(_allreduce(xp.max() if xp.size else -np.inf, dist.ReduceOp.MAX)[0])
            zk = (xp + eps_rel * mx) * p if mx > 0 else p.copy()
        Z.append(zk)
        w = A_loc @ _allgather(zk, n_blocks)
        if method == "sflsqr":
            SAZ.append(_allreduce(sk.apply_partial(w)))
        for j in range(max(1, k - ell), k + 1):
            h = dot(W[j - 1], w)
            H[j - 1, k - 1] = h
            w = w - h * W[j - 1]
        hn = np.sqrt(dot(w, w))
        H[k, k - 1] = hn
        W.append(w / hn)
        z = transpose_product(W[k])
        if method == "sflsqr":
            M = np.column_stack(SAZ)
        else:
            Sz = _allreduce(sk.apply_partial(z))
            M = np.column_stack(STW + [Sz]) @ H[:k + 1, :k]
            STW.append(Sz)
        y, _, _ = householder_qr_solve(M, rhs)
        sk_res.append(float(np.linalg.norm(rhs - M @ y)))
        x_loc = np.column_stack(Z) @ y
        r_loc = b_loc - A_loc @ _allgather(x_loc, n_blocks)
        true_res.append(float(np.sqrt(dot(r_loc, r_loc))))
        x_prev = x_loc
    return x_prev, true_res, sk_res
