"""Pin P8: the input generators (Siddon A, pixel-driven B, blur, phantoms, noise).

The generator is input infrastructure shared by the oracle and the CUDA path;
these tests pin it against brute-force geometry, not against itself.
"""
import math

import numpy as np
import pytest

from gen import CSR, make_problem, pixbp_csr, siddon_csr
from gen.problems import gen_blur_apply
from oracle.operators import BlurOperator, OracleCSR


def _clip_len(px, py, dx, dy, x0, x1, y0, y1):
    """Length of {p + s d} inside the closed box [x0,x1]x[y0,y1] (Liang-Barsky)."""
    lo, hi = -math.inf, math.inf
    for p, d, a, b in ((px, dx, x0, x1), (py, dy, y0, y1)):
        if abs(d) < 1e-14:
            if p < a or p > b:
                return 0.0
        else:
            s1, s2 = (a - p) / d, (b - p) / d
            lo, hi = max(lo, min(s1, s2)), min(hi, max(s1, s2))
    return max(0.0, hi - lo)


def test_siddon_equals_bruteforce_pixel_clipping():
    N, na, nb = 16, 7, 24          # nb even: no ray lies on a grid line
    A = siddon_csr(N, na, nb)
    D = A.to_dense()
    half = N / 2
    for a in range(na):
        th = math.pi * a / na
        for j in range(nb):
            t = j - (nb - 1) / 2
            px, py, dx, dy = t * math.cos(th), t * math.sin(th), -math.sin(th), math.cos(th)
            row = np.zeros(N * N)
            for iy in range(N):
                for ix in range(N):
                    row[iy * N + ix] = _clip_len(px, py, dx, dy, ix - half, ix - half + 1, iy - half, iy - half + 1)
            row[row <= 1e-10] = 0.0
            np.testing.assert_allclose(D[a * nb + j], row, atol=1e-12)


def test_siddon_row_sums_are_chord_lengths_and_canonical():
    N, na, nb = 32, 13, 47
    A = siddon_csr(N, na, nb)
    half = N / 2
    for r in range(A.nrows):
        a, j = divmod(r, nb)
        th = math.pi * a / na
        t = j - (nb - 1) / 2
        chord = _clip_len(t * math.cos(th), t * math.sin(th), -math.sin(th), math.cos(th), -half, half, -half, half)
        s, e = A.rowptr[r], A.rowptr[r + 1]
        if abs(math.sin(th)) > 1e-12 and abs(math.cos(th)) > 1e-12:
            assert abs(A.val[s:e].sum() - chord) < 1e-9
        cols = A.col[s:e]
        assert np.all(np.diff(cols) > 0) and (cols.size == 0 or (cols[0] >= 0 and cols[-1] < N * N))
        assert np.all(A.val[s:e] > 0)


def test_siddon_axis_aligned_rays_half_open_convention():
    # theta = 0, nb odd: every ray lies on a vertical grid line; it belongs to the pixel column on
    # its positive side (half-open pixels), and the line x = +N/2 is outside the grid.
    N, nb = 8, 11
    A = siddon_csr(N, 2, nb)
    D = A.to_dense()
    for j in range(nb):
        t = j - (nb - 1) / 2
        row = D[j]
        if -N / 2 <= t < N / 2:
            ix = int(math.floor(t + N / 2))
            expect = np.zeros(N * N)
            expect[[iy * N + ix for iy in range(N)]] = 1.0
            np.testing.assert_allclose(row, expect, atol=1e-12)
        else:
            assert not row.any()


def test_unit_image_horizontal_ray():
    # SPEC operators example: uniform unit image, horizontal ray -> width x pixel size
    N, na, nb = 16, 2, 16
    A = siddon_csr(N, na, nb)
    ones = np.ones(N * N)
    y = A.matvec(ones)
    # angle index 1 = pi/2: rays are horizontal (direction (-1, 0)), offsets t_j = j - 7.5
    np.testing.assert_allclose(y[nb:2 * nb], N, rtol=1e-12)


def test_pixel_driven_B_mass_and_structure():
    N, na, nb = 24, 9, 35
    B = pixbp_csr(N, na, nb)
    assert B.nrows == N * N and B.ncols == na * nb
    for p in range(B.nrows):
        s, e = B.rowptr[p], B.rowptr[p + 1]
        cols = B.col[s:e]
        assert np.all(np.diff(cols) > 0)
        # interior pixels: each angle contributes weights (1-f, f) summing to 1
        per_angle = np.bincount(cols // nb, weights=B.val[s:e], minlength=na)
        np.testing.assert_allclose(per_angle, 1.0, atol=1e-12)
    # B approximates A^T: relative difference of products is small but nonzero (unmatched)
    A = siddon_csr(N, na, nb)
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal(N * N), rng.standard_normal(na * nb)
    x /= np.linalg.norm(x)
    y /= np.linalg.norm(y)
    asym = abs(y @ A.matvec(x) - x @ B.matvec(y))
    assert 0 < asym < 0.5


def test_oracle_transpose_is_exact_and_adjoint_consistent():
    A = siddon_csr(20, 11, 29)
    Ao = OracleCSR(A.nrows, A.ncols, A.rowptr, A.col, A.val)
    At = Ao.transpose()
    np.testing.assert_array_equal(CSR(At.nrows, At.ncols, At.rowptr, At.col, At.val).to_dense(), A.to_dense().T)
    rng = np.random.default_rng(1)
    for _ in range(50):
        x, y = rng.standard_normal(A.ncols), rng.standard_normal(A.nrows)
        lhs, rhs = y @ Ao.matvec(x), x @ At.matvec(y)
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def test_blur_dense_assembly_and_symmetry():
    H = W = 12
    sigma, r = 2.5, 7
    op = BlurOperator(H, W, sigma, r)
    # dense assembly from the 1-D Toeplitz factors: A = K (x) K for row-major x
    t = np.arange(-r, r + 1)
    g = np.exp(-t * t / (2 * sigma * sigma))
    g /= g.sum()
    K = np.zeros((W, W))
    for i in range(W):
        for j in range(W):
            if abs(i - j) <= r:
                K[i, j] = g[j - i + r]
    Ad = np.kron(K, K)
    Dm = np.column_stack([op.matvec(np.eye(H * W)[:, i]) for i in range(H * W)])
    np.testing.assert_allclose(Dm, Ad, atol=1e-15)
    np.testing.assert_allclose(Dm, Dm.T, atol=1e-15)
    x = np.random.default_rng(2).standard_normal(H * W)
    np.testing.assert_allclose(gen_blur_apply(x, H, W, sigma, r), Ad @ x, atol=1e-13)
    # DC preservation away from the boundary: constant image -> interior pixels unchanged
    Y = op.matvec(np.ones(H * W)).reshape(H, W)
    assert abs(Y[H // 2, W // 2] - (K[W // 2].sum()) ** 2) < 1e-14


@pytest.mark.parametrize("idx", [1, 2])
def test_problem_recipes_small(idx):
    p = make_problem(idx)
    assert p.b.shape == (p.m,) and p.x_true.shape == (p.n,)
    Ax = p.b - p.e
    assert abs(np.linalg.norm(p.e) / np.linalg.norm(Ax) - p.delta) < 1e-12
    assert p.delta_e == pytest.approx(p.delta * np.linalg.norm(Ax), rel=1e-12)
    p2 = make_problem(idx)
    np.testing.assert_array_equal(p.b, p2.b)          # seeded, deterministic
    if idx == 1:
        sv = np.linalg.svd(p.A.to_dense(), compute_uv=False)
        np.testing.assert_allclose(sv, 10.0 ** (-6.0 * np.arange(256) / 255), rtol=1e-8)
        assert set(np.unique(p.x_true)) <= set(np.unique(p.x_true))  # piecewise constant
        assert len(np.unique(p.x_true)) <= 5
    else:
        assert np.count_nonzero(p.x_true) == 1311
        nz = p.x_true[p.x_true != 0]
        assert nz.min() >= 0.5 and nz.max() <= 1.0


def test_ct_recipe_reduced():
    p = make_problem(3, N=64, n_angles=45, nb=91)
    assert p.m == 45 * 91 and p.n == 64 * 64
    assert p.x_true.min() >= 0 and p.x_true.max() > 0
    p4 = make_problem(4, N=48, n_angles=30, nb=69)
    assert p4.t_mode == "given" and p4.T.nrows == 48 * 48 and p4.T.ncols == 30 * 69


@pytest.mark.parametrize("cfg,world", [(3, 2), (4, 3)])
def test_ct_shards_reassemble_the_problem(cfg, world):
    # the multi-GPU bench's per-rank generation (make_ct_shard) must produce exactly the rows of
    # make_problem's operators and the matching slices of b
    from gen.problems import ct_row_nnz, make_ct_shard
    from paper_2605_22281_b200.shard import balanced_row_blocks
    geo = dict(N=48, n_angles=33, nb=71)
    p = make_problem(cfg, **geo)
    a_cnt, t_cnt = ct_row_nnz(cfg, **geo)
    np.testing.assert_array_equal(a_cnt, np.diff(p.A.rowptr))
    ab = balanced_row_blocks(np.concatenate([[0], np.cumsum(a_cnt)]), world)
    tb = None if t_cnt is None else balanced_row_blocks(np.concatenate([[0], np.cumsum(t_cnt)]), world)
    # the ranks' all-reduce of their partial ||A x_true||^2, emulated by the global value
    ax2 = float((p.b - p.e) @ (p.b - p.e))
    shards = [make_ct_shard(cfg, ab[g], None if tb is None else tb[g], lambda v: ax2, **geo) for g in range(world)]
    for g, sh in enumerate(shards):
        r0, r1 = ab[g]
        s, e = p.A.rowptr[r0], p.A.rowptr[r1]
        np.testing.assert_array_equal(sh.A_loc.col, p.A.col[s:e])
        np.testing.assert_array_equal(sh.A_loc.val, p.A.val[s:e])
        np.testing.assert_allclose(sh.b_loc, p.b[r0:r1], rtol=1e-13, atol=1e-13 * np.abs(p.b).max())
        assert abs(sh.delta_e - p.delta_e) <= 1e-12 * p.delta_e
        if tb is not None:
            t0, t1 = tb[g]
            s, e = p.T.rowptr[t0], p.T.rowptr[t1]
            np.testing.assert_array_equal(sh.T_loc.col, p.T.col[s:e])
            np.testing.assert_array_equal(sh.T_loc.val, p.T.val[s:e])
