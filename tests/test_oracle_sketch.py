"""Pin P1: Philox4x32-10 and the sparse-sign sketch table (oracle side).

Sketch definition: DESIGN.md readings R5/R6 (paper: Gaussian L550-552,
CountSketch L1390/L1615; BASELINE.json: sparse-sign with s nonzeros/column).
"""
import os

import numpy as np
import pytest

from oracle.philox import philox4x32_10
from oracle.sketch import SparseSignSketch, sparse_sign_table

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kat():
    out = []
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        w = [int(t, 16) for t in line.split()]
        out.append((w[0:4], w[4:6], w[6:10]))
    return out


def test_philox_known_answer_vectors():
    kats = _kat()
    assert len(kats) == 3
    for ctr, key, exp in kats:
        got = [int(v) for v in philox4x32_10(ctr, key)]
        assert got == exp


def test_philox_vectorised_equals_scalar():
    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2**32, size=(50, 4), dtype=np.uint64)
    key = np.array([0x12345678, 0x9ABCDEF0], dtype=np.uint64)
    vec = philox4x32_10(ctr, key)
    for i in range(50):
        assert list(vec[i]) == list(philox4x32_10(ctr[i], key))


@pytest.mark.parametrize("d,s", [(80, 4), (200, 8), (7, 7), (5, 1), (600, 8)])
def test_table_structure(d, s):
    rows, signs = sparse_sign_table(0x5F1A5E, d, s, 0, 3000)
    assert rows.shape == (3000, s) and signs.shape == (3000, s)
    assert rows.min() >= 0 and rows.max() < d
    assert set(np.unique(signs)) <= {-1, 1}
    for i in range(3000):
        assert len(set(rows[i].tolist())) == s          # exactly s distinct rows


def test_table_offset_consistency():
    # a slice starting at col0 equals the same columns of the full table (global index in the hash)
    r_all, s_all = sparse_sign_table(99, 300, 8, 0, 5000)
    r_sl, s_sl = sparse_sign_table(99, 300, 8, 1234, 777)
    assert np.array_equal(r_all[1234:1234 + 777], r_sl)
    assert np.array_equal(s_all[1234:1234 + 777], s_sl)


def test_rows_uniform_and_signs_balanced():
    d, s, ncol = 50, 4, 40000
    rows, signs = sparse_sign_table(7, d, s, 0, ncol)
    cnt = np.bincount(rows.reshape(-1), minlength=d)
    expected = ncol * s / d
    chi2 = float(((cnt - expected) ** 2 / expected).sum())
    # chi^2 with 49 dof: P(chi2 > 95) < 1e-4
    assert chi2 < 95.0, chi2
    frac_neg = float((signs < 0).mean())
    assert abs(frac_neg - 0.5) < 0.01


def test_sketch_norm_unbiased():
    # E ||S v||^2 = ||v||^2 (values +-1/sqrt(s)), over 500 seeds within 10%
    rng = np.random.default_rng(3)
    v = rng.standard_normal(200)
    vals = [np.sum(SparseSignSketch(seed, 40, 4, 200).apply(v) ** 2) for seed in range(500)]
    assert abs(np.mean(vals) / np.dot(v, v) - 1.0) < 0.1


def test_countsketch_unit_vectors():
    sk = SparseSignSketch(11, 30, 1, 100)
    for j in (0, 17, 99):
        e = np.zeros(100)
        e[j] = 1.0
        y = sk.apply(e)
        nz = np.flatnonzero(y)
        assert nz.tolist() == [sk.rows[j, 0]]
        assert y[nz[0]] == float(sk.signs[j, 0])


def test_apply_equals_dense_materialisation():
    sk = SparseSignSketch(5, 60, 8, 500)
    S = sk.dense()
    rng = np.random.default_rng(1)
    for _ in range(20):
        v = rng.standard_normal(500)
        np.testing.assert_allclose(sk.apply(v), S @ v, rtol=1e-12, atol=1e-12)
    # each column has s nonzeros of magnitude 1/sqrt(s)
    assert np.all((S != 0).sum(axis=0) == 8)
    np.testing.assert_allclose(np.abs(S[S != 0]), 1 / np.sqrt(8))


def test_table_seed_sensitivity():
    r1, _ = sparse_sign_table(1, 400, 8, 0, 1000)
    r2, _ = sparse_sign_table(2, 400, 8, 0, 1000)
    assert (r1 != r2).mean() > 0.9
    r3, _ = sparse_sign_table(1 + (1 << 32), 400, 8, 0, 1000)   # high seed word is used
    assert (r1 != r3).mean() > 0.9


# ---------------------------------------------------------------- Gaussian sketch (reading R21)
def test_gaussian_sketch_is_standard_normal_iid():
    from scipy import stats
    from oracle.sketch import gaussian_table
    d, n = 64, 4000
    S = gaussian_table(0xC0FFEE, d, 0, n) * np.sqrt(d)            # N(0, 1) entries
    g = S.reshape(-1)
    assert stats.kstest(g, "norm").pvalue > 1e-3                   # marginal: standard normal
    assert abs(g.mean()) < 4 / np.sqrt(g.size) and abs(g.var() - 1) < 5 * np.sqrt(2 / g.size)
    C = np.corrcoef(S)                                              # rows uncorrelated
    off = C[~np.eye(d, dtype=bool)]
    assert np.abs(off).max() < 6 / np.sqrt(n)
    # cos/sin pair of one Box-Muller draw: independent, jointly rotation invariant
    assert abs(np.corrcoef(S[0], S[1])[0, 1]) < 6 / np.sqrt(n)
    assert stats.kstest(np.arctan2(S[1], S[0]) / (2 * np.pi) + 0.5, "uniform").pvalue > 1e-3


def test_gaussian_sketch_norm_preservation_and_columns():
    from oracle.sketch import GaussianSketch, gaussian_table
    rng = np.random.default_rng(0)
    v = rng.standard_normal(300)
    r = [np.linalg.norm(GaussianSketch(seed, 50, 300).apply(v)) ** 2 for seed in range(200)]
    assert abs(np.mean(r) / (v @ v) - 1) < 0.05                   # E||S v||^2 = ||v||^2
    S = gaussian_table(7, 9, 0, 40)                                 # column windows = the full table
    np.testing.assert_array_equal(gaussian_table(7, 9, 13, 20), S[:, 13:33])
    # row r of the draw does not depend on d (pairs (2t, 2t+1) share one counter)
    np.testing.assert_allclose(gaussian_table(7, 10, 0, 40)[:9] * np.sqrt(10), S * np.sqrt(9), rtol=1e-15)
