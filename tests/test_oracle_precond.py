"""Pin P9: the flexible preconditioners' weights, oracle.sflsqr.tau_apply (readings R7, R8).

PAPER.md L59-64 fixes only the mechanism: IRLS approximates the l_p (semi)norm by a weighted
2-norm, and "the inverses of the weights ... appear as variable preconditioners on the right of
A".  So with D = W^{-1} the weight W(x) must satisfy the two textbook IRLS properties, which are
checked here against definitions that do not pass through tau_apply's formula:

  * the weighted 2-norm reproduces the l_p norm: sum_i x_i^2 W_i^2 -> ||x||_p^p as eps -> 0,
    with an error that vanishes like eps^2 (a sign error in the exponent gives ||x||_{4-p}^{4-p});
  * majorisation / gradient matching: W(x)^2 ⊙ x is the gradient of the smoothed penalty
    Phi(x) = (1/p) sum_i (x_i^2 + eps^2)^{p/2} at the current x (finite differences of Phi);
  * p = 2 (the plain 2-norm) gives W = I; D_1 = I (x_0 = 0).

NONNEG (BASELINE.json config 3, not in the paper; reading R8) is pinned by the properties that
define a multiplicative nonnegativity scaling: D > 0, D depends on x only through x_+, it is
monotone in x_+, positively homogeneous, and D = I when x has no positive entry.
"""
import numpy as np
import pytest

from oracle.sflsqr import tau_apply


def _D(kind, x, p=1.0, eps_rel=1e-3, k=2):
    # the diagonal of tau_k, read off tau_k applied to the all-ones direction
    return tau_apply(kind, np.ones_like(x), x, k, p_exp=p, eps_rel=eps_rel)


def _x(seed, n=400, lo=1e-2):
    rng = np.random.default_rng(seed)
    mag = rng.uniform(lo, 1.0, n)                 # bounded away from 0 so the eps -> 0 limit is uniform
    return mag * rng.choice([-1.0, 1.0], n) * rng.uniform(0.5, 3.0)


# ---------------------------------------------------------------- IRN (R7) ----
@pytest.mark.parametrize("p", [1.0, 0.5, 1.5])
def test_irn_weighted_norm_tends_to_lp_norm(p):
    x = _x(1)
    lp = float(np.sum(np.abs(x) ** p))
    errs = []
    for eps_rel in (1e-2, 1e-3, 1e-4, 1e-6):
        W = 1.0 / _D("irn", x, p, eps_rel)
        errs.append(abs(float(np.sum((W * x) ** 2)) - lp) / lp)
    assert errs[-1] < 1e-8, errs
    # second-order convergence in eps: each 10x smaller eps cuts the error ~100x
    assert errs[1] < 2e-2 * errs[0] and errs[2] < 2e-2 * errs[1], errs
    # the mirrored exponent (p - 2)/4 would give the (4 - p)-norm instead
    wrong = float(np.sum(np.abs(x) ** (4.0 - p)))
    assert abs(float(np.sum((x / _D("irn", x, p, 1e-6)) ** 2)) - wrong) > 1e-3 * wrong


@pytest.mark.parametrize("p", [1.0, 0.5])
def test_irn_weights_match_gradient_of_smoothed_penalty(p):
    x = _x(2, n=60)
    eps_rel = 0.05
    eps = eps_rel * float(np.max(np.abs(x)))

    def phi(v):                                   # (1/p) sum (v^2 + eps^2)^{p/2}, eps held fixed
        return float(np.sum((v * v + eps * eps) ** (p / 2.0))) / p

    h = 1e-6
    grad = np.array([(phi(x + h * e) - phi(x - h * e)) / (2 * h) for e in np.eye(x.size)])
    W2 = 1.0 / _D("irn", x, p, eps_rel) ** 2
    np.testing.assert_allclose(W2 * x, grad, rtol=1e-7, atol=1e-9)


def test_irn_special_cases():
    x = _x(3)
    np.testing.assert_array_equal(_D("irn", x, p=2.0), np.ones_like(x))      # plain 2-norm: no reweighting
    np.testing.assert_array_equal(_D("irn", x, k=1), np.ones_like(x))        # D_1 = I (x_0 = 0)
    np.testing.assert_array_equal(_D("irn", np.zeros(7)), np.ones(7))        # x = 0: no scale to weight by
    # eps relative to max|x|: D(c x) = |c|^{(2-p)/2} D(x)
    for p, c in ((1.0, 7.0), (0.5, -0.3)):
        np.testing.assert_allclose(_D("irn", c * x, p), abs(c) ** ((2 - p) / 2) * _D("irn", x, p), rtol=1e-13)
    # l_p with p < 2 penalises small entries more: the preconditioner amplifies large |x_i| most
    D = _D("irn", x, 1.0)
    order = np.argsort(np.abs(x))
    assert np.all(np.diff(D[order]) >= 0)
    # tau is the diagonal scaling itself: tau(v) = D ⊙ v for any direction v
    v = np.random.default_rng(4).standard_normal(x.size)
    np.testing.assert_array_equal(tau_apply("irn", v, x, 3), D * v)


# ---------------------------------------------------------------- NONNEG (R8) --
def test_nonneg_positive_and_depends_only_on_positive_part():
    rng = np.random.default_rng(5)
    x = rng.standard_normal(500)
    D = _D("nonneg", x)
    assert np.all(D > 0)                                  # SPD scaling: reduction P4b applies
    np.testing.assert_array_equal(D, _D("nonneg", np.maximum(x, 0.0)))
    # entries at or below zero share the smallest weight; positive entries are strictly above it
    neg = x <= 0
    assert np.ptp(D[neg]) == 0 and D[~neg].min() > D[neg][0]
    # D(c x) = c D(x) for c > 0 (a multiplicative scaling, MRNSD-like)
    np.testing.assert_allclose(_D("nonneg", 3.5 * x), 3.5 * D, rtol=1e-15)


def test_nonneg_monotone_in_each_positive_entry():
    rng = np.random.default_rng(6)
    x = np.abs(rng.standard_normal(50))
    x[0] = 2 * x.max()                                   # keep max fixed while other entries move
    D0 = _D("nonneg", x)
    for i in range(1, 50):
        y = x.copy()
        y[i] = y[i] * 1.5
        Dy = _D("nonneg", y)
        assert Dy[i] > D0[i]
        np.testing.assert_array_equal(np.delete(Dy, i), np.delete(D0, i))


def test_nonneg_identity_fallbacks():
    np.testing.assert_array_equal(_D("nonneg", -np.abs(_x(7))), np.ones(400))  # no positive entry
    np.testing.assert_array_equal(_D("nonneg", _x(7), k=1), np.ones(400))       # D_1 = I
    np.testing.assert_array_equal(_D("nonneg", np.zeros(9)), np.ones(9))
    # the floor keeps zero entries reachable: smallest / largest weight = eps_rel / (1 + eps_rel)
    x = np.array([0.0, 1.0, 4.0])
    D = _D("nonneg", x, eps_rel=1e-3)
    assert D.min() / D.max() == pytest.approx(1e-3 / (1 + 1e-3), rel=1e-14)
