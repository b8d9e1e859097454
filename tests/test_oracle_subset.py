"""Pins of O4, the subset-lattice DP oracle (oracle/subset.c): against the definition written out
(O1 dense contraction), the paper's region recursion (O3, §4.2), closed
forms, and the tangent against the dense cost-weighted product."""
import math

import numpy as np
import pytest

from oracle import dense, regions, subset


def _phis(seed, l, N, lo=0.1, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, (l, N))


@pytest.mark.parametrize("l,N", [(2, 7), (3, 6), (4, 5), (5, 4), (6, 3), (7, 4), (8, 3)])
@pytest.mark.parametrize("lam", [0.3, 0.8])
def test_subset_equals_dense_definition(l, N, lam):
    phis = _phis(10 * l + N, l, N)
    w = regions.edge_weights_lambda(l, lam)
    h = 1.0 / (N - 1)
    eta = -h / math.log(lam)
    K = dense.kernel_tensor(l, N, h, eta)
    for k in range(l):
        got = subset.marginal_product(list(phis), k, w)
        want = dense.contract(K, list(phis), k)
        np.testing.assert_allclose(got, want, rtol=1e-13)


@pytest.mark.parametrize("l", [3, 4, 5, 6])
def test_subset_equals_region_chains(l):
    N = 150
    phis = _phis(77 + l, l, N)
    w = regions.edge_weights(l, 1.0 / (N - 1), 0.05)
    for k in range(l):
        got, gh = subset.marginal_product(list(phis), k, w, want_hat=True)
        want, wh = regions.marginal_product(list(phis), k, w, want_hat=True)
        np.testing.assert_allclose(got, want, rtol=1e-13)
        np.testing.assert_allclose(gh, wh, rtol=1e-12)


@pytest.mark.parametrize("l", [3, 4, 7, 8])
def test_subset_tangent_equals_cost_weighted_dense(l):
    """Jhat_k = sum_i E(i) lambda^E(i) prod phi: the dense (E . K) contraction."""
    N = 5 if l <= 4 else 3
    phis = _phis(5 + l, l, N)
    h, eta = 1.0 / (N - 1), 0.3
    w = regions.edge_weights(l, h, eta)
    K = dense.kernel_tensor(l, N, h, eta)
    E = dense.exponent_tensor(l, N)
    for k in range(l):
        _, jh = subset.marginal_product(list(phis), k, w, want_hat=True)
        np.testing.assert_allclose(jh, dense.contract(E * K, list(phis), k), rtol=1e-13)


def test_subset_closed_forms():
    """lambda = 1: J_k = prod_{q != k} sum phi_q; lambda -> 0 (w_a = 0 for 0 < a < l):
    J_k[m] = prod_{q != k} phi_q[m]; N = 1: prod phi_q[0]."""
    l, N = 5, 40
    phis = _phis(3, l, N)
    for k in range(l):
        ones = subset.marginal_product(list(phis), k, np.ones(l + 1))
        np.testing.assert_allclose(ones, np.prod([phis[q].sum() for q in range(l) if q != k]), rtol=1e-13)
        w0 = np.array([1.0] + [0.0] * (l - 1) + [1.0])
        diag = subset.marginal_product(list(phis), k, w0)
        np.testing.assert_allclose(diag, np.prod([phis[q] for q in range(l) if q != k], axis=0), rtol=1e-14)
    one = subset.marginal_product([np.array([2.0]), np.array([3.0]), np.array([5.0])], 1, np.ones(4))
    assert one[0] == 10.0


@pytest.mark.parametrize("l", [3, 5, 7, 8])
def test_subset_log_equals_plain_and_handles_zeros(l):
    N = 120
    phis = _phis(9 + l, l, N)
    phis[1, 30:60] = 0.0
    h, eta = 1.0 / (N - 1), 0.02
    w = regions.edge_weights(l, h, eta)
    lw = np.array([-(a * (l - a)) * h / eta for a in range(l + 1)])
    with np.errstate(divide="ignore"):
        gs = np.log(phis)
    for k in range(l):
        plain = subset.marginal_product(list(phis), k, w)
        lg = subset.marginal_product_log(list(gs), k, lw)
        np.testing.assert_allclose(np.exp(lg), plain, rtol=1e-12)
    # beyond fp64 range: shifting g_q by c_q with sum c_q = 0 leaves plan entries unchanged, and
    # J_k shifts by -c_k (A16)
    c = np.array([900.0, -400.0, -500.0] + [0.0] * (l - 3))
    lg0 = subset.marginal_product_log(list(gs), 0, lw)
    lg1 = subset.marginal_product_log(list(gs + c[:, None]), 0, lw)
    fin = np.isfinite(lg0)
    np.testing.assert_allclose(lg1[fin], lg0[fin] - c[0], rtol=0, atol=1e-10)


def test_sinkhorn_engines_agree():
    """The Sinkhorn driver on O4 products equals the driver on O3 products (plain and log)."""
    from oracle import sinkhorn
    rng = np.random.default_rng(5)
    l, N = 5, 200
    mus = rng.uniform(0.1, 1, (l, N))
    mus /= mus.sum(axis=1, keepdims=True)
    h, eta = 1.0 / (N - 1), 0.02
    for dom in ("plain", "log"):
        a, _, ra = sinkhorn.sinkhorn(mus, h, eta, 4, tol=1e-300, domain=dom)
        b, _, rb = sinkhorn.sinkhorn(mus, h, eta, 4, tol=1e-300, domain=dom, engine="subset")
        np.testing.assert_allclose(a, b, rtol=1e-11, atol=1e-12)
        assert ra == pytest.approx(rb, rel=1e-10)
