"""Pins of O3 (oracle/regions.c: §4.2 region chains) against the definitions and invariants."""
import itertools
import math

import numpy as np
import pytest

from oracle import dense, paper3, regions

SIZES = {2: 11, 3: 9, 4: 7, 5: 5, 6: 4}


def _rand(seed, l, N, lo=0.1, hi=1.0):
    rng = np.random.default_rng(seed)
    return [rng.uniform(lo, hi, N) for _ in range(l)]


@pytest.mark.parametrize("l", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("lam", [1e-3, 0.3, 0.8, 0.999])
def test_regions_equal_dense(l, lam):
    N = SIZES[l]
    ph = _rand(l * 100 + int(lam * 1000), l, N)
    K = dense.kernel_tensor_lambda(l, N, lam)
    E = dense.exponent_tensor(l, N).astype(float)
    w = regions.edge_weights_lambda(l, lam)
    for k in range(l):
        J, Jh = regions.marginal_product(ph, k, w, want_hat=True)
        np.testing.assert_allclose(J, dense.contract(K, ph, k), rtol=1e-13)
        np.testing.assert_allclose(Jh, dense.contract(E * K, ph, k), rtol=1e-13)


@pytest.mark.parametrize("l", [3, 4])
def test_each_region_is_its_order_set(l):
    """Region r of the chain code sums exactly the tuples of its order set (strictness S:412)."""
    N = 4
    ph = _rand(7 + l, l, N)
    w = regions.edge_weights_lambda(l, 0.6)
    K = dense.kernel_tensor_lambda(l, N, 0.6)
    perms = list(itertools.permutations(range(l)))
    total = np.zeros(N)
    for ridx, pi in enumerate(perms):
        got = regions.marginal_product(ph, 0, w, region=ridx)
        want = np.zeros(N)
        for idx in itertools.product(range(N), repeat=l):
            pos = [idx[q] for q in pi]
            ok = all(pos[r] < pos[r + 1] if pi[r] > pi[r + 1] else pos[r] <= pos[r + 1] for r in range(l - 1))
            if ok:
                term = K[idx]
                for q in range(1, l):
                    term *= ph[q][idx[q]]
                want[idx[0]] += term
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-300)
        total += got
    np.testing.assert_allclose(total, dense.contract(K, ph, 0), rtol=1e-13)


def test_regions_l3_equals_algorithm2():
    ph = _rand(3, 3, 200)
    lam = 0.97
    w = regions.edge_weights_lambda(3, lam)
    np.testing.assert_allclose(regions.marginal_product(ph, 2, w), paper3.ftvp1(ph[0], ph[1], lam), rtol=1e-12)
    h = 0.05
    _, Jh = regions.marginal_product(ph, 2, w, want_hat=True)
    np.testing.assert_allclose(h * Jh, paper3.ftvp2(ph[0], ph[1], lam, h), rtol=1e-12)


@pytest.mark.parametrize("l", [2, 3, 4, 5, 6])
def test_closed_forms(l):
    N = 6
    ph = _rand(50 + l, l, N)
    for k in range(l):
        J1 = regions.marginal_product(ph, k, regions.edge_weights_lambda(l, 1.0))
        np.testing.assert_allclose(J1, np.prod([ph[q].sum() for q in range(l) if q != k]), rtol=1e-13)
        J0 = regions.marginal_product(ph, k, regions.edge_weights_lambda(l, 0.0))
        np.testing.assert_allclose(J0, np.prod([ph[q] for q in range(l) if q != k], axis=0), rtol=1e-14)
    one = [p[:1] for p in ph]
    assert regions.marginal_product(one, 0, regions.edge_weights_lambda(l, 0.5))[0] == pytest.approx(
        np.prod([p[0] for p in one[1:]]), rel=1e-15)


@pytest.mark.parametrize("l", [3, 4, 5])
def test_invariants(l):
    """Symmetry in the bound vectors, reversal equivariance, multilinearity,
    mass identity <phi_k, J_k> independent of k (= plan mass)."""
    N = 37
    ph = _rand(77 + l, l, N)
    w = regions.edge_weights_lambda(l, 0.9)
    J0 = regions.marginal_product(ph, 0, w)
    perm = [0] + list(reversed(range(1, l)))
    np.testing.assert_allclose(regions.marginal_product([ph[q] for q in perm], 0, w), J0, rtol=1e-13)
    Jr = regions.marginal_product([p[::-1].copy() for p in ph], 0, w)
    np.testing.assert_allclose(Jr[::-1], J0, rtol=1e-13)
    ph2 = list(ph)
    ph2[1] = 2.5 * ph[1]
    np.testing.assert_allclose(regions.marginal_product(ph2, 0, w), 2.5 * J0, rtol=1e-14)
    masses = [np.dot(ph[k], regions.marginal_product(ph, k, w)) for k in range(l)]
    np.testing.assert_allclose(masses, masses[0], rtol=1e-13)


@pytest.mark.parametrize("l", [2, 4, 6])
def test_log_domain_equals_plain(l):
    N = 300
    ph = _rand(9 + l, l, N)
    h, eta = 1.0 / (N - 1), 0.01
    w = regions.edge_weights(l, h, eta)
    lw = np.array([-(a * (l - a)) * h / eta for a in range(l + 1)])
    for k in (0, l - 1):
        J = regions.marginal_product(ph, k, w)
        Jl = regions.marginal_product_log([np.log(p) for p in ph], k, lw)
        np.testing.assert_allclose(np.exp(Jl), J, rtol=1e-12)


def test_log_domain_handles_zero_scalings():
    l, N = 4, 20
    ph = _rand(5, l, N)
    ph[1][3:7] = 0.0
    h, eta = 0.05, 0.1
    w = regions.edge_weights(l, h, eta)
    lw = np.log(w)
    with np.errstate(divide="ignore"):
        g = [np.log(p) for p in ph]
    J = regions.marginal_product(ph, 0, w)
    Jl = regions.marginal_product_log(g, 0, lw)
    assert np.all(np.isfinite(Jl))
    np.testing.assert_allclose(np.exp(Jl), J, rtol=1e-12)


def test_tangent_equals_central_difference():
    """hat J = lambda dJ/dlambda (SURVEY [verified]); central difference in log lambda."""
    l, N = 4, 30
    ph = _rand(99, l, N)
    lam, d = 0.8, 1e-5
    _, Jh = regions.marginal_product(ph, 1, regions.edge_weights_lambda(l, lam), want_hat=True)
    Jp = regions.marginal_product(ph, 1, regions.edge_weights_lambda(l, lam * math.exp(d)))
    Jm = regions.marginal_product(ph, 1, regions.edge_weights_lambda(l, lam * math.exp(-d)))
    np.testing.assert_allclose(Jh, (Jp - Jm) / (2 * d), rtol=1e-8)
