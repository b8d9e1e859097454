"""Pins of the non-uniform-grid oracle (oracle/points.py; paper footnote P:182)."""
import numpy as np
import pytest

import mmot_inputs
from oracle import points, regions, sinkhorn as osk


def _grid(seed, N, ratio=4.0):
    rng = np.random.default_rng(seed)
    h = rng.uniform(1.0, ratio, N - 1)
    x = np.concatenate([[0.0], np.cumsum(h)])
    return x / x[-1]


@pytest.mark.parametrize("l", [2, 3, 4])
def test_points_product_equals_brute_force(l):
    N = {2: 30, 3: 12, 4: 8}[l]
    x = _grid(l, N)
    phis = list(mmot_inputs.random_positive(70 + l, l, N))
    for eta in (0.05, 0.3):
        for k in range(l):
            J, Jh = points.product(phis, x, eta, k, want_hat=True)
            Jd = points.marginal_dense(phis, x, eta, k)
            assert np.max(np.abs(J - Jd) / Jd) <= 1e-13
        W = float(np.dot(phis[l - 1], Jh))
        assert W == pytest.approx(points.cost_dense(phis, x, eta), rel=1e-12)


def test_points_product_equals_uniform_oracle_on_uniform_grid():
    l, N, eta = 4, 200, 0.02
    x = np.linspace(0.0, 1.0, N)
    phis = list(mmot_inputs.random_positive(81, l, N))
    w = regions.edge_weights(l, x[1] - x[0], eta)
    for k in range(l):
        J, Jh = points.product(phis, x, eta, k, want_hat=True)
        Ju, Juh = regions.marginal_product(phis, k, w, want_hat=True)
        assert np.max(np.abs(J - Ju) / Ju) <= 1e-12
        assert np.max(np.abs(Jh - (x[1] - x[0]) * Juh) / np.abs(Jh)) <= 1e-12


def test_points_grid_refinement_with_zero_scalings():
    """Integer-multiple spacings: the non-uniform product equals the uniform product on the refined
    grid in which the inserted points carry zero scalings (they contribute no tuples; their edges
    multiply to the long edge's decay)."""
    l, eta = 3, 0.05
    steps = np.array([1, 3, 2, 1, 4, 1, 2, 5, 1, 1, 3])
    x = np.concatenate([[0], np.cumsum(steps)]).astype(float) * 0.01
    N = len(x)
    phis = list(mmot_inputs.random_positive(90, l, N))
    fine = np.arange(0, int(steps.sum()) + 1)
    pos = np.concatenate([[0], np.cumsum(steps)])
    Nf = len(fine)
    phif = [np.zeros(Nf) for _ in range(l)]
    for q in range(l):
        phif[q][pos] = phis[q]
    w = regions.edge_weights(l, 0.01, eta)
    for k in range(l):
        J = points.product(phis, x, eta, k)
        Jf = regions.marginal_product(phif, k, w)[pos]
        assert np.max(np.abs(J - Jf) / Jf) <= 1e-12


def test_points_sinkhorn_matches_uniform_driver_on_uniform_grid():
    l, N, eta, T = 3, 60, 0.05, 5
    mus = np.stack(mmot_inputs.random_marginals(5, l, N))
    x = np.linspace(0.0, 1.0, N)
    got = points.sinkhorn(mus, x, eta, T)
    ref, _, _ = osk.sinkhorn(mus, x[1] - x[0], eta, T, domain="plain")
    assert np.max(np.abs(got - ref) / ref) <= 1e-12
