"""Pins of O6 (oracle/grid2d.py, 2-D grids, §4.1): Algorithm 6 against the tensor-vector
product written out, the separable closed forms, the transposition symmetry, and the 2-D cost
against the explicit plan."""
import math

import numpy as np
import pytest

from oracle import grid2d, paper3


def _rand(seed, n):
    return np.random.default_rng(seed).uniform(0.1, 1.0, n)


@pytest.mark.parametrize("N,M", [(1, 1), (1, 5), (5, 1), (2, 3), (4, 4), (5, 6), (7, 3)])
@pytest.mark.parametrize("eps", [0.3, 0.05])
def test_ftvp_2d_equals_dense(N, M, eps):
    h1, h2 = 1.0 / max(N - 1, 1), 0.7 / max(M - 1, 1)
    phis = [_rand(10 * N + M + q, N * M) for q in range(3)]
    for k in range(3):
        got = grid2d.product(phis, k, N, M, h1, h2, eps)
        want = grid2d.dense_product(phis, k, N, M, h1, h2, eps)
        np.testing.assert_allclose(got, want, rtol=1e-13)


def test_ftvp_2d_separable_inputs():
    """phi = a (x) c, psi = b (x) d (rank one): J = FTVP-1(a, b; lambda1) (x) FTVP-1(c, d; lambda2)."""
    N, M = 9, 7
    lam1, lam2 = 0.6, 0.8
    a, b, c, d = _rand(1, N), _rand(2, N), _rand(3, M), _rand(4, M)
    phi = np.outer(c, a).reshape(-1)      # column-major: phi[i1 + N i2] = a[i1] c[i2]
    psi = np.outer(d, b).reshape(-1)
    J = grid2d.ftvp_2d(phi, psi, lam1, lam2, N, M)
    want = np.outer(paper3.ftvp1(c, d, lam2), paper3.ftvp1(a, b, lam1)).reshape(-1)
    np.testing.assert_allclose(J, want, rtol=1e-13)


def test_ftvp_2d_lambda2_zero_reduces_to_columnwise_1d():
    """lambda2 -> 0 (0^0 = 1): only same-column tuples survive, J_{k2} = FTVP-1(phi_{k2}, psi_{k2})."""
    N, M = 6, 5
    phi, psi = _rand(5, N * M), _rand(6, N * M)
    J = grid2d.ftvp_2d(phi, psi, 0.7, 0.0, N, M).reshape(M, N)
    for c in range(M):
        np.testing.assert_allclose(J[c], paper3.ftvp1(phi.reshape(M, N)[c], psi.reshape(M, N)[c], 0.7), rtol=1e-14)


def test_transpose_symmetry():
    """Swapping the roles of rows and columns (and h1, h2) transposes J."""
    N, M, eps = 6, 4, 0.2
    h1, h2 = 0.2, 0.3
    phis = [_rand(20 + q, N * M) for q in range(3)]
    J = grid2d.product(phis, 2, N, M, h1, h2, eps)
    tr = [grid2d._transpose(p, N, M) for p in phis]
    Jt = grid2d.product(tr, 2, M, N, h2, h1, eps)
    np.testing.assert_allclose(grid2d._transpose(J, N, M), Jt, rtol=1e-13)


@pytest.mark.parametrize("N,M", [(3, 4), (5, 5), (6, 2), (2, 3)])
@pytest.mark.parametrize("eps", [0.15, 0.02])
def test_cost_2d_equals_plan_cost(N, M, eps):
    h1, h2 = 1.0 / (N - 1), 0.5 / (M - 1)
    phis = [_rand(30 + q + N, N * M) for q in range(3)]
    np.testing.assert_allclose(grid2d.cost_2d(phis, N, M, h1, h2, eps),
                               grid2d.dense_cost(phis, N, M, h1, h2, eps), rtol=1e-12)


def test_sinkhorn_2d_marginals():
    """After the sweep's last update the third marginal is exact; the plan has unit mass."""
    N, M, eps = 5, 4, 0.2
    rng = np.random.default_rng(3)
    mus = rng.uniform(0.1, 1, (3, N * M))
    mus /= mus.sum(axis=1, keepdims=True)
    phis = grid2d.sinkhorn_2d(mus, N, M, 0.25, 1.0 / 3, eps, 5)
    m = grid2d.marginals(phis, N, M, 0.25, 1.0 / 3, eps)
    np.testing.assert_allclose(m[2], mus[2], rtol=1e-13)
    assert abs(m[0].sum() - 1.0) < 1e-13


def test_algorithm3_cancels_for_small_lambda():
    """Why cost_2d does not use Algorithm 3 inside Algorithm 6: FTVP-2 builds the E-weights from
    absolute index sums, so its relative error grows like lambda^-2 (A21)."""
    from oracle import dense
    N = 3
    rng = np.random.default_rng(1)
    a, b = rng.uniform(0.1, 1, N), rng.uniform(0.1, 1, N)
    for lam, bad in ((0.5, False), (math.exp(-50), True)):
        K = dense.kernel_tensor_lambda(3, N, lam)
        E = dense.exponent_tensor(3, N)
        want = dense.contract(E * K, [a, b, np.ones(N)], 2)
        err = np.max(np.abs(paper3.ftvp2(a, b, lam, 1.0) - want) / want)
        assert (err > 1e-3) == bad, (lam, err)
        np.testing.assert_allclose(grid2d._cost_inner(1.0)(a, b, lam), want, rtol=1e-13)
