"""Pins of the Sinkhorn driver (oracle/sinkhorn.py) and W_0 (oracle/comonotone.py)."""
import itertools
import math

import numpy as np
import pytest
from scipy.optimize import linprog

import mmot_inputs
from oracle import comonotone, dense, sinkhorn


def _mus(seed, l, N):
    rng = np.random.default_rng(seed)
    m = rng.uniform(0, 1, (l, N))
    return m / m.sum(axis=1, keepdims=True)


@pytest.mark.parametrize("l,N", [(3, 6), (4, 5)])
def test_fast_vs_dense_lockstep(l, N):
    """SURVEY [verified]: dense and fast Sinkhorn agree in lockstep (Table 1 magnitudes)."""
    mus = _mus(l * 10 + N, l, N)
    h, eta = 1.0 / (N - 1), 0.2
    for T in (1, 3, 40):
        pf, _, _ = sinkhorn.sinkhorn(mus, h, eta, T)
        pd, _, _ = dense.sinkhorn(mus, h, eta, T)
        np.testing.assert_allclose(pf, pd, rtol=1e-12)
        K = dense.kernel_tensor(l, N, h, eta)
        assert np.linalg.norm(dense.plan(K, list(pf)) - dense.plan(K, list(pd))) < 1e-15


def test_marginal_satisfied_after_update_and_unit_mass():
    l, N = 4, 40
    mus = _mus(3, l, N)
    h, eta = 1.0 / (N - 1), 0.05
    seen = []

    def rec(t, phis):
        seen.append(phis)

    sinkhorn.sinkhorn(mus, h, eta, 3, record=rec)
    phis = seen[-1]
    m = sinkhorn.marginals(phis, h, eta)
    np.testing.assert_allclose(m[l - 1], mus[l - 1], rtol=1e-12)  # last update exact
    np.testing.assert_allclose(m.sum(axis=1), 1.0, rtol=1e-12)      # plan mass 1 after an update


def test_init_constant_invariance():
    """DESIGN.md A5: marginals and W do not depend on the init constant (gauge only)."""
    l, N = 3, 25
    mus = _mus(8, l, N)
    h, eta = 1.0 / (N - 1), 0.1
    p1, _, _ = sinkhorn.sinkhorn(mus, h, eta, 7)
    p2, _, _ = sinkhorn.sinkhorn(mus, h, eta, 7, phis0=np.full((l, N), 3.7))
    np.testing.assert_allclose(sinkhorn.marginals(p1, h, eta), sinkhorn.marginals(p2, h, eta), rtol=1e-12)
    assert sinkhorn.cost(p1, h, eta) == pytest.approx(sinkhorn.cost(p2, h, eta), rel=1e-12)


def test_cost_three_ways():
    """W = <C, T> (dense) = h <phi_l, hatJ_l> (regions tangent) = h dZ/dlog(lambda) (difference)."""
    l, N = 4, 6
    mus = _mus(12, l, N)
    h, eta = 1.0 / (N - 1), 0.3
    phis, _, _ = sinkhorn.sinkhorn(mus, h, eta, 20)
    K = dense.kernel_tensor(l, N, h, eta)
    Wd = dense.distance(dense.cost_tensor(l, N, h), K, list(phis))
    for k in range(l):
        assert sinkhorn.cost(phis, h, eta, k) == pytest.approx(Wd, rel=1e-13)
    d = 1e-5
    Zp = np.dot(phis[0], sinkhorn.product(phis, 0, h, eta * (1 - d)))  # lambda^(1/(1-d))
    Zm = np.dot(phis[0], sinkhorn.product(phis, 0, h, eta * (1 + d)))

    # log lambda = -h/eta ; eta(1-d) -> log lambda (1/(1-d)); central difference in log lambda
    llp = -h / (eta * (1 - d))
    llm = -h / (eta * (1 + d))
    assert h * (Zp - Zm) / (llp - llm) == pytest.approx(Wd, rel=1e-7)


def test_log_and_plain_drivers_agree():
    mus = mmot_inputs.c1_marginals(0, N=64)
    h = mmot_inputs.grid_h(64)
    pp, _, _ = sinkhorn.sinkhorn(mus, h, 0.05, 30)
    gl, _, _ = sinkhorn.sinkhorn(mus, h, 0.05, 30, domain="log")
    np.testing.assert_allclose(np.exp(gl), pp, rtol=1e-11)


def test_w0_matches_lp():
    """Comonotone W_0 equals the LP optimum on tiny instances."""
    for seed in range(3):
        l, N = 3, 4
        mus = _mus(40 + seed, l, N)
        h = 1.0 / (N - 1)
        C = dense.cost_tensor(l, N, h).ravel()
        A, b = [], []
        idx = list(itertools.product(range(N), repeat=l))
        for q in range(l):
            for m in range(N):
                A.append([1.0 if t[q] == m else 0.0 for t in idx])
                b.append(mus[q][m])
        lp = linprog(C, A_eq=np.array(A), b_eq=np.array(b), bounds=(0, None), method="highs")
        assert comonotone.w0(mus, h) == pytest.approx(lp.fun, abs=1e-10)


def test_entropic_cost_above_w0_and_converges():
    l, N = 4, 30
    mus = _mus(5, l, N)
    h = 1.0 / (N - 1)
    W0 = comonotone.w0(mus, h)
    prev = None
    for eta in (0.5, 0.2, 0.1, 0.05):
        phis, t, res = sinkhorn.sinkhorn(mus, h, eta, 5000, tol=1e-11, domain="plain")
        assert res <= 1e-11
        W = sinkhorn.cost(phis, h, eta)
        assert W >= W0 - 1e-12
        if prev is not None:
            assert W - W0 < prev - W0 + 1e-12     # W_eta -> W_0 as eta -> 0 (trend)
        prev = W


def test_tol_stop_rule():
    """stop at the first t with Res <= tol."""
    l, N = 3, 20
    mus = _mus(6, l, N)
    h, eta = 1.0 / (N - 1), 0.2
    trace = []
    phis, t, res = sinkhorn.sinkhorn(mus, h, eta, 500, tol=1e-9)
    assert res <= 1e-9
    _, t2, res2 = sinkhorn.sinkhorn(mus, h, eta, t - 1, tol=1e-9)
    assert res2 > 1e-9


@pytest.mark.parametrize("eps", [0.5, 0.1, 0.03])
def test_residual_pinned_to_algorithm4_line7(eps):
    """The residual (oracle/sinkhorn.residual) equals, sweep by sweep, the literal Algorithm 4
    line 7: Res = ||phi (.) FTVP-1(psi, varphi) - u||_1 + ||psi (.) FTVP-1(phi, varphi) - v||_1,
    with Algorithm 2's FTVP-1 computing the products -- an independent evaluation of the
    same l = 3 quantity (A6: the sum over k < l of the L1 marginal violations)."""
    from oracle import paper3
    N = 14
    h = 1.0 / (N - 1)
    u, v, w = _mus(700 + int(100 * eps), 3, N)
    mus = np.stack([u, v, w])
    for T in (1, 2, 3, 7):
        _, _, _, t, res_paper, _ = paper3.fast_sinkhorn_3(u, v, w, h, eps, T, 0.0)
        assert t == T
        phis, t2, res = sinkhorn.sinkhorn(mus, h, eps, T, tol=1e-300)
        assert t2 == T
        assert res == pytest.approx(res_paper, rel=1e-12, abs=1e-17), (T, res, res_paper)
        assert sinkhorn.residual(phis, mus, h, eps) == pytest.approx(res_paper, rel=1e-12, abs=1e-17)


@pytest.mark.parametrize("l", [3, 4])
def test_residual_pinned_to_plan_marginals(l):
    """The residual equals the L1 violation of the marginals of the explicit plan tensor
    T = K (.) (phi_1 x ... x phi_l), summed over k < l (Algorithm 1 line 7, P:168,
    generalised), with the plan built by an outer product and summed over all axes but k -- not by a
    tensor-vector product.  The l-th term vanishes after the sweep's last update."""
    N = 5
    h, eta = 1.0 / (N - 1), 0.15
    mus = _mus(800 + l, l, N)
    K = dense.kernel_tensor(l, N, h, eta)
    for T in (1, 2, 5):
        phis, _, res = sinkhorn.sinkhorn(mus, h, eta, T, tol=1e-300)
        outer = phis[0]
        for q in range(1, l):
            outer = np.multiply.outer(outer, phis[q])
        plan = K * outer
        viol = [np.abs(plan.sum(axis=tuple(a for a in range(l) if a != k)) - mus[k]).sum() for k in range(l)]
        assert res == pytest.approx(sum(viol[:-1]), rel=1e-11, abs=1e-17), T
        assert viol[-1] < 1e-15
        # the dense driver's stop rule sees the same residual: same stop sweep for a tolerance
        tol = 0.5 * res
        _, t_fast, _ = sinkhorn.sinkhorn(mus, h, eta, 200, tol=tol)
        _, t_dense, _ = dense.sinkhorn(mus, h, eta, 200, tol=tol)
        assert t_fast == t_dense
