"""Pins of O2 (oracle/paper3.py: Algorithms 2, 3, 5, 4 for l=3) against the dense definitions."""
import json
import math
import os

import numpy as np
import pytest

from oracle import dense, paper3

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _dense_J(ph, ps, lam):
    N = len(ph)
    K = dense.kernel_tensor_lambda(3, N, lam)
    return dense.contract(K, [ph, ps, None], 2)


@pytest.mark.parametrize("lam", [0.1, 0.5, 0.9])
def test_ftvp1_equals_dense(lam):
    """N <= 30, lambda in {0.1,0.5,0.9}, seeded random pairs: rel err <= 1e-10."""
    for seed in range(8):
        rng = np.random.default_rng(seed)
        N = int(rng.integers(1, 31))
        ph, ps = rng.uniform(0.1, 1, N), rng.uniform(0.1, 1, N)
        J = paper3.ftvp1(ph, ps, lam)
        np.testing.assert_allclose(J, _dense_J(ph, ps, lam), rtol=1e-12)


def test_ftvp1_regions_match_restricted_sums():
    """each J_{k,p} equals the dense sum restricted to D_p."""
    rng = np.random.default_rng(11)
    N, lam = 7, 0.6
    ph, ps = rng.uniform(0.1, 1, N), rng.uniform(0.1, 1, N)
    _, parts, _ = paper3.ftvp1(ph, ps, lam, return_parts=True)
    t = GOLD["coefficient_table"]
    inside = [
        lambda i, j, k: i <= j <= k, lambda i, j, k: j < i <= k, lambda i, j, k: i <= k < j,
        lambda i, j, k: j <= k < i, lambda i, j, k: k < i <= j, lambda i, j, k: k < j < i,
    ]
    for p in range(6):
        want = np.zeros(N)
        for i in range(1, N + 1):
            for j in range(1, N + 1):
                for k in range(1, N + 1):
                    if inside[p](i, j, k):
                        want[k - 1] += ph[i - 1] * ps[j - 1] * lam ** (t["a"][p] * i + t["b"][p] * j + t["c"][p] * k)
        np.testing.assert_allclose(parts[p], want, rtol=1e-12, atol=1e-300)


def test_ftvp1_closed_forms():
    rng = np.random.default_rng(5)
    ph, ps = rng.uniform(0.1, 1, 9), rng.uniform(0.1, 1, 9)
    np.testing.assert_allclose(paper3.ftvp1(ph, ps, 1.0), ph.sum() * ps.sum(), rtol=1e-14)
    assert paper3.ftvp1(ph[:1], ps[:1], 0.4)[0] == pytest.approx(ph[0] * ps[0], rel=1e-15)
    # argument symmetry and linearity
    np.testing.assert_allclose(paper3.ftvp1(ph, ps, 0.7), paper3.ftvp1(ps, ph, 0.7), rtol=1e-13)
    np.testing.assert_allclose(paper3.ftvp1(3.0 * ph, ps, 0.7), 3.0 * paper3.ftvp1(ph, ps, 0.7), rtol=1e-14)


def test_ftvp2_spec_example():
    ex = GOLD["ftvp2"][0]
    out = paper3.ftvp2(np.array(ex["phi"], float), np.array(ex["psi"], float), ex["lambda"], ex["h"])
    np.testing.assert_allclose(out, ex["value"], rtol=1e-15)


@pytest.mark.parametrize("lam", [0.2, 0.6, 0.95])
def test_ftvp2_equals_dense_cost_product(lam):
    for seed in range(5):
        rng = np.random.default_rng(100 + seed)
        N = int(rng.integers(2, 20))
        h = 0.1
        ph, ps = rng.uniform(0.1, 1, N), rng.uniform(0.1, 1, N)
        E = dense.exponent_tensor(3, N).astype(float)
        CK = h * E * np.power(lam, E)
        want = dense.contract(CK, [ph, ps, None], 2)
        np.testing.assert_allclose(paper3.ftvp2(ph, ps, lam, h), want, rtol=1e-12, atol=1e-300)


def test_ftvp2_printed_init_is_wrong():
    """DESIGN.md A11: R_{N,5}, R_{N,6} printed without the factor N give wrong results."""
    rng = np.random.default_rng(7)
    N, lam, h = 6, 0.6, 0.2
    ph, ps = rng.uniform(0.1, 1, N), rng.uniform(0.1, 1, N)
    E = dense.exponent_tensor(3, N).astype(float)
    want = dense.contract(h * E * np.power(lam, E), [ph, ps, None], 2)
    bad = paper3.ftvp2(ph, ps, lam, h, paper_typos=True)
    assert np.max(np.abs(bad - want) / want) > 1e-3


def _rescaled_dense(ph, ps, al, be, ga, lam, eps):
    N = len(ph)
    K = dense.kernel_tensor_lambda(3, N, lam)
    K = K * np.exp((al[:, None, None] + be[None, :, None] + ga[None, None, :]) / eps)
    return dense.contract(K, [ph, ps, None], 2)


def test_ftvp_log_equals_rescaled_dense():
    for seed in range(6):
        rng = np.random.default_rng(200 + seed)
        N = int(rng.integers(1, 16))
        lam, eps = 0.7, 0.1
        ph, ps = rng.uniform(0.1, 1, N), rng.uniform(0.1, 1, N)
        al, be, ga = (rng.normal(0, 0.05, N) for _ in range(3))
        out = paper3.ftvp_log(ph, ps, al, be, ga, lam, eps)
        np.testing.assert_allclose(out, _rescaled_dense(ph, ps, al, be, ga, lam, eps), rtol=1e-12)
        # zero potentials reduce to FTVP-1
        z = np.zeros(N)
        np.testing.assert_allclose(paper3.ftvp_log(ph, ps, z, z, z, lam, eps), paper3.ftvp1(ph, ps, lam), rtol=1e-14)


def test_ftvp_log_printed_lines_are_wrong():
    rng = np.random.default_rng(9)
    N, lam, eps = 8, 0.7, 0.1
    ph, ps = rng.uniform(0.1, 1, N), rng.uniform(0.1, 1, N)
    al, be, ga = (rng.normal(0, 0.05, N) for _ in range(3))
    want = _rescaled_dense(ph, ps, al, be, ga, lam, eps)
    bad = paper3.ftvp_log(ph, ps, al, be, ga, lam, eps, paper_typos=True)
    assert np.max(np.abs(bad - want) / want) > 1e-3


def test_algorithm4_lockstep_with_dense_sinkhorn():
    """Table 1: fast and dense Sinkhorn plans agree to ~1e-16 (here: 1e-15 Frobenius)."""
    rng = np.random.default_rng(21)
    N, l = 8, 3
    h = 1.0 / (N - 1)
    eps = 0.1
    mus = rng.uniform(0, 1, (l, N))
    mus /= mus.sum(axis=1, keepdims=True)
    phi, psi, vphi, t, res, W = paper3.fast_sinkhorn_3(mus[0], mus[1], mus[2], h, eps, 100, -1.0)
    phis_d, _, _ = dense.sinkhorn(mus, h, eps, 100)
    K = dense.kernel_tensor(l, N, h, eps)
    Pf = dense.plan(K, [phi, psi, vphi])
    Pd = dense.plan(K, list(phis_d))
    assert np.linalg.norm(Pf - Pd) <= GOLD["plan_difference_bound"]["max_frobenius"]
    C = dense.cost_tensor(l, N, h)
    assert W == pytest.approx(dense.distance(C, K, [phi, psi, vphi]), rel=1e-12)
    _, _, _, _, _, W2 = paper3.fast_sinkhorn_3(mus[0], mus[1], mus[2], h, eps, 100, -1.0, paper_double_h=True)
    assert W2 == pytest.approx(W * h, rel=1e-14)   # P:652 as printed is off by a factor h (A8)
