"""Pins of O1 (oracle/dense.py) against values and closed forms fixed by the paper / mathematics."""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy.signal import lfilter

from oracle import dense

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", GOLD["cost_entries"])
def test_cost_entries_spec(ex):
    C = dense.cost_tensor(ex["l"], ex["N"], ex["h"])
    idx = tuple(i - 1 for i in ex["index_1based"])
    assert C[idx] == pytest.approx(ex["value"], abs=1e-15)


def test_lambda_spec():
    ex = GOLD["lambda"][0]
    K = dense.kernel_tensor(2, 2, ex["h"], ex["eps"])
    assert K[0, 1] == pytest.approx(math.exp(ex["value_exponent"]), rel=1e-15)


def test_coefficient_table_regions():
    """inside D_p the exponent |i-j|+|i-k|+|j-k| equals a_p i + b_p j + c_p k."""
    t = GOLD["coefficient_table"]
    N = 5
    regions = [
        lambda i, j, k: i <= j <= k, lambda i, j, k: j < i <= k, lambda i, j, k: i <= k < j,
        lambda i, j, k: j <= k < i, lambda i, j, k: k < i <= j, lambda i, j, k: k < j < i,
    ]
    E = dense.exponent_tensor(3, N)
    count = np.zeros((N, N, N), dtype=int)
    for p, inside in enumerate(regions):
        for i, j, k in itertools.product(range(1, N + 1), repeat=3):
            if inside(i, j, k):
                count[i - 1, j - 1, k - 1] += 1
                assert E[i - 1, j - 1, k - 1] == t["a"][p] * i + t["b"][p] * j + t["c"][p] * k
    assert np.all(count == 1)  # D_1..D_6 partition the index set


def test_kernel_symmetry_and_diagonal():
    for l in (2, 3, 4):
        K = dense.kernel_tensor(l, 4, 0.25, 0.3)
        for perm in itertools.permutations(range(l)):
            assert np.array_equal(K, np.transpose(K, perm))
        for i in range(4):
            assert K[(i,) * l] == 1.0


def test_contract_vs_tuple_loop():
    rng = np.random.default_rng(1)
    for l in (2, 3, 4):
        N = 4
        K = dense.kernel_tensor(l, N, 0.3, 0.5)
        ph = [rng.uniform(0.1, 1, N) for _ in range(l)]
        for k in range(l):
            np.testing.assert_allclose(dense.contract(K, ph, k), dense.contract_loops(K, ph, k), rtol=1e-14)


def test_closed_forms_lambda_limits():
    rng = np.random.default_rng(2)
    for l in (2, 3, 4):
        N = 5
        ph = [rng.uniform(0.1, 1, N) for _ in range(l)]
        K1 = dense.kernel_tensor_lambda(l, N, 1.0)
        K0 = dense.kernel_tensor_lambda(l, N, 0.0)
        for k in range(l):
            prod_sum = np.prod([ph[q].sum() for q in range(l) if q != k])
            np.testing.assert_allclose(dense.contract(K1, ph, k), prod_sum, rtol=1e-14)
            diag = np.prod([ph[q] for q in range(l) if q != k], axis=0)
            np.testing.assert_allclose(dense.contract(K0, ph, k), diag, rtol=1e-14)


def test_closed_form_N2():
    """N=2: J_k[0] = sum_{T subset B} lambda^{|T|(l-|T|)} prod_{T} phi[1] prod_{B\\T} phi[0]."""
    rng = np.random.default_rng(3)
    lam = 0.37
    for l in (2, 3, 4, 5):
        ph = [rng.uniform(0.1, 1, 2) for _ in range(l)]
        K = dense.kernel_tensor_lambda(l, 2, lam)
        for k in range(l):
            B = [q for q in range(l) if q != k]
            want = 0.0
            for r in range(len(B) + 1):
                for T in itertools.combinations(B, r):
                    term = lam ** (r * (l - r))
                    for q in B:
                        term *= ph[q][1] if q in T else ph[q][0]
                    want += term
            assert dense.contract(K, ph, k)[0] == pytest.approx(want, rel=1e-14)
        ones = [np.ones(2)] * l
        want1 = sum(math.comb(l - 1, j) * lam ** (j * (l - j)) for j in range(l))
        assert dense.contract(K, ones, 0)[0] == pytest.approx(want1, rel=1e-14)


def test_l2_is_two_sided_exponential_smoothing():
    """l=2: J[m] = sum_j lambda^{|m-j|} phi[j] = forward IIR + backward IIR - diagonal (textbook filter)."""
    rng = np.random.default_rng(4)
    N, lam = 40, 0.83
    phi = rng.uniform(0.1, 1, N)
    K = dense.kernel_tensor_lambda(2, N, lam)
    fwd = lfilter([1.0], [1.0, -lam], phi)
    bwd = lfilter([1.0], [1.0, -lam], phi[::-1])[::-1]
    np.testing.assert_allclose(dense.contract(K, [None, phi], 0), fwd + bwd - phi, rtol=1e-13)


def test_dense_sinkhorn_point_mass():
    """all mass at one point -> plan concentrated there, distance 0."""
    N, l = 4, 3
    mus = np.zeros((l, N))
    mus[:, 1] = 1.0
    phis, t, res = dense.sinkhorn(mus, 1.0 / 3, 0.1, 50, tol=1e-13)
    K = dense.kernel_tensor(l, N, 1.0 / 3, 0.1)
    T = dense.plan(K, phis)
    assert T[1, 1, 1] == pytest.approx(1.0, abs=1e-12)
    assert dense.distance(dense.cost_tensor(l, N, 1.0 / 3), K, phis) == pytest.approx(0.0, abs=1e-12)
