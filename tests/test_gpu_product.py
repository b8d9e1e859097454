"""GPU parity of a single tensor-vector product (mmot_marginal) and of the cost (mmot_cost)
against the fp64 CPU oracle (oracle/regions.c, §4.2 region chains), elementwise.

Tolerance (north_star, fp64): max elementwise relative error <= 1e-10.  All terms of J_k are
positive, so the elementwise relative error is well defined; the fp64 scans re-associate a
positive sum, whose rounding error is bounded by ~(scan depth) * 2^-53.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import regions  # noqa: E402

DEV = "cuda:0"
RTOL = 1e-10


def _to_dev(vs):
    return [torch.from_numpy(np.ascontiguousarray(v)).to(DEV) for v in vs]


def _gpu_marginals(l, N, eta, phis, chunk=0, repr_="linear"):
    ctx = mm.Context(l, N, eta, repr=repr_, chunk=chunk)
    u = _to_dev(phis if repr_ == "linear" else [np.log(p) for p in phis])
    out = [ctx.marginal(k, u).cpu().numpy() for k in range(l)]
    ctx.close()
    return out


def _oracle_marginals(phis, h, eta):
    l = len(phis)
    w = regions.edge_weights(l, h, eta)
    return [phis[k] * regions.marginal_product(list(phis), k, w) for k in range(l)]


def _rel(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


# grid sizes spanning one point, ragged tails, chunk and sub-block boundaries, many chunks
SIZES = [1, 2, 3, 5, 8, 9, 31, 32, 33, 127, 128, 129, 255, 257, 1000, 4097]


@pytest.mark.parametrize("l", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("N", SIZES)
def test_marginal_parity_sizes(l, N):
    if l == 6 and N > 1000:
        pytest.skip("oracle cost")
    phis = mmot_inputs.random_positive(1000 * l + N, l, N)
    h = mmot_inputs.grid_h(N)
    eta = 0.05
    got = _gpu_marginals(l, N, eta, phis)
    want = _oracle_marginals(phis, h, eta)
    for k in range(l):
        assert _rel(got[k], want[k]) <= RTOL, (l, N, k)


@pytest.mark.parametrize("l", [3, 4, 5])
@pytest.mark.parametrize("chunk", [1, 2, 4, 7, 16])
def test_marginal_parity_small_chunks_many_levels(l, chunk):
    """Small chunks force thousands of chunks and 3-4 levels of the operator scan."""
    N = 6000 if l < 5 else 2000
    phis = mmot_inputs.random_positive(77 + l + chunk, l, N)
    h = mmot_inputs.grid_h(N)
    eta = 0.02
    got = _gpu_marginals(l, N, eta, phis, chunk=chunk)
    want = _oracle_marginals(phis, h, eta)
    for k in range(l):
        assert _rel(got[k], want[k]) <= RTOL, (l, chunk, k)


@pytest.mark.parametrize("hoe", [1e-6, 1e-3, 0.3, 3.0, 30.0])
def test_marginal_parity_lambda_range(hoe):
    """lambda = e^{-h/eta} from 1-1e-6 (near-constant kernel) to e^{-30} (near-diagonal)."""
    l, N = 4, 700
    h = mmot_inputs.grid_h(N)
    eta = h / hoe
    phis = mmot_inputs.random_positive(5, l, N)
    got = _gpu_marginals(l, N, eta, phis)
    want = _oracle_marginals(phis, h, eta)
    for k in range(l):
        assert _rel(got[k], want[k]) <= RTOL


def test_log_and_linear_repr_agree():
    l, N, eta = 4, 3000, 0.01
    phis = mmot_inputs.random_positive(9, l, N)
    a = _gpu_marginals(l, N, eta, phis, repr_="linear")
    b = _gpu_marginals(l, N, eta, phis, repr_="log")
    for k in range(l):
        assert _rel(b[k], a[k]) <= 1e-13


def test_reversal_equivariance_on_gpu():
    """Reverse every input -> reversed output; exercises prefix vs suffix carries (the chunking is not
    reversal symmetric)."""
    l, N, eta = 4, 5003, 0.003
    phis = mmot_inputs.random_positive(10, l, N)
    a = _gpu_marginals(l, N, eta, phis, chunk=5)
    b = _gpu_marginals(l, N, eta, [p[::-1].copy() for p in phis], chunk=5)
    for k in range(l):
        assert _rel(b[k][::-1], a[k]) <= RTOL


def test_mass_identity_on_gpu():
    """<phi_k, J_k> = sum_m m_k[m] is the plan mass for every k."""
    l, N, eta = 5, 2048, 0.01
    phis = mmot_inputs.random_positive(11, l, N)
    got = _gpu_marginals(l, N, eta, phis)
    masses = [g.sum() for g in got]
    np.testing.assert_allclose(masses, masses[0], rtol=1e-12)


@pytest.mark.parametrize("l", [2, 3, 4, 5, 6])
def test_cost_parity(l):
    N = {2: 3000, 3: 2000, 4: 1500, 5: 600, 6: 200}[l]
    eta = 0.02
    h = mmot_inputs.grid_h(N)
    phis = mmot_inputs.random_positive(300 + l, l, N)
    ctx = mm.Context(l, N, eta, repr="linear")
    W = ctx.cost(_to_dev(phis))
    ctx.close()
    w = regions.edge_weights(l, h, eta)
    _, jh = regions.marginal_product(list(phis), l - 1, w, want_hat=True)
    W_ref = h * float(np.dot(phis[l - 1], jh))
    assert abs(W - W_ref) <= RTOL * abs(W_ref)


@pytest.mark.slow
def test_marginal_parity_c4_full_size():
    """C4 shape (l=4, N=1e8, eta=1e-4) in the bench's launch configuration, whole vector."""
    cfg = mmot_inputs.CONFIGS["C4"]
    l, N, eta = cfg.l, cfg.N, cfg.eta
    h = mmot_inputs.grid_h(N)
    mus = mmot_inputs.make_marginals("C4", 0)
    phis = mus * N  # a positive, smooth scaling field of the config's shape
    ctx = mm.Context(l, N, eta, repr="linear")
    u = _to_dev(phis)
    out = ctx.marginal(1, u).cpu().numpy()
    ctx.close()
    del u
    w = regions.edge_weights(l, h, eta)
    want = phis[1] * regions.marginal_product(list(phis), 1, w)
    assert _rel(out, want) <= RTOL
