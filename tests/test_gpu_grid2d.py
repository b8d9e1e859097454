"""2-D grids (NEXT-2; §4.1): mmot_create_2d's products, cost and Sinkhorn against
the fp64 oracle O6 (oracle/grid2d.py: Algorithm 6 step by step with Algorithm 2 inside, pinned
against the product written out).  Tolerance 1e-10 (north_star fp64)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import grid2d  # noqa: E402

DEV = "cuda:0"
RTOL = 1e-10


def _dev(vs):
    return [torch.from_numpy(np.ascontiguousarray(v)).to(DEV) for v in vs]


def _h(n, lo, hi):
    return (hi - lo) / (n - 1) if n > 1 else 1.0


@pytest.mark.parametrize("N1,N2", [(1, 1), (1, 7), (9, 1), (2, 3), (16, 16), (33, 20), (64, 48), (128, 96)])
@pytest.mark.parametrize("eps", [0.1, 0.02])
def test_grid2d_marginals_and_cost(N1, N2, eps):
    g = (0.0, 1.0, 0.0, 0.7)
    h1, h2 = _h(N1, 0.0, 1.0), _h(N2, 0.0, 0.7)
    rng = np.random.default_rng(N1 * 100 + N2)
    phis = rng.uniform(0.1, 1.0, (3, N1 * N2))
    ctx = mm.Context(3, N1 * N2, eps, repr="linear", shape2d=(N1, N2), grid=g)
    assert ctx.info["kernel"] == "grid2d"
    u = _dev(phis)
    for k in range(3):
        got = ctx.marginal(k, u).cpu().numpy()
        want = phis[k] * grid2d.product(list(phis), k, N1, N2, h1, h2, eps)
        assert np.max(np.abs(got - want) / want) <= RTOL, (N1, N2, k)
    W = ctx.cost(u)
    ctx.close()
    W_ref = grid2d.cost_2d(list(phis), N1, N2, h1, h2, eps)
    assert abs(W - W_ref) <= RTOL * abs(W_ref) + 1e-300, (W, W_ref)
    if (N1 * N2) ** 3 <= 2e8:
        assert abs(W - grid2d.dense_cost(list(phis), N1, N2, h1, h2, eps)) <= 1e-10 * abs(W_ref) + 1e-300


@pytest.mark.parametrize("N1,N2,T", [(8, 6, 10), (32, 32, 5)])
def test_grid2d_sinkhorn_lockstep(N1, N2, T):
    eps = 0.05
    h1, h2 = _h(N1, 0, 1), _h(N2, 0, 1)
    rng = np.random.default_rng(7 + N1)
    x, y = np.meshgrid(np.arange(N1) / max(N1 - 1, 1), np.arange(N2) / max(N2 - 1, 1), indexing="ij")
    mus = []
    for q in range(3):   # Gaussian bumps on the mesh (column-major flattening)
        cx, cy, sd = rng.uniform(0.2, 0.8), rng.uniform(0.2, 0.8), rng.uniform(0.1, 0.2)
        m = np.exp(-((x - cx) ** 2 + (y - cy) ** 2) / (2 * sd * sd)) + 1e-6
        mus.append((m / m.sum()).T.reshape(-1))
    mus = np.stack(mus)
    ctx = mm.Context(3, N1 * N2, eps, repr="log", shape2d=(N1, N2), check_every=1)
    u = [torch.empty(N1 * N2, dtype=torch.float64, device=DEV) for _ in range(3)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev(mus), T, 1e-300, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    marg = [ctx.marginal(k, u).cpu().numpy() for k in range(3)]
    g = np.stack([v.cpu().numpy() for v in u])
    W = ctx.cost(u)
    ctx.close()
    phis = grid2d.sinkhorn_2d(mus, N1, N2, h1, h2, eps, T)
    assert np.max(np.abs(g - np.log(phis))) <= 1e-9
    m_ref = grid2d.marginals(phis, N1, N2, h1, h2, eps)
    for k in range(3):
        assert np.abs(marg[k] - m_ref[k]).sum() / np.abs(m_ref[k]).sum() <= RTOL, k
    res_ref = sum(np.abs(m_ref[k] - mus[k]).sum() for k in range(2))
    assert rep["residual"] == pytest.approx(res_ref, rel=1e-8)
    W_ref = grid2d.cost_2d(list(phis), N1, N2, h1, h2, eps)
    assert abs(W - W_ref) <= RTOL * abs(W_ref)


def test_grid2d_argument_errors():
    with pytest.raises(mm.MMOTError) as e:
        mm.Context(4, 16, 0.1, shape2d=(4, 4))
    assert e.value.name == "MMOT_EUNSUPPORTED"
    with pytest.raises(mm.MMOTError) as e:
        mm.Context(3, 15, 0.1, shape2d=(4, 4))
    assert e.value.name == "MMOT_ESHAPE"
