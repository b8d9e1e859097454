"""GPU parity on non-uniform 1-D grids (mmot_create_points / _batched_points; paper footnote P:182,
SURVEY §8(f) NEXT-3) against the fp64 oracle oracle/points.py (pinned in test_oracle_points.py).
Tolerance: north_star fp64, 1e-10 relative."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import points  # noqa: E402

DEV = "cuda:0"
RTOL = 1e-10


def _grid(seed, N, lo=1.0, hi=4.0):
    rng = np.random.default_rng(seed)
    h = rng.uniform(lo, hi, N - 1)
    x = np.concatenate([[0.0], np.cumsum(h)])
    return x / x[-1]


def _dev(vs):
    return [torch.from_numpy(np.ascontiguousarray(v)).to(DEV) for v in vs]


@pytest.mark.parametrize("l,N", [(2, 333), (3, 257), (4, 300), (5, 129), (4, 5000)])
def test_points_marginals_and_cost(l, N):
    x = _grid(100 + l, N)
    eta = 0.02
    phis = list(mmot_inputs.random_positive(200 + l, l, N))
    ctx = mm.Context(l, N, eta, repr="linear", points=x)
    assert ctx.info["kernel"] == ("persistent" if N <= 4096 else "two_walk")
    u = _dev(phis)
    for k in range(l):
        got = ctx.marginal(k, u).cpu().numpy()
        want = phis[k] * points.product(phis, x, eta, k)
        assert np.max(np.abs(got - want) / want) <= RTOL, k
    W = ctx.cost(u)
    ctx.close()
    assert abs(W - points.cost(phis, x, eta)) <= RTOL * abs(W)


def test_points_wide_spacing_ratio():
    """Spacings over three decades (a refined patch inside a coarse grid)."""
    l, N, eta = 3, 400, 0.01
    h = np.where(np.arange(N - 1) % 100 < 50, 1e-3, 1.0)
    x = np.concatenate([[0.0], np.cumsum(h)])
    x /= x[-1]
    phis = list(mmot_inputs.random_positive(7, l, N))
    ctx = mm.Context(l, N, eta, repr="linear", points=x)
    u = _dev(phis)
    for k in range(l):
        got = ctx.marginal(k, u).cpu().numpy()
        want = phis[k] * points.product(phis, x, eta, k)
        assert np.max(np.abs(got - want) / want) <= RTOL, k
    ctx.close()


@pytest.mark.parametrize("l", [3, 4])
def test_points_sinkhorn_lockstep(l):
    N, eta, T = 240, 0.03, 5
    x = _grid(300 + l, N)
    mus = np.stack(mmot_inputs.random_marginals(400 + l, l, N))
    ctx = mm.Context(l, N, eta, repr="log", points=x)
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev(mus), T, 0.0, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    g = np.stack([v.cpu().numpy() for v in u])
    ctx.close()
    ref = points.sinkhorn(mus, x, eta, T)
    assert np.max(np.abs(g - np.log(ref))) <= 1e-9


def test_points_batched_per_instance_eta():
    l, N, B = 4, 200, 40
    x = _grid(9, N)
    etas = [float(e) for e in np.geomspace(0.01, 0.2, B)]
    rng = np.random.default_rng(11)
    phis = rng.uniform(0.1, 1.0, (B, l, N))
    ctx = mm.Context(l, N, etas, batch=B, repr="linear", points=x)
    u = _dev([phis[:, q, :] for q in range(l)])
    k = 2
    got = ctx.marginal(k, u).cpu().numpy()
    W = ctx.cost(u)
    ctx.close()
    for b in (0, 13, 27, 39):
        pb = list(phis[b])
        want = pb[k] * points.product(pb, x, etas[b], k)
        assert np.max(np.abs(got[b] - want) / want) <= RTOL, b
        assert abs(W[b] - points.cost(pb, x, etas[b])) <= RTOL * abs(W[b])


def test_uniform_points_equal_uniform_context():
    l, N, eta = 5, 700, 0.05
    x = np.linspace(0.0, 1.0, N)
    phis = list(mmot_inputs.random_positive(12, l, N))
    a = mm.Context(l, N, eta, repr="linear", points=x)
    b = mm.Context(l, N, eta, repr="linear", kernel="two_walk")
    u = _dev(phis)
    for k in range(l):
        ga, gb = a.marginal(k, u).cpu().numpy(), b.marginal(k, u).cpu().numpy()
        assert np.max(np.abs(ga - gb) / gb) <= RTOL
    assert abs(a.cost(u) - b.cost(u)) <= RTOL * abs(b.cost(u))
    a.close()
    b.close()


@pytest.mark.parametrize("l,N", [(3, 9000), (4, 20000), (6, 2500)])
def test_points_two_walk_family(l, N):
    """Instances above the persistent-kernel size run on the two-walk family with per-edge decays."""
    x = _grid(500 + l, N)
    eta = 0.01
    phis = list(mmot_inputs.random_positive(600 + l, l, N))
    ctx = mm.Context(l, N, eta, repr="linear", points=x)
    assert ctx.info["kernel"] == "two_walk"
    u = _dev(phis)
    for k in (0, l - 1):
        got = ctx.marginal(k, u).cpu().numpy()
        want = phis[k] * points.product(phis, x, eta, k)
        assert np.max(np.abs(got - want) / want) <= RTOL, k
    W = ctx.cost(u)
    ctx.close()
    assert abs(W - points.cost(phis, x, eta)) <= RTOL * abs(W)


def test_points_two_walk_sinkhorn_with_residual():
    l, N, eta, T = 3, 6000, 0.02, 3
    x = _grid(77, N)
    mus = np.stack(mmot_inputs.random_marginals(78, l, N))
    ctx = mm.Context(l, N, eta, repr="log", points=x, check_every=1)
    assert ctx.info["kernel"] == "two_walk"
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev(mus), T, 1e-300, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    g = np.stack([v.cpu().numpy() for v in u])
    ctx.close()
    ref = points.sinkhorn(mus, x, eta, T)
    assert np.max(np.abs(g - np.log(ref))) <= 1e-9
    m = points.marginals(ref, x, eta)
    res_ref = float(sum(np.abs(m[k] - mus[k]).sum() for k in range(l - 1)))
    assert rep["residual"] == pytest.approx(res_ref, rel=1e-8)


@pytest.mark.parametrize("N", [1, 2, 3, 9])
def test_points_tiny_grids(N):
    l, eta = 3, 0.1
    x = np.sort(np.random.default_rng(N).uniform(0, 1, N)) if N > 1 else np.array([0.25])
    if N > 1:
        x = np.unique(x)
        assert len(x) == N
    phis = list(mmot_inputs.random_positive(40 + N, l, N))
    ctx = mm.Context(l, N, eta, repr="linear", points=x)
    u = _dev(phis)
    for k in range(l):
        got = ctx.marginal(k, u).cpu().numpy()
        want = phis[k] * points.product(phis, x, eta, k)
        assert np.max(np.abs(got - want) / want) <= RTOL, k
    W = ctx.cost(u)
    ctx.close()
    Wr = points.cost(phis, x, eta)
    assert abs(W - Wr) <= RTOL * max(abs(Wr), 1e-300) or (Wr == 0.0 and W == 0.0)


def test_points_rejects_single_walk_and_sharding_is_uniform_only():
    x = np.linspace(0.0, 1.0, 100) ** 2
    with pytest.raises(mm.MMOTError) as e:
        mm.Context(3, 100, 0.1, points=x, kernel="single_walk")
    assert e.value.name == "MMOT_EUNSUPPORTED"
    ctx = mm.Context(3, 100, 0.1, points=x, kernel="two_walk")
    assert ctx.info["kernel"] == "two_walk"
    ctx.close()
    with pytest.raises(mm.MMOTError) as e:
        mm.Context(3, 100, 0.1, points=x, shard=(0, 1, mm.nccl_unique_id()))
    assert e.value.name == "MMOT_EUNSUPPORTED"


@pytest.mark.parametrize("N", [600, 8000])
def test_points_f32_io_matches_f64(N):
    l, eta, T = 3, 0.02, 3
    x = _grid(21, N)
    mus = np.stack(mmot_inputs.random_marginals(22, l, N)).astype(np.float32)
    res = {}
    for dt in ("f32", "f64"):
        ctx = mm.Context(l, N, eta, dtype=dt, points=x)
        u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
        ctx.init_uniform(u)
        src = mus if dt == "f32" else mus.astype(np.float64)
        ctx.sinkhorn(_dev(src), T, 0.0, u)
        res[dt] = (np.stack([v.cpu().numpy() for v in u]), ctx.marginal(0, u).cpu().numpy())
        ctx.close()
    assert np.max(np.abs(res["f32"][0] - res["f64"][0])) <= 1e-12 * max(1.0, np.abs(res["f64"][0]).max())
    assert np.array_equal(res["f32"][1], res["f64"][1].astype(np.float32))
