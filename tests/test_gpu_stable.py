"""The stabilised family (MMOT_KERNEL_STABLE, csrc/stable.cu: the subset recurrence in the log domain,
the paper's log-domain stabilisation -- Remark 1 P:138-151, Algorithm 5) and the automatic
range fallback of the plain families (include/mmot.h mmot_stable_fallback_count), against the fp64
CPU oracle: plain products where fp64 represents them, the log-domain driver (P:1029-1035 with
log-domain products) where it does not.  Tolerance 1e-10 (north_star fp64)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import regions, sinkhorn as osk, subset  # noqa: E402

DEV = "cuda:0"
RTOL = 1e-10


def _dev(vs):
    return [torch.from_numpy(np.ascontiguousarray(v)).to(DEV) for v in vs]


def _log_marginals(g, h, eta):
    l = len(g)
    lw = np.array([-(a * (l - a)) * h / eta for a in range(l + 1)])
    return [np.exp(g[k] + subset.marginal_product_log(list(g), k, lw)) for k in range(l)]


def _gclose(g, g_ref, tol=1e-9):
    fin = np.isfinite(g_ref)
    assert np.array_equal(fin, np.isfinite(g))
    return float(np.max(np.abs(g[fin] - g_ref[fin]) / np.maximum(1.0, np.abs(g_ref[fin])))) <= tol


@pytest.mark.parametrize("l", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("N", [1, 7, 300])
def test_stable_marginal_and_cost_parity(l, N):
    h = mmot_inputs.grid_h(N)
    eta = 0.02
    phis = mmot_inputs.random_positive(3100 + 10 * l + N, l, N)
    ctx = mm.Context(l, N, eta, repr="linear", kernel="stable")
    assert ctx.info["kernel"] == "stable"
    u = _dev(phis)
    w = regions.edge_weights(l, h, eta)
    for k in range(l):
        got = ctx.marginal(k, u).cpu().numpy()
        want = phis[k] * regions.marginal_product(list(phis), k, w)
        assert np.max(np.abs(got - want) / want) <= RTOL, (l, N, k)
    W = ctx.cost(u)
    ctx.close()
    W_ref = osk.cost(phis, h, eta)
    assert abs(W - W_ref) <= RTOL * abs(W_ref) + 1e-300, (W, W_ref)


@pytest.mark.parametrize("l,N,eta,T", [(3, 200, 0.01, 10), (4, 150, 0.003, 6), (5, 64, 0.05, 4)])
def test_stable_sinkhorn_lockstep(l, N, eta, T):
    h = mmot_inputs.grid_h(N)
    mus = np.stack(mmot_inputs.c2_marginals(1, N, l))
    ctx = mm.Context(l, N, eta, repr="log", kernel="stable", check_every=1)
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev(mus), T, 1e-300, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    g = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    g_ref, _, res_ref = osk.sinkhorn(mus, h, eta, T, tol=1e-300, domain="log", engine="subset")
    assert _gclose(g, g_ref)
    assert rep["residual"] == pytest.approx(res_ref, rel=1e-8)


def _disjoint(N):
    x = np.arange(N) / (N - 1)
    mus = np.stack([(x < 0.3).astype(float), (x > 0.7).astype(float), np.ones(N)])
    return mus / mus.sum(axis=1, keepdims=True)


@pytest.mark.parametrize("kernel,N,eta,T", [("two_walk", 400, 1e-4, 5), ("persistent", 400, 1e-4, 5),
                                            ("persistent", 12000, 1e-3, 3), ("auto", 3000, 1e-4, 3)])
def test_disjoint_supports_fall_back_to_log_domain(kernel, N, eta, T):
    """Disjoint supports 0.4 apart at eta = 1e-4 / 1e-3: crossing the gap costs e^-0.8/eta, far below
    e^-708 -- the plain fp64 families cannot represent J_k and report EOVERFLOW internally; the call is
    redone on the stabilised family and runs in lockstep with the log-domain oracle (round-1 behaviour:
    the solve stopped with MMOT_EOVERFLOW at sweep 1)."""
    l = 3
    h = mmot_inputs.grid_h(N)
    mus = _disjoint(N)
    ctx = mm.Context(l, N, eta, repr="log", kernel=kernel)
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev(mus), T, 0.0, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    assert ctx.stable_fallbacks >= 1
    g = np.stack([x.cpu().numpy() for x in u])
    marg = [ctx.marginal(k, u).cpu().numpy() for k in range(l)]
    ctx.close()
    g_ref, _, _ = osk.sinkhorn(mus, h, eta, T, domain="log", engine="subset")
    assert np.nanmax(np.abs(g_ref)) > 709           # beyond fp64's exponent range
    assert _gclose(g, g_ref)
    m_ref = _log_marginals(g_ref, h, eta)
    for k in range(l):
        assert np.abs(marg[k] - m_ref[k]).sum() / np.abs(m_ref[k]).sum() <= RTOL, k


def test_batched_fallback_redoes_only_failed_instances():
    """A batch where one instance has disjoint supports at eta = 1e-4: that instance alone is redone on
    the stabilised family, the others keep the persistent kernel's results; all match the oracle."""
    l, N = 3, 300
    h = mmot_inputs.grid_h(N)
    etas = [0.05, 1e-4, 0.01]
    mus = [np.stack(mmot_inputs.c2_marginals(0, N, l)), _disjoint(N), np.stack(mmot_inputs.c2_marginals(2, N, l))]
    B, T = len(etas), 4
    ctx = mm.Context(l, N, etas, batch=B, repr="log")
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev([np.stack([mus[b][q] for b in range(B)]) for q in range(l)]), T, 0.0, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    assert ctx.stable_fallbacks == 1
    g = np.stack([x.cpu().numpy() for x in u])   # [l][B][N]
    ctx.close()
    for b in range(B):
        g_ref, _, _ = osk.sinkhorn(mus[b], h, etas[b], T, domain="log", engine="subset")
        assert _gclose(g[:, b, :], g_ref), b


def test_stable_batched_explicit():
    l, N = 4, 100
    h = mmot_inputs.grid_h(N)
    etas = [1e-3, 0.02]
    B, T = 2, 5
    mus = [np.stack(mmot_inputs.c2_marginals(b + 5, N, l)) for b in range(B)]
    ctx = mm.Context(l, N, etas, batch=B, repr="log", kernel="stable")
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev([np.stack([mus[b][q] for b in range(B)]) for q in range(l)]), T, 0.0, u)
    assert rep["status"] == 0
    g = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    for b in range(B):
        g_ref, _, _ = osk.sinkhorn(mus[b], h, etas[b], T, domain="log", engine="subset")
        assert _gclose(g[:, b, :], g_ref), b


# ---- l = 7, 8 (include/mmot.h MMOT_MAX_L = 8; SURVEY §8(b) l in [2, 8]): 64 / 128 subset states, 2 / 4
# per lane of the instance's warp, bound marginals 5, 6 pairing registers instead of lanes.  The
# oracle is O4 (oracle/subset.c, pinned against the dense definition at l = 7, 8 in
# tests/test_oracle_subset.py); the region-chain oracle would need l! = 5040 / 40320 chains.

def _subset_cost(phis, h, eta):
    l = len(phis)
    w = regions.edge_weights(l, h, eta)
    _, jh = subset.marginal_product(list(phis), l - 1, w, want_hat=True)
    return float(h * np.dot(phis[l - 1], jh))


@pytest.mark.parametrize("l", [7, 8])
@pytest.mark.parametrize("N", [1, 7, 130])
def test_l78_marginal_and_cost_parity(l, N):
    h = mmot_inputs.grid_h(N)
    eta = 0.05
    phis = mmot_inputs.random_positive(4100 + 10 * l + N, l, N)
    ctx = mm.Context(l, N, eta, repr="linear")  # AUTO: l > 6 takes the stabilised family
    assert ctx.info["kernel"] == "stable"
    u = _dev(phis)
    w = regions.edge_weights(l, h, eta)
    for k in range(l):
        got = ctx.marginal(k, u).cpu().numpy()
        want = phis[k] * subset.marginal_product(list(phis), k, w)
        assert np.max(np.abs(got - want) / want) <= RTOL, (l, N, k)
    W = ctx.cost(u)
    ctx.close()
    W_ref = _subset_cost(phis, h, eta)
    assert abs(W - W_ref) <= RTOL * abs(W_ref) + 1e-300, (W, W_ref)


@pytest.mark.parametrize("l,N,eta,T", [(7, 96, 0.02, 4), (8, 64, 0.05, 3), (7, 200, 1e-3, 3)])
def test_l78_sinkhorn_lockstep(l, N, eta, T):
    h = mmot_inputs.grid_h(N)
    mus = np.stack(mmot_inputs.c2_marginals(2, N, l))
    ctx = mm.Context(l, N, eta, repr="log", kernel="stable", check_every=1)
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev(mus), T, 1e-300, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    g = np.stack([x.cpu().numpy() for x in u])
    # after the last update of a sweep the l-th marginal of the plan is mu_l
    m_last = ctx.marginal(l - 1, u).cpu().numpy()
    ctx.close()
    g_ref, _, res_ref = osk.sinkhorn(mus, h, eta, T, tol=1e-300, domain="log", engine="subset")
    assert _gclose(g, g_ref)
    assert rep["residual"] == pytest.approx(res_ref, rel=1e-8)
    assert np.abs(m_last - mus[l - 1]).sum() <= 1e-12


def test_l78_batched_and_host_buffers():
    l, N, B, T = 7, 60, 3, 3
    h = mmot_inputs.grid_h(N)
    etas = [0.01, 0.05, 0.2]
    mus = [np.stack(mmot_inputs.c2_marginals(b + 11, N, l)) for b in range(B)]
    ctx = mm.Context(l, N, etas, batch=B, repr="log")
    assert ctx.info["kernel"] == "stable"
    mh = [torch.from_numpy(np.stack([mus[b][q] for b in range(B)])).pin_memory() for q in range(l)]
    uh = [torch.full((B, N), -np.log(N), dtype=torch.float64).pin_memory() for _ in range(l)]
    rep = ctx.sinkhorn_host(mh, T, 0.0, uh)
    assert rep["status"] == 0
    g = np.stack([x.numpy() for x in uh])
    ctx.close()
    for b in range(B):
        g_ref, _, _ = osk.sinkhorn(mus[b], h, etas[b], T, domain="log", engine="subset")
        assert _gclose(g[:, b, :], g_ref), b


def test_l78_unsupported_requests():
    with pytest.raises(mm.MMOTError):
        mm.Context(7, 50, 0.05, kernel="two_walk")
    with pytest.raises(mm.MMOTError):
        mm.Context(8, 50, 0.05, dtype="f32")
