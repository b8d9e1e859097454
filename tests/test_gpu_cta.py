"""GPU parity of the CTA family (cta.cu: a thread block per small instance, 256 chains, warp-level
operator scans, every sweep and residual check in one launch) against the fp64 CPU oracle.

Small single-instance contexts (C1, C2) and batches of at most one wave run on it when every
instance is inside (l-1)(x_max - x_min)/eta <= 500.  Cases: N from 1 to 4096 (chain lengths 1 .. 16,
ragged padding), l = 2 .. 4, fixed sweeps and the residual stop rule, several instances
with different eta, and the routing limits.  Tolerances (north_star fp64): marginals 1e-10
L1-relative, log phi 1e-9, the stop sweep exactly.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import regions, sinkhorn as osk  # noqa: E402

DEV = "cuda:0"


def _check(l, N, eta, mus_b, T, g_b, tol=0.0):
    h = mmot_inputs.grid_h(N)
    g_ref, t_ref, _ = osk.sinkhorn(mus_b, h, eta, T, tol=tol, domain="log", engine="subset")
    fin = np.isfinite(g_ref)
    assert np.array_equal(np.isfinite(g_b), fin)
    assert np.max(np.abs(g_b[fin] - g_ref[fin]) / np.maximum(1.0, np.abs(g_ref[fin]))) <= 1e-9
    lw = np.array([-(a * (l - a)) * h / eta for a in range(l + 1)])
    for k in range(l):
        m_ref = np.exp(g_ref[k] + regions.marginal_product_log(list(g_ref), k, lw))
        m_got = np.exp(g_b[k] + regions.marginal_product_log(list(g_b), k, lw))
        assert np.abs(m_got - m_ref).sum() / np.abs(m_ref).sum() <= 1e-10, k
    return t_ref


@pytest.mark.parametrize("l,N,eta,T", [(3, 64, 0.05, 40), (4, 1000, 0.01, 12), (2, 257, 0.02, 10),
                                       (3, 4096, 0.05, 4), (4, 1, 0.1, 3), (3, 2, 0.1, 5), (4, 300, 0.008, 8),
                                       (2, 3000, 0.1, 5)])
def test_cta_single_instance_lockstep(l, N, eta, T):
    mus = mmot_inputs.c2_marginals(40 + N, N, l)
    ctx = mm.Context(l, N, eta, repr="log")
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn([torch.from_numpy(m).to(DEV) for m in mus], T, 0.0, u)
    assert ctx.cta_solves == 1
    assert rep["status"] == 0 and rep["iters_done"] == T
    g = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    _check(l, N, eta, mus, T, g)


def test_cta_c2_stop_rule():
    """C2 as the bench runs it: tol = 1e-9 with the residual every sweep; the stop sweep and the
    scalings match the oracle's."""
    cfg = mmot_inputs.CONFIGS["C2"]
    l, N, eta = cfg.l, cfg.N, cfg.eta
    mus = mmot_inputs.make_marginals("C2", 0)
    ctx = mm.Context(l, N, eta, repr="log", check_every=1)
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn([torch.from_numpy(m).to(DEV) for m in mus], cfg.iters, cfg.tol, u)
    assert ctx.cta_solves == 1 and rep["converged"] and rep["status"] == 0
    g = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    t_ref = _check(l, N, eta, mus, rep["iters_done"], g)
    h = mmot_inputs.grid_h(N)
    _, t_stop, res = osk.sinkhorn(mus, h, eta, cfg.iters, tol=cfg.tol, domain="log", engine="subset")
    assert rep["iters_done"] == t_stop, (rep["iters_done"], t_stop)
    assert abs(rep["residual"] - res) <= 1e-6 * cfg.tol + 1e-3 * res


def test_cta_batch_and_routing(monkeypatch):
    """Several instances, one block each, per-instance eta; a batch member outside the range bound
    sends the whole batch to the persistent kernel; MMOT_NO_CTA=1 likewise; same iterates."""
    l, N, T = 4, 700, 8
    etas = [0.1, 0.02, 0.009, 0.05]
    mus = [mmot_inputs.c2_marginals(70 + b, N, l) for b in range(len(etas))]
    md = [torch.from_numpy(np.ascontiguousarray(np.stack([mus[b][q] for b in range(len(etas))]))).to(DEV)
          for q in range(l)]

    def run(etas_):
        ctx = mm.Context(l, N, etas_, batch=len(etas_))
        u = [torch.empty((len(etas_), N), dtype=torch.float64, device=DEV) for _ in range(l)]
        ctx.init_uniform(u)
        rep = ctx.sinkhorn(md, T, 0.0, u)
        n = ctx.cta_solves
        ctx.close()
        assert rep["status"] == 0
        return np.stack([x.cpu().numpy() for x in u]), n

    g, n = run(etas)
    assert n == 1
    for b in range(len(etas)):
        _check(l, N, etas[b], mus[b], T, g[:, b, :])
    _, n2 = run(etas[:3] + [0.004])          # 3 / 0.004 = 750 > 500
    assert n2 == 0
    monkeypatch.setenv("MMOT_NO_CTA", "1")
    g3, n3 = run(etas)
    assert n3 == 0
    fin = np.isfinite(g)
    assert np.max(np.abs(g3[fin] - g[fin]) / np.maximum(1.0, np.abs(g[fin]))) <= 1e-9
