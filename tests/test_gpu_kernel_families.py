"""The four kernel families (two-walk, single-walk, persistent, sharded at world size 1) on the
same problems: each against the fp64 CPU oracle (1e-10), so a bug in any family cannot hide behind
another.  Problems sit inside the single-walk stability bound."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import regions, sinkhorn as osk  # noqa: E402

DEV = "cuda:0"


def _dev(vs):
    return [torch.from_numpy(np.ascontiguousarray(v)).to(DEV) for v in vs]


FAMILIES = [("two_walk", {}), ("single_walk", {"chunk": 32}), ("persistent", {}), ("sharded", {"chunk": 32})]


def _ctx(l, N, eta, fam, opts, repr_):
    if fam == "sharded":
        return mm.Context(l, N, eta, repr=repr_, shard=(0, 1, mm.nccl_unique_id()), kernel="single_walk", **opts)
    return mm.Context(l, N, eta, repr=repr_, kernel=fam, **opts)


@pytest.mark.parametrize("fam,opts", FAMILIES)
@pytest.mark.parametrize("l", [3, 4, 5])
def test_family_sinkhorn_marginals_cost(fam, opts, l):
    N = 3000
    h = mmot_inputs.grid_h(N)
    eta = h / (0.9 / (32 * ((l // 2) * ((l + 1) // 2))))  # single-walk bound at chain length 32
    mus = np.stack(mmot_inputs.random_marginals(900 + l, l, N))
    T = 3
    ctx = _ctx(l, N, eta, fam, opts, "log")
    assert ctx.info["kernel"] == ("single_walk" if fam == "sharded" else fam)
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev(mus), T, 0.0, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    marg = [ctx.marginal(k, u).cpu().numpy() for k in range(l)]
    W = ctx.cost(u)
    g = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    phis_ref, _, _ = osk.sinkhorn(mus, h, eta, T, domain="plain")
    assert np.max(np.abs(g - np.log(phis_ref))) <= 1e-9
    m_ref = osk.marginals(phis_ref, h, eta)
    for k in range(l):
        assert np.abs(marg[k] - m_ref[k]).sum() / np.abs(m_ref[k]).sum() <= 1e-10, k
    W_ref = osk.cost(phis_ref, h, eta)
    assert abs(W - W_ref) <= 1e-10 * abs(W_ref)
