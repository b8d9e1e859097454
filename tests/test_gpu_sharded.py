"""Sharded contexts (mmot_create_sharded: one instance split by contiguous grid chunks over the
ranks, whole-shard operators exchanged with ncclAllGather) on ONE GPU: world_size 1, so the
NCCL exchange, the carry composition kernel and the shard bookkeeping all run, and the results
must equal the fp64 CPU oracle (1e-10).  The world_size > 1 composition logic is covered on CPU
by tests/test_shard_cpu.py (gloo); this run has a single GPU."""
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


@pytest.mark.parametrize("kernel,chunk,eta", [("two_walk", 0, 0.01), ("single_walk", 64, 2.0)])
def test_sharded_world1_marginal_and_cost(kernel, chunk, eta):
    l, N = 4, 20000
    h = mmot_inputs.grid_h(N)
    phis = mmot_inputs.random_positive(31, l, N)
    uid = mm.nccl_unique_id()
    ctx = mm.Context(l, N, eta, repr="linear", shard=(0, 1, uid), kernel=kernel, chunk=chunk)
    assert ctx.N == N and ctx.info["kernel"] == kernel
    u = _dev(phis)
    w = regions.edge_weights(l, h, eta)
    for k in range(l):
        got = ctx.marginal(k, u).cpu().numpy()
        want = phis[k] * regions.marginal_product(list(phis), k, w)
        assert np.max(np.abs(got - want) / want) <= 1e-10, k
    W = ctx.cost(u)
    W_ref = osk.cost(phis, h, eta)
    assert abs(W - W_ref) <= 1e-10 * abs(W_ref)
    ctx.close()


def test_sharded_world1_sinkhorn_lockstep():
    l, N, eta, T = 4, 6000, 0.02, 4
    h = mmot_inputs.grid_h(N)
    mus = np.stack(mmot_inputs.random_marginals(77, l, N))
    uid = mm.nccl_unique_id()
    ctx = mm.Context(l, N, eta, repr="log", shard=(0, 1, uid), check_every=1)
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev(mus), T, 1e-300, u)   # tol > 0: residual path with its all-reduce
    assert rep["status"] == 0 and rep["iters_done"] == T
    g = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    g_ref, _, res_ref = osk.sinkhorn(mus, h, eta, T, tol=1e-300, domain="log")
    assert np.max(np.abs(g - g_ref)) <= 1e-9
    assert rep["residual"] == pytest.approx(res_ref, rel=1e-8)


def test_sharded_small_shard_uses_scan_kernel():
    """A shard small enough for the persistent kernel still gets a scan-based family (the
    persistent kernel has no cross-rank exchange); an explicit persistent request is refused."""
    l, N, eta, T = 4, 1000, 0.05, 3
    h = mmot_inputs.grid_h(N)
    mus = np.stack(mmot_inputs.random_marginals(78, l, N))
    uid = mm.nccl_unique_id()
    ctx = mm.Context(l, N, eta, repr="log", shard=(0, 1, uid))
    assert ctx.info["kernel"] in ("two_walk", "single_walk")
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev(mus), T, 0.0, u)
    assert rep["status"] == 0
    g = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    g_ref, _, _ = osk.sinkhorn(mus, h, eta, T, domain="log")
    assert np.max(np.abs(g - g_ref)) <= 1e-9
    with pytest.raises(mm.MMOTError) as e:
        mm.Context(l, N, eta, shard=(0, 1, mm.nccl_unique_id()), kernel="persistent")
    assert e.value.name == "MMOT_EUNSUPPORTED"
