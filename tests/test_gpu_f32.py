"""MMOT_F32 contexts (fp32 I/O): float marginals in, float marginal outputs out, fp64 scans.
The fp64 reference of an fp32 run is computed from the same fp32-rounded inputs;
north_star's fp32 tolerance is 1e-4 relative, and since the arithmetic is fp64 the results also
agree with the fp64 path on the rounded inputs to fp64 rounding."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import sinkhorn as osk  # noqa: E402

DEV = "cuda:0"


@pytest.mark.parametrize("l,N,eta,kernel", [(3, 300, 0.05, "auto"), (4, 5000, 0.01, "auto"),
                                            (4, 200_000, 1e-4, "auto"), (5, 3000, 0.02, "two_walk")])
def test_f32_sinkhorn_and_marginal(l, N, eta, kernel):
    mus = np.stack(mmot_inputs.random_marginals(900 + l, l, N)).astype(np.float32)
    mus64 = mus.astype(np.float64)
    T = 3
    h = mmot_inputs.grid_h(N)
    ctx = mm.Context(l, N, eta, dtype="f32", kernel=kernel)
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn([torch.from_numpy(m).to(DEV) for m in mus], T, 0.0, u)
    assert rep["status"] == 0
    m0 = ctx.marginal(0, u)
    assert m0.dtype == torch.float32
    g = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    if N <= 5000:
        g_ref, _, _ = osk.sinkhorn(mus64, h, eta, T, domain="log")
        assert np.max(np.abs(g - g_ref)) <= 1e-9
        m_ref = osk.marginals(np.exp(g_ref), h, eta)[0]
        assert np.abs(m0.cpu().numpy() - m_ref).sum() / m_ref.sum() <= 1e-4
    # same as the fp64 path on the rounded inputs
    c64 = mm.Context(l, N, eta, kernel=kernel)
    u64 = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    c64.init_uniform(u64)
    c64.sinkhorn([torch.from_numpy(m).to(DEV) for m in mus64], T, 0.0, u64)
    g64 = np.stack([x.cpu().numpy() for x in u64])
    m64 = c64.marginal(0, u64).cpu().numpy()
    c64.close()
    assert np.max(np.abs(g - g64)) <= 1e-12 * max(1.0, np.abs(g64).max())
    assert np.max(np.abs(m0.cpu().numpy() - m64.astype(np.float32))) == 0.0


def test_f32_batched_and_host_path():
    l, N, B, T = 5, 512, 24, 3
    etas = [float(e) for e in mmot_inputs.c5_etas(B)]
    mus = mmot_inputs.c5_batch_marginals(0, B, N, l).astype(np.float32)   # [l][B][N]
    ctx = mm.Context(l, N, etas, batch=B, dtype="f32")
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    ctx.sinkhorn([torch.from_numpy(np.ascontiguousarray(mus[q])).to(DEV) for q in range(l)], T, 0.0, u)
    g = np.stack([x.cpu().numpy() for x in u])
    # host path: float marginals cross PCIe, every instance's planes copied
    mh = [torch.from_numpy(np.ascontiguousarray(mus[q])).pin_memory() for q in range(l)]
    uh = [torch.full((B, N), -np.log(N), dtype=torch.float64).pin_memory() for _ in range(l)]
    ctx.sinkhorn_host(mh, T, 0.0, uh)
    gh = np.stack([x.numpy() for x in uh])
    ctx.close()
    assert np.array_equal(g, gh)
    h = mmot_inputs.grid_h(N)
    for b in (0, 11, 23):
        g_ref, _, _ = osk.sinkhorn(mus[:, b, :].astype(np.float64), h, etas[b], T, domain="log")
        assert np.max(np.abs(g[:, b, :] - g_ref)) <= 1e-8 * max(1.0, np.abs(g_ref).max())


def test_f64_batched_host_path_copies_every_instance():
    """mmot_sinkhorn_host on a batched fp64 context moves all batch x N elements per vector."""
    l, N, B, T = 3, 200, 7, 4
    mus = np.stack([mmot_inputs.c2_marginals(b, N, l) for b in range(B)])   # [B][l][N]
    ctx = mm.Context(l, N, [0.05] * B, batch=B)
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    ctx.sinkhorn([torch.from_numpy(np.ascontiguousarray(mus[:, q, :])).to(DEV) for q in range(l)], T, 0.0, u)
    g = np.stack([x.cpu().numpy() for x in u])
    mh = [torch.from_numpy(np.ascontiguousarray(mus[:, q, :])).pin_memory() for q in range(l)]
    uh = [torch.full((B, N), -np.log(N), dtype=torch.float64).pin_memory() for _ in range(l)]
    ctx.sinkhorn_host(mh, T, 0.0, uh)
    ctx.close()
    assert np.array_equal(g, np.stack([x.numpy() for x in uh]))


def test_f32_sharded_world1_matches_f64():
    l, N, eta, T = 4, 30000, 0.005, 2
    mus = np.stack(mmot_inputs.random_marginals(31, l, N)).astype(np.float32)
    res = {}
    for dt in ("f32", "f64"):
        ctx = mm.Context(l, N, eta, dtype=dt, shard=(0, 1, mm.nccl_unique_id()))
        u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
        ctx.init_uniform(u)
        src = mus if dt == "f32" else mus.astype(np.float64)
        ctx.sinkhorn([torch.from_numpy(m).to(DEV) for m in src], T, 0.0, u)
        res[dt] = (np.stack([x.cpu().numpy() for x in u]), ctx.marginal(1, u).cpu().numpy(), ctx.cost(u))
        ctx.close()
    assert np.max(np.abs(res["f32"][0] - res["f64"][0])) <= 1e-12 * max(1.0, np.abs(res["f64"][0]).max())
    assert res["f32"][1].dtype == np.float32
    assert np.array_equal(res["f32"][1], res["f64"][1].astype(np.float32))
    assert res["f32"][2] == pytest.approx(res["f64"][2], rel=1e-12)
