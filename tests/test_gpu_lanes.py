"""The l = 6 lane-state family (csrc/lanes.cu: one warp per 32-point chain, the 32 subset states on
the lanes, two-level operator scan) against the fp64 oracle (O4 subset DP, pinned against O1 / O3)
and against the two-walk kernels (MMOT_NO_LANES=1).  Tolerance 1e-10 (north_star fp64)."""
import os

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


@pytest.mark.parametrize("N", [1, 5, 31, 32, 33, 1000, 1024 + 17, 32 * 32 * 3 + 5, 100_000])
def test_lanes_marginal_parity(N):
    l, eta = 6, 1e-3
    h = mmot_inputs.grid_h(N)
    phis = mmot_inputs.random_positive(6100 + N % 977, l, N)
    ctx = mm.Context(l, N, eta, repr="linear")
    assert ctx.info["kernel"] == "lanes"
    u = _dev(phis)
    w = regions.edge_weights(l, h, eta)
    for k in (0, 3, 5):
        got = ctx.marginal(k, u).cpu().numpy()
        want = phis[k] * subset.marginal_product(list(phis), k, w)
        assert np.max(np.abs(got - want) / want) <= RTOL, (N, k)
    ctx.close()


def _solve(N, eta, mus, T, tol, lanes):
    if lanes:
        os.environ.pop("MMOT_NO_LANES", None)
    else:
        os.environ["MMOT_NO_LANES"] = "1"
    try:
        ctx = mm.Context(6, N, eta, repr="log", check_every=1)
        kern = ctx.info["kernel"]
        u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(6)]
        ctx.init_uniform(u)
        rep = ctx.sinkhorn(_dev(mus), T, tol, u)
        g = np.stack([x.cpu().numpy() for x in u])
        W = ctx.cost(u)
        ctx.close()
    finally:
        os.environ.pop("MMOT_NO_LANES", None)
    return rep, g, W, kern


@pytest.mark.parametrize("tol", [0.0, 1e-300])
def test_lanes_sinkhorn_lockstep(tol):
    """C3-shaped (5-component mixtures + 1e-4 noise, eta = 1e-3) at N = 20000, 3 sweeps, vs the
    oracle and vs the two-walk kernels."""
    N, eta, T = 20_000, 1e-3, 3
    mus = mmot_inputs.c3_marginals(0, N, 6)
    rep, g, W, kern = _solve(N, eta, mus, T, tol, True)
    assert kern == "lanes" and rep["status"] == 0 and rep["iters_done"] == T
    phis, _, res_ref = osk.sinkhorn(mus, mmot_inputs.grid_h(N), eta, T, tol=tol, domain="plain", engine="subset")
    assert np.max(np.abs(g - np.log(phis))) <= 1e-9
    if tol > 0:
        assert rep["residual"] == pytest.approx(res_ref, rel=1e-9)
    rep2, g2, W2, kern2 = _solve(N, eta, mus, T, tol, False)
    assert kern2 == "two_walk"
    assert np.max(np.abs(g - g2)) <= 1e-11
    assert W == pytest.approx(W2, rel=1e-12)
