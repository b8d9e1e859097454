"""Device-resident Sinkhorn loop: the sweep loop of mmot_sinkhorn as one launch of a
cached CUDA graph with a conditional WHILE node (include/mmot.h mmot_graph_solves).  The graph
replays exactly the launch sequence of the host-issued loop, so results must be bit-identical to
MMOT_NO_GRAPH=1 runs, and the device stop rule must stop at the same sweep; both are then
checked against the fp64 oracle."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import sinkhorn as osk  # noqa: E402

DEV = "cuda:0"


def _solve(l, N, eta, mus, T, tol, graph, **kw):
    if graph:
        os.environ.pop("MMOT_NO_GRAPH", None)
    else:
        os.environ["MMOT_NO_GRAPH"] = "1"
    try:
        ctx = mm.Context(l, N, eta, repr="log", **kw)
        u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
        ctx.init_uniform(u)
        rep = ctx.sinkhorn([torch.from_numpy(m).to(DEV) for m in mus], T, tol, u)
        g = np.stack([x.cpu().numpy() for x in u])
        gs, kern = ctx.graph_solves, ctx.info["kernel"]
        ctx.close()
    finally:
        os.environ.pop("MMOT_NO_GRAPH", None)
    return rep, g, gs, kern


@pytest.mark.parametrize("l,N,eta,kw,T,tol", [
    (3, 200_000, 0.05, dict(kernel="single_walk", chunk=64), 9, 0.0),     # restricted scan, odd l: period 2
    (4, 200_000, 0.05, dict(kernel="single_walk", chunk=64), 7, 0.0),     # restricted scan, period 1
    (4, 50_000, 0.02, dict(kernel="two_walk"), 6, 0.0),                    # fused next-update operators
    (6, 20_000, 0.01, dict(kernel="two_walk"), 5, 0.0),                    # l = 6: operators every update
    (4, 50_000, 0.02, dict(kernel="two_walk", check_every=3), 11, 1e-300),  # residual every 3 sweeps, ragged end
    (3, 200_000, 0.05, dict(kernel="single_walk", chunk=64, check_every=2), 8, 1e-300),
])
def test_graph_loop_bit_identical_to_host_loop(l, N, eta, kw, T, tol):
    mus = np.stack(mmot_inputs.random_marginals(4400 + l + T, l, N))
    rep_g, g_g, gs, kern = _solve(l, N, eta, mus, T, tol, True, **kw)
    rep_h, g_h, gs_h, _ = _solve(l, N, eta, mus, T, tol, False, **kw)
    assert gs == 1 and gs_h == 0, (gs, gs_h, kern)
    assert rep_g["status"] == 0 and rep_g["iters_done"] == rep_h["iters_done"] == T
    assert np.array_equal(g_g, g_h)
    if tol > 0:
        assert rep_g["residual"] == rep_h["residual"]
    phis, _, res_ref = osk.sinkhorn(mus, mmot_inputs.grid_h(N), eta, T, tol=tol, domain="plain", engine="subset",
                                    check_every=kw.get("check_every", 1))
    assert np.max(np.abs(g_g - np.log(phis))) <= 1e-9
    if tol > 0:
        assert rep_g["residual"] == pytest.approx(res_ref, rel=1e-9)


def test_graph_loop_device_stop_rule():
    """tol > 0: the WHILE node stops at the oracle's stop sweep (first residual <= tol), which is not a
    multiple of the host's polling cadence."""
    l, N, eta, tol = 3, 20_000, 0.1, 1e-6
    mus = mmot_inputs.c4_marginals(8, N, l, width=200)
    _, t_ref, res_ref = osk.sinkhorn(mus, mmot_inputs.grid_h(N), eta, 500, tol=tol, domain="plain", engine="subset")
    rep, g, gs, _ = _solve(l, N, eta, mus, 500, tol, True, kernel="two_walk", check_every=1)
    assert gs == 1
    assert rep["converged"] and rep["iters_done"] == t_ref
    assert rep["residual"] == pytest.approx(res_ref, rel=1e-8)
    rep_h, g_h, _, _ = _solve(l, N, eta, mus, 500, tol, False, kernel="two_walk", check_every=1)
    assert np.array_equal(g, g_h)
