"""NEXT-1: the all-marginals residual pass (MODE_ALLRES; include/mmot.h mmot_allres_checks).  One pass
of the subset recurrence over all l scalings (2^l states) yields every J_k; the residual
sum_{k<l-1} ||phi_k J_k - mu_k||_1 (Algorithm 1 line 7, generalised) from it must equal the
oracle's residual, give the oracle's stop sweep, and leave the solve identical to the l-1-product
path (MMOT_NO_ALLRES=1)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import sinkhorn as osk  # noqa: E402

DEV = "cuda:0"


def _solve(l, N, eta, mus, T, tol, allres, check_every=1):
    if allres:
        os.environ.pop("MMOT_NO_ALLRES", None)
    else:
        os.environ["MMOT_NO_ALLRES"] = "1"
    try:
        ctx = mm.Context(l, N, eta, repr="log", kernel="two_walk", check_every=check_every)
        u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
        ctx.init_uniform(u)
        rep = ctx.sinkhorn([torch.from_numpy(m).to(DEV) for m in mus], T, tol, u)
        g = np.stack([x.cpu().numpy() for x in u])
        n = ctx.allres_checks
        ctx.close()
    finally:
        os.environ.pop("MMOT_NO_ALLRES", None)
    return rep, g, n


@pytest.mark.parametrize("l,N,eta", [(2, 7000, 0.02), (3, 20001, 0.02), (4, 9000, 0.01), (5, 3000, 0.02)])
def test_allres_residual_matches_oracle(l, N, eta):
    T = 5
    mus = np.stack(mmot_inputs.random_marginals(5300 + l, l, N))
    rep, g, n = _solve(l, N, eta, mus, T, 1e-300, True, check_every=2)
    assert n == 3   # sweeps 2, 4 and the forced check at the last sweep
    _, _, res_ref = osk.sinkhorn(mus, mmot_inputs.grid_h(N), eta, T, tol=1e-300, domain="plain", engine="subset",
                                 check_every=2)
    assert rep["residual"] == pytest.approx(res_ref, rel=1e-9)
    rep_h, g_h, n_h = _solve(l, N, eta, mus, T, 1e-300, False, check_every=2)
    assert n_h == 0
    # the check pass leaves the update sequence untouched (the next update reuses its fused operators
    # instead of recomputing them: same values up to rounding order)
    assert np.max(np.abs(g - g_h)) <= 1e-12
    assert rep["residual"] == pytest.approx(rep_h["residual"], rel=1e-12)


def test_allres_stop_sweep():
    """tol > 0 through the single-pass residual: the oracle's stop sweep."""
    l, N, eta, tol = 4, 20000, 0.1, 1e-6
    mus = mmot_inputs.c4_marginals(11, N, l, width=200)
    _, t_ref, res_ref = osk.sinkhorn(mus, mmot_inputs.grid_h(N), eta, 400, tol=tol, domain="plain", engine="subset")
    assert t_ref < 400
    rep, _, n = _solve(l, N, eta, mus, 400, tol, True)
    assert rep["converged"] and rep["iters_done"] == t_ref and n >= t_ref
    assert rep["residual"] == pytest.approx(res_ref, rel=1e-8)
