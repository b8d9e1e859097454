"""The paper's Ricker-wavelet problem (§5.2): three
shifted Ricker wavelets on [-2, 2], N = 100, epsilon = 1e-3 (h/eta = 40.4).  The paper reports that
its recursion without log-domain stabilisation stops at the 89th iteration (Fig. 2b) while the
stabilised one runs on.  Pinned here: the generator (closed-form properties), the plain-domain
oracle's breakdown and the log-domain oracle's survival (CPU), and the GPU path -- whose scalings
are mantissas with per-chain binary exponents -- running all sweeps in lockstep with the
log-domain oracle (GPU)."""
import math
import warnings

import numpy as np
import pytest

import mmot_inputs
from oracle import sinkhorn as osk

N, ETA, T = 100, 1e-3, 200
X_MIN, X_MAX = -2.0, 2.0


def _h():
    return (X_MAX - X_MIN) / (N - 1)


def test_ricker_generator_closed_forms():
    mus = mmot_inputs.ricker_marginals(N)
    assert mus.shape == (3, N)
    assert np.allclose(mus.sum(axis=1), 1.0, rtol=0, atol=1e-14)
    assert mus.min() >= 1e-3 / (1 + N * 1e-3) - 1e-18       # the delta floor
    # f_1 = R(t) is even and the grid is symmetric about 0
    assert np.allclose(mus[0], mus[0][::-1], rtol=1e-12, atol=0)
    # R(t - tau) peaks at t = tau: the mode of mu_j sits at the grid point nearest tau_j
    t = np.linspace(X_MIN, X_MAX, N)
    for j, tau in enumerate((0.0, 0.75, 1.5)):
        assert abs(t[np.argmax(mus[j])] - tau) <= _h()
    # R vanishes at t = tau + 1/(sqrt 2 pi): the minimum of mu_j right of its mode lies within one
    # grid step of that zero
    for j, tau in enumerate((0.0, 0.75, 1.5)):
        z = tau + 1.0 / (math.sqrt(2.0) * math.pi)
        win = (t > tau) & (t < tau + 0.4)
        i = int(np.argmin(np.where(win, mus[j], np.inf)))
        assert abs(t[i] - z) <= _h()


def test_plain_domain_breaks_down_log_domain_survives():
    """Without stabilisation the scalings leave the fp64 range within the run (paper: iteration 89,
    here the first non-finite or zero scaling); the log-domain iteration stays finite throughout."""
    mus = mmot_inputs.ricker_marginals(N)
    first_bad = []

    def rec(t, xs):
        if not first_bad and not all(np.all(np.isfinite(x)) and np.all(x > 0) for x in xs):
            first_bad.append(t)

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        osk.sinkhorn(mus, _h(), ETA, T, domain="plain", record=rec)
    assert first_bad and first_bad[0] < T
    seen = []
    g, t, _ = osk.sinkhorn(mus, _h(), ETA, T, domain="log", record=lambda t, xs: seen.append(max(np.abs(x).max() for x in xs)))
    assert t == T and np.all(np.isfinite(g))
    assert max(seen) > 709.0  # |log phi| beyond exp's fp64 range: linear scalings cannot hold it


@pytest.mark.gpu
def test_ricker_gpu_lockstep_with_log_oracle():
    torch = pytest.importorskip("torch")
    import paper_2405_19246_b200 as mm
    mus = mmot_inputs.ricker_marginals(N)
    ctx = mm.Context(3, N, ETA, grid=(X_MIN, X_MAX), repr="log")
    u = [torch.empty(N, dtype=torch.float64, device="cuda:0") for _ in range(3)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn([torch.from_numpy(m).to("cuda:0") for m in mus], T, 0.0, u)
    g = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    assert rep["status"] == 0 and rep["iters_done"] == T
    g_ref, _, _ = osk.sinkhorn(mus, _h(), ETA, T, domain="log")
    assert np.max(np.abs(g - g_ref)) <= 1e-10 * max(1.0, np.abs(g_ref).max())
