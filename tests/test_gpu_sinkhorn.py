"""GPU Sinkhorn (mmot_sinkhorn) in lockstep with the fp64 CPU oracle driver, plus error paths.

Measured per SURVEY §8(c): for every k, ||m_gpu - m_ref||_1 / ||m_ref||_1 <= 1e-10 at each
checkpoint, |W_gpu - W_ref| / |W_ref| <= 1e-10; diagnostic: max |log phi_gpu - log phi_ref|.
Parity runs use a fixed iteration count (A7), except the tol test which checks the
stop iteration itself.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import dense, sinkhorn as osk  # noqa: E402

DEV = "cuda:0"


def _dev(vs):
    return [torch.from_numpy(np.ascontiguousarray(v)).to(DEV) for v in vs]


def _run_gpu(mus, eta, T, tol=0.0, repr_="log", check_every=0, chunk=0, kernel="auto"):
    l, N = mus.shape
    ctx = mm.Context(l, N, eta, repr=repr_, check_every=check_every, chunk=chunk, kernel=kernel)
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev(mus), T, tol, u)
    g = np.stack([x.cpu().numpy() for x in u])
    marg = np.stack([ctx.marginal(k, u).cpu().numpy() for k in range(l)])
    W = ctx.cost(u)
    ctx.close()
    if repr_ == "linear":
        g = np.log(g)
    return rep, g, marg, W


def _l1rel(a, b):
    return float(np.abs(a - b).sum() / np.abs(b).sum())


@pytest.mark.parametrize("T", [1, 2, 5, 10, 20, 200])
def test_c1_lockstep_with_dense_and_oracle(T):
    """C1: l=3, N=64, eta=0.05, fp64; dense N^3 brute force cross-check (BASELINE configs[0])."""
    cfg = mmot_inputs.CONFIGS["C1"]
    mus = mmot_inputs.make_marginals("C1", 0)
    h = mmot_inputs.grid_h(cfg.N)
    rep, g, marg, W = _run_gpu(mus, cfg.eta, T)
    assert rep["status"] == 0 and rep["iters_done"] == T
    g_ref, _, _ = osk.sinkhorn(mus, h, cfg.eta, T, domain="log")
    phis_ref = np.exp(g_ref)
    m_ref = osk.marginals(phis_ref, h, cfg.eta)
    for k in range(cfg.l):
        assert _l1rel(marg[k], m_ref[k]) <= 1e-10
    assert abs(W - osk.cost(phis_ref, h, cfg.eta)) <= 1e-10 * abs(W)
    assert np.max(np.abs(g - g_ref)) <= 1e-9
    if T <= 20:
        p_dense, _, _ = dense.sinkhorn(mus, h, cfg.eta, T)
        np.testing.assert_allclose(np.exp(g), p_dense, rtol=1e-9)


def test_c2_to_tolerance():
    """C2: l=4, N=1000, eta=0.01, Sinkhorn to Res <= 1e-9 (max 2000): the GPU stops at the same
    sweep as the oracle and the solutions agree (A7: the stop iteration is compared, then the state)."""
    cfg = mmot_inputs.CONFIGS["C2"]
    mus = mmot_inputs.make_marginals("C2", 0)
    h = mmot_inputs.grid_h(cfg.N)
    rep, g, marg, W = _run_gpu(mus, cfg.eta, cfg.iters, tol=cfg.tol)
    g_ref, t_ref, res_ref = osk.sinkhorn(mus, h, cfg.eta, cfg.iters, tol=cfg.tol, domain="log")
    assert rep["converged"] and rep["iters_done"] == t_ref, (rep, t_ref, res_ref)
    assert rep["residual"] == pytest.approx(res_ref, rel=1e-4)
    phis_ref = np.exp(g_ref)
    m_ref = osk.marginals(phis_ref, h, cfg.eta)
    for k in range(cfg.l):
        assert _l1rel(marg[k], m_ref[k]) <= 1e-10
    assert abs(W - osk.cost(phis_ref, h, cfg.eta)) <= 1e-10 * abs(W)


@pytest.mark.parametrize("T", [1, 3])
def test_c3_fp64_reduced_lockstep(T):
    """C3 shape (l=6, eta=1e-3, 5-comp mixtures + noise) at reduced N=3000."""
    cfg = mmot_inputs.CONFIGS["C3"]
    N = 3000
    mus = mmot_inputs.make_marginals("C3", 0, N)
    h = mmot_inputs.grid_h(N)
    rep, g, marg, W = _run_gpu(mus, cfg.eta, T)
    assert rep["status"] == 0
    g_ref, _, _ = osk.sinkhorn(mus, h, cfg.eta, T, domain="log")
    phis_ref = np.exp(g_ref)
    m_ref = osk.marginals(phis_ref, h, cfg.eta)
    for k in range(cfg.l):
        assert _l1rel(marg[k], m_ref[k]) <= 1e-10


def test_c3_full_size_first_sweep():
    """C3 at its full size (l=6, N=1e5, eta=1e-3) in the bench's launch configuration: one sweep
    of six fused updates, compared with the oracle's first sweep (plain fp64 region chains,
    which represent C3), marginals elementwise-L1 and log phi."""
    cfg = mmot_inputs.CONFIGS["C3"]
    mus = mmot_inputs.make_marginals("C3", 0)
    h = mmot_inputs.grid_h(cfg.N)
    rep, g, marg, W = _run_gpu(mus, cfg.eta, 1)
    assert rep["status"] == 0 and rep["iters_done"] == 1
    phis_ref, _, _ = osk.sinkhorn(mus, h, cfg.eta, 1, domain="plain")
    assert np.max(np.abs(g - np.log(phis_ref))) <= 1e-9
    m_ref = osk.marginals(phis_ref, h, cfg.eta)
    for k in range(cfg.l):
        assert _l1rel(marg[k], m_ref[k]) <= 1e-10, k


def test_c4_shape_reduced_lockstep():
    """C4 recipe (l=4, eta=1e-4, smoothed random field) at N=2e5, 3 sweeps."""
    N = 200_000
    mus = mmot_inputs.make_marginals("C4", 0, N)
    h = mmot_inputs.grid_h(N)
    eta = 1e-4
    rep, g, marg, W = _run_gpu(mus, eta, 3)
    g_ref, _, _ = osk.sinkhorn(mus, h, eta, 3, domain="plain")
    g_ref = np.log(g_ref)
    phis_ref = np.exp(g_ref)
    m_ref = osk.marginals(phis_ref, h, eta)
    for k in range(4):
        assert _l1rel(marg[k], m_ref[k]) <= 1e-10
    assert abs(W - osk.cost(phis_ref, h, eta)) <= 1e-10 * abs(W)


def test_linear_repr_and_host_entry_agree():
    mus = mmot_inputs.make_marginals("C2", 1, 500)
    l, N = mus.shape
    rep_a, g_a, _, _ = _run_gpu(mus, 0.02, 15, repr_="log")
    rep_b, g_b, _, _ = _run_gpu(mus, 0.02, 15, repr_="linear")
    np.testing.assert_allclose(g_b, g_a, atol=1e-11)
    ctx = mm.Context(l, N, 0.02)
    with pytest.raises(mm.MMOTError):
        ctx.cost_staged()  # nothing staged yet
    u = [np.full(N, -math.log(N)) for _ in range(l)]
    rep = ctx.sinkhorn_host([np.ascontiguousarray(m) for m in mus], 15, 0.0, u)
    W = ctx.cost_staged()  # mmot_cost of the scalings the host call left on the device
    ctx.close()
    np.testing.assert_allclose(np.stack(u), g_a, atol=1e-11)
    W_ref = osk.cost(np.exp(np.stack(u)), mmot_inputs.grid_h(N), 0.02)
    assert abs(W - W_ref) <= 1e-10 * abs(W_ref)


def test_residual_cadence():
    mus = mmot_inputs.make_marginals("C2", 2, 400)
    rep, *_ = _run_gpu(mus, 0.05, 300, tol=1e-8, check_every=7)
    assert rep["converged"] and rep["iters_done"] % 7 == 0


@pytest.mark.parametrize("bad,code", [("nan", "MMOT_ENONFINITE"), ("neg", "MMOT_ENEGMASS"), ("zero", "MMOT_EZEROMASS")])
def test_data_errors(bad, code):
    mus = mmot_inputs.make_marginals("C1", 0).copy()
    if bad == "nan":
        mus[1, 5] = np.nan
    elif bad == "neg":
        mus[2, 7] = -1e-3
    else:
        mus[0, :] = 0.0
    with pytest.raises(mm.MMOTError) as ei:
        _run_gpu(mus, 0.05, 5)
    assert ei.value.name == code


def test_overflow_reported_without_stabilised_fallback(monkeypatch):
    """Plain fp64 scalings cannot represent disjoint supports at eta = 1e-4 (the kernel between the
    supports underflows to 0, so phi = mu / 0): with the range fallback disabled (MMOT_NO_STABLE=1)
    the run stops with EOVERFLOW and the sweep index (the analogue of the paper's unstabilised
    failure); tests/test_gpu_stable.py covers the default, stabilised behaviour."""
    monkeypatch.setenv("MMOT_NO_STABLE", "1")
    N = 400
    x = np.arange(N) / (N - 1)
    mus = np.stack([(x < 0.3).astype(float), (x > 0.7).astype(float), np.ones(N)])
    mus /= mus.sum(axis=1, keepdims=True)
    with pytest.raises(mm.MMOTError) as ei:
        _run_gpu(mus, 1e-4, 50, kernel="two_walk")
    assert ei.value.name == "MMOT_EOVERFLOW"
    assert ei.value.report["fail_iter"] == 1


@pytest.mark.parametrize("kernel", ["two_walk", "persistent"])
def test_c2_to_tolerance_both_kernels(kernel):
    """C2 stop iteration and solution through both kernel families (the persistent one runs the
    residual checks inside its single launch)."""
    cfg = mmot_inputs.CONFIGS["C2"]
    mus = mmot_inputs.make_marginals("C2", 0)
    h = mmot_inputs.grid_h(cfg.N)
    rep, g, marg, W = _run_gpu(mus, cfg.eta, cfg.iters, tol=cfg.tol, kernel=kernel)
    g_ref, t_ref, res_ref = osk.sinkhorn(mus, h, cfg.eta, cfg.iters, tol=cfg.tol, domain="log")
    assert rep["converged"] and rep["iters_done"] == t_ref, (rep, t_ref, res_ref)
    assert rep["residual"] == pytest.approx(res_ref, rel=1e-4)
    m_ref = osk.marginals(np.exp(g_ref), h, cfg.eta)
    for k in range(cfg.l):
        assert _l1rel(marg[k], m_ref[k]) <= 1e-10


def test_argument_errors():
    with pytest.raises(mm.MMOTError) as ei:
        mm.Context(3, 100, -1.0)
    assert ei.value.name == "MMOT_EINVAL"
    ctx = mm.Context(3, 100, 0.1)
    u = [torch.zeros(100, dtype=torch.float64, device=DEV) for _ in range(3)]
    with pytest.raises(mm.MMOTError) as ei:
        ctx.marginal(3, u)
    assert ei.value.name == "MMOT_EINVAL"
    with pytest.raises(mm.MMOTError) as ei:
        ctx.marginal(0, u[:2])
    assert ei.value.name == "MMOT_ESHAPE"
    ctx.close()


@pytest.mark.parametrize("N,eta", [(400, 1e-4), (12000, 1e-3)])
def test_overflow_reported_by_persistent_kernel(N, eta, monkeypatch):
    """Disjoint supports at small eta: J_k between the supports is below e^-708 relative to the
    chain scale (the cost of crossing the gap is 0.8 / eta), beyond what per-chain exponents of
    the scalings can absorb -- with the range fallback disabled the persistent kernel reports
    EOVERFLOW with the sweep, like the plain fp64 families, instead of returning garbage."""
    monkeypatch.setenv("MMOT_NO_STABLE", "1")
    x = np.arange(N) / (N - 1)
    mus = np.stack([(x < 0.3).astype(float), (x > 0.7).astype(float), np.ones(N)])
    mus /= mus.sum(axis=1, keepdims=True)
    with pytest.raises(mm.MMOTError) as ei:
        _run_gpu(mus, eta, 3, kernel="persistent")
    assert ei.value.name == "MMOT_EOVERFLOW"
    assert ei.value.report["fail_iter"] == 1
