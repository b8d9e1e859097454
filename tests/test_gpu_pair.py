"""GPU parity of the pair family (pair.cu: two threads per instance, no chain operators, mantissas
with one exponent per 8 grid points) against the fp64 CPU oracle.

The family runs batched Sinkhorn solves with a fixed sweep count once the batch reaches
MMOT_PAIR_MIN (default 4096; C5's 8192-instance tests in test_gpu_batched.py run on it).  Here
MMOT_PAIR_MIN=1 routes small batches through it: ragged blocks of 16 instances, odd N (the mirrored
right half one point shorter), N = 1 (an empty right half), per-instance eta down to 1e-3 (|log phi|
in the hundreds: the slab exponents carry the range).  Tolerances as test_gpu_batched.py (north_star
fp64): marginals 1e-10 L1-relative, log phi 1e-9; fp32 storage (MMOT_F32 contexts): 1e-5.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import regions, sinkhorn as osk  # noqa: E402

DEV = "cuda:0"


def _planes(arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).to(DEV) for a in arrs]


def _batch(l, N, B, seed):
    etas = list(np.geomspace(1e-3, 1e-1, B))
    mus = [np.stack([mmot_inputs.c2_marginals(seed + b, N, l)[q] for q in range(l)]) for b in range(B)]
    return etas, mus


def _solve(l, N, etas, mus, T, dtype="f64"):
    B = len(etas)
    md = [np.stack([mus[b][q] for b in range(B)]) for q in range(l)]
    if dtype == "f32":
        md = [m.astype(np.float32) for m in md]
    mu_d = _planes(md)
    ctx = mm.Context(l, N, etas, batch=B, dtype=dtype)
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(mu_d, T, 0.0, u)
    solves = ctx.pair_solves
    ctx.close()
    return rep, np.stack([x.cpu().numpy() for x in u]), solves


def _check(l, N, etas, mus, T, g, rtol_m, rtol_g, picks=None):
    h = mmot_inputs.grid_h(N)
    for b in (picks if picks is not None else range(len(etas))):
        g_ref, _, _ = osk.sinkhorn(mus[b], h, etas[b], T, domain="log", engine="subset")
        fin = np.isfinite(g_ref)
        gg = g[:, b, :]
        assert np.array_equal(np.isfinite(gg), fin), b
        assert np.max(np.abs(gg[fin] - g_ref[fin]) / np.maximum(1.0, np.abs(g_ref[fin]))) <= rtol_g, b
        lw = np.array([-(a * (l - a)) * h / etas[b] for a in range(l + 1)])
        for k in range(l):
            m_ref = np.exp(g_ref[k] + regions.marginal_product_log(list(g_ref), k, lw))
            m_got = np.exp(gg[k] + regions.marginal_product_log(list(gg), k, lw))
            err = np.abs(m_got - m_ref).sum() / np.abs(m_ref).sum()
            assert err <= rtol_m, (b, k, err)


@pytest.mark.parametrize("l,N,B,T", [(2, 64, 5, 10), (3, 257, 37, 8), (4, 1000, 19, 6), (5, 96, 33, 5),
                                     (5, 4096, 17, 3), (3, 7, 16, 12), (4, 1, 3, 4), (3, 2, 3, 4)])
def test_pair_sinkhorn_lockstep(monkeypatch, l, N, B, T):
    monkeypatch.setenv("MMOT_PAIR_MIN", "1")
    etas, mus = _batch(l, N, B, 300 + N)
    rep, g, solves = _solve(l, N, etas, mus, T)
    assert solves == 1
    assert rep["status"] == 0 and rep["iters_done"] == T
    picks = sorted({0, B // 2, B - 1, min(B - 1, 16)})
    _check(l, N, etas, mus, T, g, 1e-10, 1e-9, picks)


def test_pair_matches_persistent_kernel(monkeypatch):
    """Whole batch, pair family vs the one-warp-per-instance kernel (both fp64): same iterates."""
    l, N, B, T = 5, 512, 64, 20
    etas, mus = _batch(l, N, B, 900)
    monkeypatch.setenv("MMOT_PAIR_MIN", "1")
    _, g_pair, s1 = _solve(l, N, etas, mus, T)
    monkeypatch.setenv("MMOT_NO_PAIR", "1")
    _, g_ref, s2 = _solve(l, N, etas, mus, T)
    assert s1 == 1 and s2 == 0
    fin = np.isfinite(g_ref)
    assert np.array_equal(np.isfinite(g_pair), fin)
    assert np.max(np.abs(g_pair[fin] - g_ref[fin]) / np.maximum(1.0, np.abs(g_ref[fin]))) <= 1e-9


def test_pair_f32_storage(monkeypatch):
    """MMOT_F32 context (default): fp32 mantissas and marginals in the pair layout, fp64
    arithmetic; the fp32 bar of north_star (1e-4) with margin."""
    monkeypatch.setenv("MMOT_PAIR_MIN", "1")
    l, N, B, T = 4, 500, 20, 10
    etas, mus = _batch(l, N, B, 700)
    mus = [m.astype(np.float32).astype(np.float64) for m in mus]   # the values the context sees
    rep, g, solves = _solve(l, N, etas, mus, T, dtype="f32")
    assert solves == 1 and rep["status"] == 0
    _check(l, N, etas, mus, T, g, 1e-5, 1e-5, [0, 9, 19])


def test_pair_zero_runs_and_linear_repr(monkeypatch):
    """Marginals with zero runs (whole slabs and a half of the grid empty): the zero slabs take a
    neighbour's exponent; LINEAR representation in and out."""
    monkeypatch.setenv("MMOT_PAIR_MIN", "1")
    l, N, B, T = 3, 200, 4, 8
    etas = [0.05, 0.02, 0.1, 0.03]
    rng = np.random.default_rng(5)
    mus = []
    for b in range(B):
        m = rng.uniform(0.1, 1.0, (l, N))
        m[0, 10:40] = 0.0
        m[1, 100:] = 0.0 if b % 2 else m[1, 100:]
        m[2, :17] = 0.0
        mus.append(m / m.sum(axis=1, keepdims=True))
    md = _planes([np.stack([mus[b][q] for b in range(B)]) for q in range(l)])
    ctx = mm.Context(l, N, etas, batch=B, repr="linear")
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(md, T, 0.0, u)
    assert ctx.pair_solves == 1 and rep["status"] == 0
    phis = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    h = mmot_inputs.grid_h(N)
    for b in range(B):
        p_ref, _, _ = osk.sinkhorn(mus[b], h, etas[b], T)
        assert np.array_equal(phis[:, b, :] == 0.0, p_ref == 0.0), b
        nz = p_ref > 0
        assert np.max(np.abs(phis[:, b, :][nz] - p_ref[nz]) / p_ref[nz]) <= 1e-9, b


def test_pair_tol_runs_on_persistent_kernel(monkeypatch):
    """tol > 0 needs the residual: the persistent kernel runs it (the pair family is fixed-sweep)."""
    monkeypatch.setenv("MMOT_PAIR_MIN", "1")
    l, N, B = 3, 100, 4
    etas, mus = _batch(l, N, B, 50)
    md = _planes([np.stack([mus[b][q] for b in range(B)]) for q in range(l)])
    ctx = mm.Context(l, N, etas, batch=B)
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    ctx.sinkhorn(md, 50, 1e-6, u)
    assert ctx.pair_solves == 0
    ctx.init_uniform(u)
    ctx.sinkhorn(md, 5, 0.0, u)
    assert ctx.pair_solves == 1
    ctx.close()


def _solve_f32c(l, N, etas, mus, T):
    B = len(etas)
    md = _planes([np.stack([mus[b][q] for b in range(B)]).astype(np.float32) for q in range(l)])
    ctx = mm.Context(l, N, etas, batch=B, dtype="f32")
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(md, T, 0.0, u)
    counts = (ctx.pair_solves, ctx.pair_f32_solves, ctx.stable_fallbacks, ctx.pair_redo)
    ctx.close()
    return rep, np.stack([x.cpu().numpy() for x in u]), counts


@pytest.mark.parametrize("l,N,B,T,redo", [(5, 4096, 17, 30, False), (4, 1000, 19, 40, False),
                                          (3, 257, 37, 50, False), (2, 64, 5, 20, None), (5, 96, 33, 60, None),
                                          (3, 7, 16, 12, None)])
def test_pair_f32_arithmetic(monkeypatch, l, N, B, T, redo):
    """MMOT_F32 context (default): fp32 storage AND fp32 arithmetic (walks, combine; the division in
    fp64), the states kept relative to the 8-point slab exponents.  Against the fp64
    oracle run on the fp32-rounded marginals: north_star's fp32 bar, 1e-4 L1-relative per marginal,
    over eta in [1e-3, 1e-1] and tens of sweeps.  Instances whose states leave the fp32 range (coarse
    grids at eta = 1e-3, h/eta ~ 10: a slab spans ~2^120 of phi) are redone in fp64 with the same
    results; the C5-like grids (redo=False) stay in fp32."""
    monkeypatch.setenv("MMOT_PAIR_MIN", "1")
    etas, mus = _batch(l, N, B, 1100 + N)
    mus = [m.astype(np.float32).astype(np.float64) for m in mus]   # the values the context sees
    rep, g, (s, s32, fb, nredo) = _solve_f32c(l, N, etas, mus, T)
    assert s == 1 and s32 == 1 and rep["status"] == 0 and rep["iters_done"] == T
    assert fb == 0  # nothing reached the stabilised family
    if redo is not None:
        assert (nredo > 0) == redo, nredo
    picks = sorted({0, B // 2, B - 1, min(B - 1, 16)})
    _check(l, N, etas, mus, T, g, 1e-4, 1e-3, picks)


def test_pair_f32_arithmetic_zero_runs(monkeypatch):
    """fp32 arithmetic with zero runs in the marginals (zero slabs take a neighbour's exponent)."""
    monkeypatch.setenv("MMOT_PAIR_MIN", "1")
    l, N, B, T = 4, 300, 6, 15
    etas = list(np.geomspace(2e-3, 5e-2, B))
    rng = np.random.default_rng(17)
    mus = []
    for b in range(B):
        m = rng.uniform(0.1, 1.0, (l, N))
        m[0, 20:60] = 0.0
        m[2, 150:] = 0.0 if b % 2 else m[2, 150:]
        m[3, :9] = 0.0
        m = (m / m.sum(axis=1, keepdims=True)).astype(np.float32).astype(np.float64)
        mus.append(m)
    rep, g, (s, s32, fb, nredo) = _solve_f32c(l, N, etas, mus, T)
    assert s == 1 and s32 == 1 and rep["status"] == 0 and fb == 0
    _check(l, N, etas, mus, T, g, 1e-4, 1e-3, list(range(B)))
