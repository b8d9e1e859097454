"""Sharded device path at world > 1 on ONE GPU: virtual shards (mmot_create_sharded_virtual).

G contexts, one per rank, each driven by its own host thread on its own CUDA stream; the
collectives of the sharded path (all-gather of the whole-shard operators / restricted-scan affine
elements between up-sweep and down-sweep, all-reduce of residual, cost and data checks) run as
cross-stream event waits plus device copies (include/mmot.h).  So the shard-boundary seeding of the
scan, k_compose / k_rx_compose with REAL predecessors and successors, and the partial reductions
run exactly as on G GPUs, and the concatenated results must equal the fp64 CPU oracle
(oracle/regions.c, §4.2) at the north_star tolerance 1e-10.

Inputs are C4-shaped (box-filtered U[0,1] fields) at N = 2e5 with eta = 0.05, which
gives C4's h/eta = 1e-4 (the same per-edge weights w_a as the full C4 config).
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import regions, sinkhorn as osk  # noqa: E402

DEV = "cuda:0"
RTOL = 1e-10


def _run_ranks(G, fn):
    """Run fn(rank, group) on G threads (one per virtual rank); return the per-rank results."""
    group = mm.VirtualGroup(G)
    out, errs = [None] * G, []

    def body(r):
        try:
            with torch.cuda.stream(torch.cuda.Stream(device=DEV)):
                out[r] = fn(r, group)
        except BaseException as e:  # noqa: BLE001
            errs.append((r, e))

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in ts), "virtual ranks hung"
    group.close()
    if errs:
        raise errs[0][1]
    return out


def _slices(N, G):
    return [mm.shard_range(N, r, G) for r in range(G)]


def _rel_l1(a, b):
    return float(np.abs(a - b).sum() / np.abs(b).sum())


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("kernel,chunk", [("two_walk", 0), ("single_walk", 64)])
def test_vshard_marginal_and_cost(G, kernel, chunk):
    l, N, eta = 4, 200_000, 0.05
    h = mmot_inputs.grid_h(N)
    phis = mmot_inputs.random_positive(900 + G, l, N)
    sl = _slices(N, G)

    def rank(r, group):
        lo, hi = sl[r]
        ctx = mm.Context(l, N, eta, repr="linear", shard=(r, G, group), kernel=kernel, chunk=chunk)
        assert ctx.N == hi - lo and ctx.info["kernel"] == kernel
        u = [torch.from_numpy(np.ascontiguousarray(p[lo:hi])).to(DEV) for p in phis]
        ms = [ctx.marginal(k, u).cpu().numpy() for k in range(l)]
        W = ctx.cost(u)
        ctx.close()
        return ms, W

    res = _run_ranks(G, rank)
    w = regions.edge_weights(l, h, eta)
    for k in range(l):
        got = np.concatenate([res[r][0][k] for r in range(G)])
        want = phis[k] * regions.marginal_product(list(phis), k, w)
        assert np.max(np.abs(got - want) / want) <= RTOL, (G, kernel, k)
    W_ref = osk.cost(phis, h, eta)
    for r in range(G):
        assert abs(res[r][1] - W_ref) <= RTOL * abs(W_ref), (r, res[r][1], W_ref)


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("kernel,chunk,tol", [("two_walk", 0, 0.0), ("single_walk", 64, 0.0), ("single_walk", 64, 1e-300)])
def test_vshard_sinkhorn_lockstep(G, kernel, chunk, tol):
    """3 sweeps of the fused updates (single-walk: the restricted next-update scan, whose affine
    elements are exchanged between the ranks), then marginals, cost and residual vs the oracle."""
    l, N, eta, T = 4, 200_000, 0.05, 3
    h = mmot_inputs.grid_h(N)
    mus = mmot_inputs.c4_marginals(7, N, l)
    sl = _slices(N, G)

    def rank(r, group):
        lo, hi = sl[r]
        ctx = mm.Context(l, N, eta, repr="log", shard=(r, G, group), kernel=kernel, chunk=chunk, check_every=1)
        u = [torch.empty(hi - lo, dtype=torch.float64, device=DEV) for _ in range(l)]
        ctx.init_uniform(u)
        mu = [torch.from_numpy(np.ascontiguousarray(m[lo:hi])).to(DEV) for m in mus]
        rep = ctx.sinkhorn(mu, T, tol, u)
        ms = [ctx.marginal(k, u).cpu().numpy() for k in range(l)]
        W = ctx.cost(u)
        g = [x.cpu().numpy() for x in u]
        ctx.close()
        return rep, ms, W, g

    res = _run_ranks(G, rank)
    phis, _, res_ref = osk.sinkhorn(mus, h, eta, T, tol=tol, domain="plain")
    m_ref = osk.marginals(phis, h, eta)
    W_ref = osk.cost(phis, h, eta)
    for r in range(G):
        rep = res[r][0]
        assert rep["status"] == 0 and rep["iters_done"] == T, (r, rep)
        if tol > 0:
            assert rep["residual"] == pytest.approx(res_ref, rel=1e-9), (r, rep["residual"], res_ref)
        assert abs(res[r][2] - W_ref) <= RTOL * abs(W_ref)
    for k in range(l):
        got = np.concatenate([res[r][1][k] for r in range(G)])
        assert _rel_l1(got, m_ref[k]) <= RTOL, (G, kernel, k)
        g = np.concatenate([res[r][3][k] for r in range(G)])
        assert np.max(np.abs(g - np.log(phis[k]))) <= 1e-9


@pytest.mark.parametrize("G", [2, 4])
def test_vshard_collective_early_exit(G):
    """tol > 0: the ranks agree on the stop flag and leave the sweep loop after the same sweep as
    the oracle's stop rule (A7)."""
    l, N, eta, tol = 3, 20_000, 0.1, 1e-6
    h = mmot_inputs.grid_h(N)
    mus = mmot_inputs.c4_marginals(8, N, l, width=200)
    sl = _slices(N, G)
    _, t_ref, res_ref = osk.sinkhorn(mus, h, eta, 500, tol=tol, domain="plain", engine="subset")
    assert t_ref < 500 and t_ref % 8 != 0   # the stop falls between two polls of the flag

    def rank(r, group):
        lo, hi = sl[r]
        ctx = mm.Context(l, N, eta, repr="log", shard=(r, G, group), check_every=1)
        u = [torch.empty(hi - lo, dtype=torch.float64, device=DEV) for _ in range(l)]
        ctx.init_uniform(u)
        mu = [torch.from_numpy(np.ascontiguousarray(m[lo:hi])).to(DEV) for m in mus]
        rep = ctx.sinkhorn(mu, 500, tol, u)
        ctx.close()
        return rep

    reps = _run_ranks(G, rank)
    for rep in reps:
        assert rep["status"] == 0 and rep["converged"], rep
        assert rep["iters_done"] == t_ref, (rep, t_ref)
        assert rep["residual"] == pytest.approx(res_ref, rel=1e-6)


def test_vshard_zero_mass_on_one_shard_is_valid():
    """A marginal with all of its mass outside rank 0's chunk is valid (the zero-mass check uses the
    whole marginal); zero entries give phi = 0 (log phi = -inf) and no NaN."""
    G, l, N, eta, T = 2, 3, 20_000, 0.05, 3
    h = mmot_inputs.grid_h(N)
    mus = mmot_inputs.c4_marginals(9, N, l, width=200)
    lo1, _ = mm.shard_range(N, 1, G)
    mus[0, :lo1] = 0.0
    mus[0] /= mus[0].sum()
    sl = _slices(N, G)

    def rank(r, group):
        lo, hi = sl[r]
        ctx = mm.Context(l, N, eta, repr="linear", shard=(r, G, group), kernel="two_walk")
        u = [torch.full((hi - lo,), 1.0 / N, dtype=torch.float64, device=DEV) for _ in range(l)]
        mu = [torch.from_numpy(np.ascontiguousarray(m[lo:hi])).to(DEV) for m in mus]
        rep = ctx.sinkhorn(mu, T, 0.0, u)
        g = [x.cpu().numpy() for x in u]
        ctx.close()
        return rep, g

    res = _run_ranks(G, rank)
    phis, _, _ = osk.sinkhorn(mus, h, eta, T, domain="plain")
    for r in range(G):
        assert res[r][0]["status"] == 0, res[r][0]
    for k in range(l):
        got = np.concatenate([res[r][1][k] for r in range(G)])
        assert np.all(np.isfinite(got))
        assert np.max(np.abs(got - phis[k]) / np.maximum(phis[k], 1e-300)) <= 1e-10


def test_vshard_error_reported_by_every_rank():
    """NaN in one rank's chunk: every rank returns MMOT_ENONFINITE (status max-reduced) and no rank
    hangs in a collective."""
    G, l, N, eta = 4, 3, 20_000, 0.05
    mus = mmot_inputs.c4_marginals(10, N, l, width=200)
    lo3, _ = mm.shard_range(N, 3, G)
    mus[1, lo3 + 5] = np.nan
    sl = _slices(N, G)

    def rank(r, group):
        lo, hi = sl[r]
        ctx = mm.Context(l, N, eta, repr="log", shard=(r, G, group), check_every=1)
        u = [torch.empty(hi - lo, dtype=torch.float64, device=DEV) for _ in range(l)]
        ctx.init_uniform(u)
        mu = [torch.from_numpy(np.ascontiguousarray(m[lo:hi])).to(DEV) for m in mus]
        try:
            ctx.sinkhorn(mu, 20, 1e-12, u)
            name = "MMOT_OK"
        except mm.MMOTError as e:
            name = e.name
        ctx.close()
        return name

    names = _run_ranks(G, rank)
    assert names == ["MMOT_ENONFINITE"] * G, names


@pytest.mark.parametrize("G", [2, 4, 8])
def test_vshard_c4_full_size_matches_single_context(G):
    """The bench's multi-GPU C4 configuration (N = 1e8 sharded by grid chunks, AUTO kernels: exact
    chain tiling per shard, restricted-scan exchange from the second update on) on G virtual shards
    against the single-context solve of the same inputs (itself compared with the oracle at full
    size in test_gpu_single_walk.py): scalings to 1e-9, W to 1e-10, and the plan's last marginal
    equal to mu_l after the last update."""
    cfg = mmot_inputs.CONFIGS["C4"]
    l, N, eta, T = cfg.l, cfg.N, cfg.eta, 2
    mus = mmot_inputs.make_marginals("C4", 0)
    mu_d = [torch.from_numpy(np.ascontiguousarray(m)).to(DEV) for m in mus]
    ctx = mm.Context(l, N, eta)
    u0 = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u0)
    rep = ctx.sinkhorn(mu_d, T, 0.0, u0)
    assert rep["status"] == 0
    W0 = ctx.cost(u0)
    ctx.close()
    sl = _slices(N, G)

    def rank(r, group):
        lo, hi = sl[r]
        c = mm.Context(l, N, eta, shard=(r, G, group))
        u = [torch.empty(hi - lo, dtype=torch.float64, device=DEV) for _ in range(l)]
        c.init_uniform(u)
        rp = c.sinkhorn([m[lo:hi] for m in mu_d], T, 0.0, u)
        W = c.cost(u)
        m_last = c.marginal(l - 1, u)
        torch.cuda.synchronize()
        kern = c.info["kernel"]
        c.close()
        return rp, u, W, m_last, kern

    res = _run_ranks(G, rank)
    for r, (rp, u, W, m_last, kern) in enumerate(res):
        lo, hi = sl[r]
        assert rp["status"] == 0 and rp["iters_done"] == T
        assert abs(W - W0) <= 1e-10 * abs(W0), (r, W, W0)
        for q in range(l):
            ref = u0[q][lo:hi]
            d = torch.max(torch.abs(u[q] - ref) / torch.clamp(torch.abs(ref), min=1.0)).item()
            assert d <= 1e-9, (r, q, d, kern)
        dm = (torch.abs(m_last - mu_d[l - 1][lo:hi]).sum() / mu_d[l - 1][lo:hi].sum()).item()
        assert dm <= 1e-10, (r, dm)
    print(f"G={G}: shard kernels {[x[4] for x in res]}")
