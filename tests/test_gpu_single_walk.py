"""GPU parity of the single-walk kernels (k_sw_apply: suffix states walked forward through the
inverse recurrence step, one extended operator walk for both scan directions) against the fp64
CPU oracle (oracle/regions.c, §4.2 region chains).

The single-walk family is selected automatically for large N at small h/eta (C4); here it is
forced (kernel="single_walk") at small sizes inside its stability bound
P * max_a a(l-a) * h/eta <= 1, with chain lengths that leave ragged tails,
chains shorter than a slab, and thousands of chains (3-4 scan levels).
Tolerance: north_star fp64, 1e-10 relative (elementwise for products, L1 for Sinkhorn).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import regions, sinkhorn as osk  # noqa: E402

DEV = "cuda:0"
RTOL = 1e-10


def _dev(vs):
    return [torch.from_numpy(np.ascontiguousarray(v)).to(DEV) for v in vs]


def _emax(l):
    return (l // 2) * ((l + 1) // 2)


def _eta_for(l, N, chunk, frac=0.9):
    """Largest h/eta inside the stability bound for this chain length (times frac)."""
    h = mmot_inputs.grid_h(N)
    return h / (frac / (chunk * _emax(l)))


def _oracle_marginals(phis, h, eta):
    l = len(phis)
    w = regions.edge_weights(l, h, eta)
    return [phis[k] * regions.marginal_product(list(phis), k, w) for k in range(l)]


def _rel(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


@pytest.mark.parametrize("l", [2, 3, 4, 5])
@pytest.mark.parametrize("N,chunk", [(1, 8), (7, 8), (64, 8), (1000, 13), (4097, 64), (20000, 8), (20001, 100)])
def test_single_walk_marginal_parity(l, N, chunk):
    phis = mmot_inputs.random_positive(4000 + 10 * l + N, l, N)
    h = mmot_inputs.grid_h(N)
    eta = _eta_for(l, N, chunk)
    ctx = mm.Context(l, N, eta, repr="linear", chunk=chunk, kernel="single_walk")
    assert ctx.info["kernel"] == "single_walk"
    u = _dev(phis)
    got = [ctx.marginal(k, u).cpu().numpy() for k in range(l)]
    fb = ctx.fallbacks
    ctx.close()
    want = _oracle_marginals(phis, h, eta)
    for k in range(l):
        assert _rel(got[k], want[k]) <= RTOL, (l, N, chunk, k)
    assert fb == 0, fb   # U[0.1, 1] scalings: the single-walk states stay accurate


@pytest.mark.parametrize("l", [3, 4])
def test_single_walk_cost_parity(l):
    N, chunk = 5000, 40
    h = mmot_inputs.grid_h(N)
    eta = _eta_for(l, N, chunk)
    phis = mmot_inputs.random_positive(500 + l, l, N)
    ctx = mm.Context(l, N, eta, repr="linear", chunk=chunk, kernel="single_walk")
    W = ctx.cost(_dev(phis))
    ctx.close()
    w = regions.edge_weights(l, h, eta)
    _, jh = regions.marginal_product(list(phis), l - 1, w, want_hat=True)
    W_ref = h * float(np.dot(phis[l - 1], jh))
    assert abs(W - W_ref) <= RTOL * abs(W_ref)


@pytest.mark.parametrize("l,N,chunk,T", [(2, 3000, 16, 6), (3, 5000, 24, 5), (4, 20000, 64, 4), (5, 3000, 16, 3)])
def test_single_walk_sinkhorn_lockstep(l, N, chunk, T):
    """Fused updates: phi_k <- mu_k / J_k with the next update's operators built in the same walk."""
    h = mmot_inputs.grid_h(N)
    eta = _eta_for(l, N, chunk)
    mus = np.stack(mmot_inputs.random_marginals(600 + l, l, N))
    ctx = mm.Context(l, N, eta, repr="log", chunk=chunk, kernel="single_walk")
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_dev(mus), T, 0.0, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    marg = np.stack([ctx.marginal(k, u).cpu().numpy() for k in range(l)])
    g = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    g_ref, _, _ = osk.sinkhorn(mus, h, eta, T, domain="plain")
    g_ref = np.log(g_ref)
    m_ref = osk.marginals(np.exp(g_ref), h, eta)
    for k in range(l):
        assert np.abs(marg[k] - m_ref[k]).sum() / np.abs(m_ref[k]).sum() <= RTOL, k
    assert np.max(np.abs(g - g_ref)) <= 1e-9


def _zero_runs(x, rng, runs, length):
    x = x.copy()
    for _ in range(runs):
        a = int(rng.integers(0, len(x) - length))
        x[a:a + length] = 0.0
    return x


@pytest.mark.parametrize("l", [3, 4, 5])
def test_single_walk_zero_runs_sinkhorn_lockstep(l):
    """Marginals with zero runs (several runs longer than a chain, and a zero tail): the scalings of
    those marginals are exactly 0 there, so the inverse step subtracts placed terms
    that vanish on the rest of the chain.  Lockstep with the oracle at 1e-10 and no fallback (the
    walked states stay accurate: the stability bound also bounds the growth across a run)."""
    N, chunk, T = 20000, 64, 4
    h = mmot_inputs.grid_h(N)
    eta = _eta_for(l, N, chunk)
    rng = np.random.default_rng(4242 + l)
    mus = np.stack(mmot_inputs.random_marginals(610 + l, l, N))
    for q in range(l):
        mus[q] = _zero_runs(mus[q], rng, 4, 3 * chunk + 5)
    mus[0, N - 700:] = 0.0
    mus /= mus.sum(axis=1, keepdims=True)
    ctx = mm.Context(l, N, eta, repr="linear", chunk=chunk, kernel="single_walk")
    u = [torch.full((N,), 1.0 / N, dtype=torch.float64, device=DEV) for _ in range(l)]
    rep = ctx.sinkhorn(_dev(mus), T, 0.0, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    marg = np.stack([ctx.marginal(k, u).cpu().numpy() for k in range(l)])
    phi = np.stack([x.cpu().numpy() for x in u])
    fb = ctx.fallbacks
    ctx.close()
    phi_ref, _, _ = osk.sinkhorn(mus, h, eta, T, domain="plain")
    m_ref = osk.marginals(phi_ref, h, eta)
    for k in range(l):
        assert np.abs(marg[k] - m_ref[k]).sum() / np.abs(m_ref[k]).sum() <= RTOL, k
        assert np.array_equal(phi[k] == 0.0, phi_ref[k] == 0.0), k
        nz = phi_ref[k] > 0
        assert np.max(np.abs(phi[k][nz] - phi_ref[k][nz]) / phi_ref[k][nz]) <= 1e-9, k
    assert fb == 0, fb


@pytest.mark.parametrize("l", [3, 4])
def test_single_walk_huge_dynamic_range(l):
    """Scalings spanning 1e+-50 between neighbouring points (i.i.d. log-uniform): single-walk parity
    at 1e-10 (the suffix states stay dominated by the largest values further right, so the
    subtractions stay well conditioned; the guard may or may not redo the call)."""
    N, chunk = 5000, 40
    h = mmot_inputs.grid_h(N)
    eta = _eta_for(l, N, chunk)
    rng = np.random.default_rng(77 + l)
    phis = 10.0 ** rng.uniform(-50, 50, (l, N))
    ctx = mm.Context(l, N, eta, repr="linear", chunk=chunk, kernel="single_walk")
    u = _dev(phis)
    got = [ctx.marginal(k, u).cpu().numpy() for k in range(l)]
    W = ctx.cost(u)
    ctx.close()
    want = _oracle_marginals(phis, h, eta)
    for k in range(l):
        assert _rel(got[k], want[k]) <= RTOL, k
    w = regions.edge_weights(l, h, eta)
    _, jh = regions.marginal_product(list(phis), l - 1, w, want_hat=True)
    W_ref = h * float(np.dot(phis[l - 1], jh))
    assert abs(W - W_ref) <= RTOL * abs(W_ref)


def _steep_tail(N, n_tail, decades_per_point):
    """1 on the grid, then a steep decreasing ramp over the last n_tail points."""
    v = np.ones(N)
    v[N - n_tail:] = 10.0 ** (-decades_per_point * np.arange(1, n_tail + 1))
    return v


@pytest.mark.parametrize("l", [3, 4])
def test_single_walk_steep_ramp(l):
    """A scaling dropping by 2.5 decades per point over the grid's last 110 points: every walked
    suffix state there is a difference of nearly equal numbers, but the lost digits sit in suffix
    components the combine weights by prefix states that the same (larger, earlier) values dominate,
    so J stays accurate: parity at 1e-10 with no fallback."""
    N, chunk = 5000, 40
    h = mmot_inputs.grid_h(N)
    eta = _eta_for(l, N, chunk)
    rng = np.random.default_rng(91 + l)
    phis = rng.uniform(0.1, 1.0, (l, N))
    phis[0] *= _steep_tail(N, 110, 2.5)
    ctx = mm.Context(l, N, eta, repr="linear", chunk=chunk, kernel="single_walk")
    got = [ctx.marginal(k, _dev(phis)).cpu().numpy() for k in range(l)]
    fb = ctx.fallbacks
    ctx.close()
    want = _oracle_marginals(phis, h, eta)
    for k in range(l):
        assert _rel(got[k], want[k]) <= RTOL, k
    assert fb == 0, fb


@pytest.mark.parametrize("l", [3, 4])
def test_single_walk_guard_trips_outside_stability_bound(l):
    """Explicit single-walk far outside its stability bound (P max_a a(l-a) h/eta = 40: the inverse
    step amplifies rounding by up to e^40 across a chain): the precision guard (walked end state vs
    the next chain's exact carry, weighted through the combine) trips and every call is redone on the
    two-walk family -- products, W and a Sinkhorn solve still match the oracle at 1e-10."""
    N, chunk = 5000, 40
    h = mmot_inputs.grid_h(N)
    eta = _eta_for(l, N, chunk, frac=40.0)
    rng = np.random.default_rng(93 + l)
    phis = rng.uniform(0.1, 1.0, (l, N))
    ctx = mm.Context(l, N, eta, repr="linear", chunk=chunk, kernel="single_walk")
    u = _dev(phis)
    got = [ctx.marginal(k, u).cpu().numpy() for k in range(l)]
    assert ctx.fallbacks == l
    W = ctx.cost(u)
    assert ctx.fallbacks == l + 1
    want = _oracle_marginals(phis, h, eta)
    for k in range(l):
        assert _rel(got[k], want[k]) <= RTOL, k
    w = regions.edge_weights(l, h, eta)
    _, jh = regions.marginal_product(list(phis), l - 1, w, want_hat=True)
    W_ref = h * float(np.dot(phis[l - 1], jh))
    assert abs(W - W_ref) <= RTOL * abs(W_ref)
    mus = np.stack(mmot_inputs.random_marginals(95 + l, l, N))
    v = [torch.full((N,), 1.0 / N, dtype=torch.float64, device=DEV) for _ in range(l)]
    rep = ctx.sinkhorn(_dev(mus), 3, 0.0, v)
    assert rep["status"] == 0 and ctx.fallbacks == l + 2
    phi = np.stack([x.cpu().numpy() for x in v])
    ctx.close()
    phi_ref, _, _ = osk.sinkhorn(mus, h, eta, 3, domain="plain")
    assert np.max(np.abs(phi - phi_ref) / phi_ref) <= 1e-9


@pytest.mark.parametrize("l", [3, 4])
def test_single_walk_smooth_large_range(l):
    """log phi a smooth wave of amplitude 115 (phi spanning 1e+-50 across the grid, smoothly):
    single-walk parity at 1e-10 (with or without the guard's fallback)."""
    N, chunk = 20000, 64
    h = mmot_inputs.grid_h(N)
    eta = _eta_for(l, N, chunk)
    x = np.arange(N) / (N - 1)
    phis = np.stack([np.exp(115.0 * np.sin(2 * np.pi * (3 + q) * x + q)) for q in range(l)])
    ctx = mm.Context(l, N, eta, repr="linear", chunk=chunk, kernel="single_walk")
    u = _dev(phis)
    got = [ctx.marginal(k, u).cpu().numpy() for k in range(l)]
    ctx.close()
    want = _oracle_marginals(phis, h, eta)
    for k in range(l):
        assert _rel(got[k], want[k]) <= RTOL, k


def test_auto_selects_single_walk_for_c4_shape():
    cfg = mmot_inputs.CONFIGS["C4"]
    ctx = mm.Context(cfg.l, cfg.N, cfg.eta)
    info = ctx.info
    ctx.close()
    h = mmot_inputs.grid_h(cfg.N)
    assert info["kernel"] == "single_walk"
    assert info["chain_len"] * _emax(cfg.l) * h / cfg.eta <= 1.0
    small = mm.Context(4, 1000, 0.01)
    assert small.info["kernel"] == "persistent"      # small instances: one warp, all sweeps per launch
    small.close()
    mid = mm.Context(4, 20000, 0.01)
    assert mid.info["kernel"] == "two_walk"
    mid.close()


@pytest.mark.slow
def test_c4_full_size_sweeps_match_two_walk_and_fix_last_marginal():
    """C4 at its full size (l=4, N=1e8, eta=1e-4) through mmot_sinkhorn in the bench's launch
    configuration (single-walk, restricted next-update scan), 2 sweeps, checked (a) against the
    two-walk family, an independent kernel path, on every element, and (b) by the property that
    holds at any size: the sweep's last update makes marginal l-1 exact, m_{l-1} = mu_{l-1}
    (P:1029-1035), with m_{l-1} from the product path verified by test_marginal_parity_c4_full_size."""
    cfg = mmot_inputs.CONFIGS["C4"]
    l, N, eta, T = cfg.l, cfg.N, cfg.eta, 2
    mus = mmot_inputs.make_marginals("C4", 0)
    mu_d = _dev(mus)
    del mus
    g = {}
    for fam in ("auto", "two_walk"):
        ctx = mm.Context(l, N, eta, repr="log", kernel=fam)
        if fam == "auto":
            assert ctx.info["kernel"] == "single_walk"
        u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
        ctx.init_uniform(u)
        rep = ctx.sinkhorn(mu_d, T, 0.0, u)
        assert rep["status"] == 0 and rep["iters_done"] == T
        if fam == "auto":
            m_last = ctx.marginal(l - 1, u)
            rel = float((m_last - mu_d[l - 1]).abs().sum() / mu_d[l - 1].abs().sum())
            assert rel <= RTOL, rel
            del m_last
        g[fam] = u
        ctx.close()
    for k in range(l):
        d = float((g["auto"][k] - g["two_walk"][k]).abs().max())
        assert d <= 1e-9, (k, d)


@pytest.mark.slow
def test_c4_full_size_sweeps_match_oracle():
    """C4 at its full size (l=4, N=1e8, eta=1e-4) through mmot_sinkhorn in exactly the bench's
    launch configuration (auto: single-walk, restricted next-update scan, 4 scan levels), 2 sweeps
    from the paper's init, then all l marginals and W through the library -- each
    compared with the fp64 CPU oracle (oracle/regions.c region chains, 2 plain Gauss-Seidel sweeps,
    P:1029-1035) on every element: 1e-10 L1-relative per marginal, 1e-10 relative for W, and
    log phi to 1e-9.  The oracle takes ~3-4 min on the host (8 sequential products, then the l
    marginals and the cost product on parallel threads)."""
    import concurrent.futures as cf
    cfg = mmot_inputs.CONFIGS["C4"]
    l, N, eta, T = cfg.l, cfg.N, cfg.eta, 2
    h = mmot_inputs.grid_h(N)
    mus = mmot_inputs.make_marginals("C4", 0)
    mu_d = _dev(mus)
    ctx = mm.Context(l, N, eta, repr="log")
    info = ctx.info
    assert info["kernel"] == "single_walk"
    u = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(mu_d, T, 0.0, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    del mu_d
    m_gpu = [ctx.marginal(k, u).cpu().numpy() for k in range(l)]
    W_gpu = ctx.cost(u)
    g_gpu = [x.cpu().numpy() for x in u]
    assert ctx.fallbacks == 0   # the precision guard held: these are single-walk results
    ctx.close()
    del u
    torch.cuda.empty_cache()
    # oracle: plain fp64 Gauss-Seidel sweeps (C4 stays representable)
    w = regions.edge_weights(l, h, eta)
    phis = [np.full(N, 1.0 / N) for _ in range(l)]
    for _ in range(T):
        for k in range(l):
            phis[k] = mus[k] / regions.marginal_product(phis, k, w)
    for k in range(l):
        assert np.max(np.abs(g_gpu[k] - np.log(phis[k]))) <= 1e-9, k
    del g_gpu
    with cf.ThreadPoolExecutor(max_workers=l + 1) as ex:   # ctypes releases the GIL
        fut = [ex.submit(regions.marginal_product, phis, k, w) for k in range(l)]
        fut_c = ex.submit(regions.marginal_product, phis, l - 1, w, True)
        for k in range(l):
            m_ref = phis[k] * fut[k].result()
            assert np.abs(m_gpu[k] - m_ref).sum() / np.abs(m_ref).sum() <= RTOL, k
            del m_ref
        _, jh = fut_c.result()
    W_ref = h * float(np.dot(phis[l - 1], jh))
    assert abs(W_gpu - W_ref) <= RTOL * abs(W_ref), (W_gpu, W_ref)
