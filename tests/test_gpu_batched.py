"""GPU parity of batched contexts (mmot_create_batched: one warp per instance, per-chain
exponents, persistent Sinkhorn) against the fp64 CPU oracle (oracle/regions.c, §4.2 region
chains; log-domain chains where linear fp64 overflows).

Tolerance (north_star fp64): 1e-10 relative -- elementwise for single products, L1-relative
per marginal for Sinkhorn, relative for W.  Instances are independent: every instance of a
batch is compared on its own (different eta per instance, as in BASELINE C5).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402
from oracle import regions, sinkhorn as osk  # noqa: E402

DEV = "cuda:0"
RTOL = 1e-10


def _planes(arrs):
    """list over q of [B][N] arrays -> list of contiguous device tensors."""
    return [torch.from_numpy(np.ascontiguousarray(a)).to(DEV) for a in arrs]


def _rel(a, b):
    return float(np.max(np.abs(a - b) / np.abs(b)))


@pytest.mark.parametrize("l", [2, 3, 4, 5])
@pytest.mark.parametrize("N", [1, 7, 64, 257, 1000])
def test_batched_marginal_parity(l, N):
    B = 3
    etas = [0.5, 0.02, 0.003]
    h = mmot_inputs.grid_h(N)
    phis = [mmot_inputs.random_positive(7000 + 100 * l + N + b, l, N) for b in range(B)]
    u = _planes([np.stack([np.log(phis[b][q]) for b in range(B)]) for q in range(l)])
    ctx = mm.Context(l, N, etas, batch=B)
    for k in range(l):
        got = ctx.marginal(k, u).cpu().numpy()
        for b in range(B):
            w = regions.edge_weights(l, h, etas[b])
            want = phis[b][k] * regions.marginal_product(list(phis[b]), k, w)
            assert _rel(got[b], want) <= RTOL, (l, N, k, b)
    ctx.close()


def test_batched_marginal_huge_dynamic_range():
    """Gauge offsets of +-1400 in log phi (beyond fp64's e^709; the C5 runs at eta = 1e-3
    drift to |log phi| ~ 1.8e3): sum_q c_q = 0 leaves every plan entry and
    marginal unchanged (A16), so the products must equal the plain oracle on the offset-free
    scalings; the per-chain exponents keep every intermediate representable."""
    l, N, B = 4, 600, 2
    etas = [1e-3, 0.05]
    h = mmot_inputs.grid_h(N)
    offs = np.array([1400.0, -1400.0, 900.0, -900.0])
    phis = [mmot_inputs.random_positive(8800 + b, l, N) for b in range(B)]
    u = _planes([np.stack([np.log(phis[b][q]) + offs[q] for b in range(B)]) for q in range(l)])
    ctx = mm.Context(l, N, etas, batch=B)
    for k in range(l):
        got = ctx.marginal(k, u).cpu().numpy()
        for b in range(B):
            w = regions.edge_weights(l, h, etas[b])
            want = phis[b][k] * regions.marginal_product(list(phis[b]), k, w)
            assert _rel(got[b], want) <= RTOL, (k, b)
    ctx.close()


@pytest.mark.parametrize("l,N,T", [(3, 64, 20), (4, 300, 10), (5, 256, 6)])
def test_batched_sinkhorn_lockstep(l, N, T):
    """Per-instance eta from 1e-3 to 1e-1; the oracle runs the log-domain driver."""
    etas = [1e-3, 1e-2, 1e-1]
    B = len(etas)
    h = mmot_inputs.grid_h(N)
    mus = [np.stack([mmot_inputs.c2_marginals(b, N, l)[q] for q in range(l)]) for b in range(B)]
    mu_d = _planes([np.stack([mus[b][q] for b in range(B)]) for q in range(l)])
    ctx = mm.Context(l, N, etas, batch=B)
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(mu_d, T, 0.0, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    marg = [ctx.marginal(k, u).cpu().numpy() for k in range(l)]
    g = np.stack([x.cpu().numpy() for x in u])  # [l][B][N]
    ctx.close()
    for b in range(B):
        g_ref, _, _ = osk.sinkhorn(mus[b], h, etas[b], T, domain="log")
        lw = np.array([-(a * (l - a)) * h / etas[b] for a in range(l + 1)])
        for k in range(l):
            m_ref = np.exp(g_ref[k] + regions.marginal_product_log(list(g_ref), k, lw))
            err = np.abs(marg[k][b] - m_ref).sum() / np.abs(m_ref).sum()
            assert err <= RTOL, (b, k, err)
        gg = g[:, b, :]
        fin = np.isfinite(g_ref)
        assert np.max(np.abs(gg[fin] - g_ref[fin]) / np.maximum(1.0, np.abs(g_ref[fin]))) <= 1e-9


def test_batched_cost_parity():
    l, N = 4, 500
    etas = [0.05, 0.02, 0.1]
    B = len(etas)
    h = mmot_inputs.grid_h(N)
    phis = [mmot_inputs.random_positive(9100 + b, l, N) for b in range(B)]
    u = _planes([np.stack([np.log(phis[b][q]) for b in range(B)]) for q in range(l)])
    ctx = mm.Context(l, N, etas, batch=B)
    W = ctx.cost(u)
    ctx.close()
    for b in range(B):
        W_ref = osk.cost(phis[b], h, etas[b])
        assert abs(W[b] - W_ref) <= RTOL * abs(W_ref), (b, W[b], W_ref)


def test_batched_c5_full_batch_sampled_instances():
    """C5 at its full size and in the bench's launch configuration (8192 instances of l=5, N=4096,
    per-instance eta, 3-component mixtures); three sampled instances (smallest, median and largest
    eta) checked against the log-domain oracle after 3 sweeps: log phi and the marginals."""
    cfg = mmot_inputs.CONFIGS["C5"]
    l, N, B, T = cfg.l, cfg.N, cfg.batch, 3
    etas = mmot_inputs.c5_etas(B)
    mus_all = mmot_inputs.c5_batch_marginals(0, B, N, l)          # [l][B][N]
    mu_d = [torch.from_numpy(mus_all[q]).to(DEV) for q in range(l)]
    ctx = mm.Context(l, N, [float(e) for e in etas], batch=B)
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(mu_d, T, 0.0, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    assert ctx.pair_solves == 1
    picks = [int(np.argmin(etas)), int(np.argsort(etas)[B // 2]), int(np.argmax(etas))]
    g = np.stack([x[picks].cpu().numpy() for x in u])               # [l][3][N]
    marg = [ctx.marginal(k, u)[picks].cpu().numpy() for k in range(l)]
    ctx.close()
    h = mmot_inputs.grid_h(N)
    for j, b in enumerate(picks):
        g_ref, _, _ = osk.sinkhorn(mus_all[:, b, :], h, float(etas[b]), T, domain="log")
        fin = np.isfinite(g_ref)
        assert np.max(np.abs(g[:, j, :][fin] - g_ref[fin]) / np.maximum(1.0, np.abs(g_ref[fin]))) <= 1e-9, b
        lw = np.array([-(a * (l - a)) * h / float(etas[b]) for a in range(l + 1)])
        for k in range(l):
            m_ref = np.exp(g_ref[k] + regions.marginal_product_log(list(g_ref), k, lw))
            assert np.abs(marg[k][j] - m_ref).sum() / np.abs(m_ref).sum() <= 1e-10, (b, k)


def test_batched_argument_errors():
    with pytest.raises(mm.MMOTError) as e:
        mm.Context(4, 100, [0.1, -1.0], batch=2)
    assert e.value.name == "MMOT_EINVAL"
    with pytest.raises(mm.MMOTError) as e:
        mm.Context(6, 100, [0.1], batch=1, kernel="persistent")  # l = 6 batches: stabilised family only
    assert e.value.name == "MMOT_EUNSUPPORTED"
    ctx = mm.Context(6, 100, [0.1], batch=1)
    assert ctx.info["kernel"] == "stable"
    ctx.close()



def test_batched_tolerance_per_instance():
    """Each instance stops at its own first residual <= tol, checked inside the launch."""
    l, N = 3, 200
    etas = [0.05, 0.02]
    B = 2
    h = mmot_inputs.grid_h(N)
    mus = [np.stack([mmot_inputs.c2_marginals(b, N, l)[q] for q in range(l)]) for b in range(B)]
    ctx = mm.Context(l, N, etas, batch=B, check_every=1)
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(_planes([np.stack([mus[b][q] for b in range(B)]) for q in range(l)]), 500, 1e-8, u)
    g = np.stack([x.cpu().numpy() for x in u])
    ctx.close()
    t_refs = []
    for b in range(B):
        g_ref, t_ref, res_ref = osk.sinkhorn(mus[b], h, etas[b], 500, tol=1e-8, domain="log")
        t_refs.append(t_ref)
        assert np.max(np.abs(g[:, b, :] - g_ref)) <= 1e-8, b
    assert rep["converged"] and rep["iters_done"] == max(t_refs)


@pytest.mark.parametrize("bad,code", [("nan", "MMOT_ENONFINITE"), ("neg", "MMOT_ENEGMASS"), ("zero", "MMOT_EZEROMASS")])
def test_batched_data_errors_per_instance(bad, code):
    """Input errors in ONE instance of a batch are reported: a zero-mass marginal of a single
    instance is EZEROMASS even though the batch as a whole has mass."""
    l, N, B = 4, 300, 5
    mus = np.stack([mmot_inputs.c2_marginals(b, N, l) for b in range(B)])  # [B][l][N]
    if bad == "nan":
        mus[3, 1, 17] = np.nan
    elif bad == "neg":
        mus[1, 2, 40] = -1e-6
    else:
        mus[2, 0, :] = 0.0
    ctx = mm.Context(l, N, [0.05] * B, batch=B)
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    with pytest.raises(mm.MMOTError) as ei:
        ctx.sinkhorn(_planes([mus[:, q, :] for q in range(l)]), 3, 0.0, u)
    ctx.close()
    assert ei.value.name == code


@pytest.mark.slow
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_batched_c5_full_run_stratified_instances(dtype):
    """C5 as the bench runs it: the full batch (8192 x (l=5, N=4096), per-instance eta ~ logU[1e-3,
    1e-1]) for the full T = 300 sweeps, then 8 stratified instances -- the median-eta instance of
    each of 8 equal log-eta strata -- against the log-domain oracle (region chains, P:1062-1125,
    in a pure log domain: Remark 1's purpose; O4 products), in parallel on the host cores:
    marginals to 1e-10 L1-relative, W to 1e-10, log phi to 1e-9 relative.  This covers the lazy
    chain-exponent renormalisation at |log phi| ~ 1.8e3 (eta = 1e-3) over a whole run.
    dtype f32 is the bench's C5 context (MMOT_F32: fp32 storage and fp32 arithmetic in the pair
    family, slab exponents): against the oracle on the fp32-rounded marginals at north_star's fp32
    bar, 1e-4 (marginals, W; log phi 1e-3 relative)."""
    import concurrent.futures as cf
    cfg = mmot_inputs.CONFIGS["C5"]
    l, N, B, T = cfg.l, cfg.N, cfg.batch, cfg.iters
    etas = mmot_inputs.c5_etas(B)
    mus_all = mmot_inputs.c5_batch_marginals(0, B, N, l)          # [l][B][N]
    rtol, rtol_g = (RTOL, 1e-9) if dtype == "f64" else (1e-4, 1e-3)
    if dtype == "f32":
        mus_all = mus_all.astype(np.float32)
        mu_d = [torch.from_numpy(mus_all[q]).to(DEV) for q in range(l)]
        mus_all = mus_all.astype(np.float64)                         # the values the context sees
    else:
        mu_d = [torch.from_numpy(mus_all[q]).to(DEV) for q in range(l)]
    ctx = mm.Context(l, N, [float(e) for e in etas], batch=B, dtype=dtype)
    u = [torch.empty((B, N), dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    rep = ctx.sinkhorn(mu_d, T, 0.0, u)
    assert rep["status"] == 0 and rep["iters_done"] == T
    assert ctx.pair_solves == 1  # the bench's family (pair.cu) at the bench's batch size
    assert ctx.pair_f32_solves == (1 if dtype == "f32" else 0)
    assert ctx.stable_fallbacks == 0  # nothing reached the stabilised family
    assert ctx.pair_redo <= 8  # fp32: the rare instances that left the fp32 range were redone in fp64
    le = np.log10(etas)
    edges = np.linspace(-3.0, -1.0, 9)
    picks = []
    for s in range(8):
        idx = np.nonzero((le >= edges[s]) & (le <= edges[s + 1]))[0]
        idx = idx[np.argsort(le[idx])]
        picks.append(int(idx[len(idx) // 2]))
    g = np.stack([x[picks].cpu().numpy() for x in u])               # [l][8][N]
    marg = [ctx.marginal(k, u)[picks].cpu().double().numpy() for k in range(l)]
    Wb = ctx.cost(u)
    ctx.close()
    h = mmot_inputs.grid_h(N)

    def ref(b):
        # O4 products (subset DP, pinned against O1/O3 in tests/test_oracle_subset.py): 4x faster
        from oracle import subset
        eta = float(etas[b])
        g_ref, _, _ = osk.sinkhorn(mus_all[:, b, :], h, eta, T, domain="log", engine="subset")
        lw = np.array([-(a * (l - a)) * h / eta for a in range(l + 1)])
        m_ref = [np.exp(g_ref[k] + subset.marginal_product_log(list(g_ref), k, lw)) for k in range(l)]
        return g_ref, m_ref

    with cf.ThreadPoolExecutor(max_workers=len(picks)) as ex:   # ctypes releases the GIL
        refs = list(ex.map(ref, picks))
    n_cost = 0
    for j, b in enumerate(picks):
        g_ref, m_ref = refs[j]
        fin = np.isfinite(g_ref)
        assert np.max(np.abs(g[:, j, :][fin] - g_ref[fin]) / np.maximum(1.0, np.abs(g_ref[fin]))) <= rtol_g, b
        for k in range(l):
            assert np.abs(marg[k][j] - m_ref[k]).sum() / np.abs(m_ref[k]).sum() <= rtol, (b, k)
        # W of the plan with the oracle's scalings, gauge-shifted towards fp64 range (A16:
        # sum_q c_q = 0 leaves the plan unchanged); the plain-fp64 cost oracle applies where every
        # shifted scaling is representable (the larger-eta strata)
        c = g_ref.max(axis=1)
        c[-1] -= c.sum()
        with np.errstate(over="ignore"):
            phis = np.exp(g_ref - c[:, None])
        if np.all(np.isfinite(phis)) and phis.max() < 1e250:
            W_ref = osk.cost(phis, h, float(etas[b]))
            assert abs(Wb[b] - W_ref) <= rtol * abs(W_ref), (b, Wb[b], W_ref)
            n_cost += 1
    assert n_cost >= 3, n_cost
