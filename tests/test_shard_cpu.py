"""Multi-GPU host logic on CPU (world_size 2, gloo): the grid partition of sharded contexts and
the composition of the gathered whole-shard operators into the carries entering each shard
(mmot_compose_rank_carries: the same template code the sharded contexts run on device).

Each rank builds the prefix and suffix operators of ITS shard with a plain numpy DP (test
infrastructure, written from dp.cuh's definitions: Op(F)[S] = sum_{U subset S} F[U] G_|U|[S\\U],
G_c = the shard's DP from the empty set with edge weights w_{c+|V|}), the operators are
all-gathered over gloo, composed by the library, and the result must equal the prefix / suffix
state at the shard boundary computed by one DP over the whole grid.  No GPU is used.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

import paper_2405_19246_b200 as mm  # noqa: E402


def _pc(x):
    return bin(x).count("1")


def _step(st, f, w, NB, c=0, limit=None, diag=True):
    """One grid point of the subset DP (diag then in-place place), weights shifted by c."""
    M = 1 << NB
    limit = NB - c if limit is None else limit
    st = st.copy()
    if diag:
        for S in range(M):
            if _pc(S) <= limit:
                st[S] *= w[c + _pc(S)]
    for b in range(NB):
        for S in range(M - 1, -1, -1):
            if (S >> b) & 1 and _pc(S) <= limit:
                st[S] += f[b] * st[S ^ (1 << b)]
    return st


def _shard_ops(f, w, NB):
    """Prefix and suffix operators of the points in f ([NB][n]) in op_store layout [(NB+1) * M]."""
    M = 1 << NB
    n = f.shape[1]
    G = np.zeros((NB + 1, M))
    R = np.zeros((NB + 1, M))
    for c in range(NB + 1):
        g = np.zeros(M)
        g[0] = 1.0
        r = g.copy()
        for x in range(n):
            g = _step(g, f[:, x], w, NB, c)
        for x in range(n - 1, -1, -1):
            r = _step(r, f[:, x], w, NB, c)
        for V in range(M):
            if _pc(V) <= NB - c:
                G[c, V] = g[V]
                R[c, V] = r[V]
    return G.reshape(-1), R.reshape(-1)


def _boundary_states(f, w, NB, lo, hi):
    """Whole-grid prefix state after points [0, lo) and suffix state of points [hi, N)."""
    M = 1 << NB
    F = np.zeros(M)
    F[0] = 1.0
    for x in range(lo):
        F = _step(F, f[:, x], w, NB)
    B = np.zeros(M)
    B[0] = 1.0
    for x in range(f.shape[1] - 1, hi - 1, -1):
        B = _step(B, f[:, x], w, NB)
    return F, B


def _worker(rank, world, port, l, N, lam, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        NB = l - 1
        w = np.array([lam ** (a * (l - a)) for a in range(l + 1)])
        rng = np.random.default_rng(123)                     # same full data on every rank
        f = rng.uniform(0.1, 1.0, size=(NB, N))
        lo, hi = mm.shard_range(N, rank, world)
        G, R = _shard_ops(f[:, lo:hi], w, NB)
        mine = torch.from_numpy(np.stack([G, R]))           # [2][SZ]
        gathered = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(gathered, mine)
        ops_all = torch.stack(gathered).numpy()              # [world][2][SZ]
        fin, bin_ = mm.compose_rank_carries(l, ops_all, world, rank)
        F, B = _boundary_states(f, w, NB, lo, hi)
        q.put((rank, lo, hi, float(np.max(np.abs(fin - F) / np.maximum(np.abs(F), 1e-300))),
               float(np.max(np.abs(bin_ - B) / np.maximum(np.abs(B), 1e-300)))))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("l,N,world", [(3, 37, 2), (4, 50, 2), (5, 23, 2), (4, 41, 3)])
def test_rank_carry_composition_gloo(l, N, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, l, N, 0.93, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == 0 and res[-1][2] == N
    for (r, lo, hi, ef, eb), nxt in zip(res, res[1:] + [None]):
        if nxt is not None:
            assert hi == nxt[1]
        assert ef <= 1e-13 and eb <= 1e-13, (r, ef, eb)


def test_shard_range_partition():
    for N in (1, 7, 100, 10 ** 8 + 3):
        for world in (1, 2, 3, 8):
            if N < world:
                continue
            rs = [mm.shard_range(N, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(hi - lo in (N // world, N // world + 1) for lo, hi in rs)


# ---------------------------------------------------------------------------------------
# Restricted next-update scan across shards (single-walk Sinkhorn updates): each rank builds the
# affine elements of its shard (new-part states of the next bound set) from exact
# whole-grid states of the current bound set, the elements are all-gathered, composed by the
# library, and must equal the next bound set's new-part states at the shard boundaries.
def _restricted_elements(fcur, fnew, w, NB, lo, hi, Fc, Bc):
    """Prefix/suffix affine elements of points [lo, hi) (numpy restatement of dp.cuh rx_*)."""
    l = NB + 1
    NO, MO = NB - 1, 1 << (NB - 1)
    L = np.zeros(MO)
    Mv = np.zeros(MO)
    G = np.zeros((NB, MO))
    G[:, 0] = 1.0
    for m in range(lo, hi):
        F = Fc[m + 1]
        B = Bc[m]
        o = fnew[m]
        f = fcur[:, m]
        if m == lo:
            for R in range(MO):
                Mv[R] += o * B[R << 1]
        else:
            s = np.array([o * w[_pc(U) + 1] * B[U << 1] for U in range(MO)])
            for R in range(MO):
                Mv[R] += sum(G[NB - _pc(R) - 1][R ^ U] * s[U] for U in range(MO) if (U & R) == U)
        if m > lo:
            for c in range(1, NB + 1):
                for V in range(MO):
                    if c + _pc(V) <= NB:
                        G[c - 1][V] *= w[c + _pc(V)]
        for c in range(1, NB + 1):
            for j in range(NO):
                for V in range(MO - 1, -1, -1):
                    if (V >> j) & 1 and c + _pc(V) <= NB:
                        G[c - 1][V] += f[j + 1] * G[c - 1][V ^ (1 << j)]
        for U in range(MO):
            L[U] *= w[_pc(U) + 1]
        for j in range(NO):
            for U in range(MO - 1, -1, -1):
                if (U >> j) & 1:
                    L[U] += f[j + 1] * L[U ^ (1 << j)]
        for U in range(MO):
            L[U] += o * F[U << 1]
    ef = np.zeros((NB + 1) * MO)
    eb = np.zeros((NB + 1) * MO)
    for c in range(1, NB + 1):
        for V in range(MO):
            if c + _pc(V) <= NB:
                ef[(c - 1) * MO + V] = w[c] * G[c - 1][V]
                eb[(c - 1) * MO + V] = w[c] * G[(l - c - _pc(V)) - 1][V]
    ef[NB * MO:] = L
    eb[NB * MO:] = Mv
    return ef, eb


def _affine_worker(rank, world, port, l, N, lam, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        NB = l - 1
        M, MO = 1 << NB, 1 << (NB - 1)
        w = np.array([lam ** (a * (l - a)) for a in range(l + 1)])
        rng = np.random.default_rng(321)
        fcur = rng.uniform(0.1, 1.0, size=(NB, N))
        fnew = rng.uniform(0.1, 1.0, size=N)
        fnext = np.vstack([fcur[1:], fnew[None]])
        # exact whole-grid states: Fc[x+1] = prefix after point x, Bc[x] = suffix of x..N-1
        Fc = [None] * (N + 1)
        s = np.zeros(M)
        s[0] = 1.0
        Fc[0] = s
        for x in range(N):
            s = _step(s, fcur[:, x], w, NB)
            Fc[x + 1] = s
        Bc = [None] * (N + 1)
        s = np.zeros(M)
        s[0] = 1.0
        Bc[N] = s
        for x in range(N - 1, -1, -1):
            s = _step(s, fcur[:, x], w, NB)
            Bc[x] = s
        lo, hi = mm.shard_range(N, rank, world)
        ef, eb = _restricted_elements(fcur, fnew, w, NB, lo, hi, Fc, Bc)
        mine = torch.from_numpy(np.stack([ef, eb]))
        gathered = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(gathered, mine)
        fin, bin_ = mm.compose_rank_affine(l, torch.stack(gathered).numpy(), world, rank)
        Fn, Bn = _boundary_states(fnext, w, NB, lo, hi)
        new = 1 << (NB - 1)
        Fw = np.array([Fn[U | new] for U in range(MO)])
        Bw = np.array([Bn[U | new] for U in range(MO)])
        ef_ = float(np.max(np.abs(fin - Fw) / np.maximum(np.abs(Fw), 1e-300))) if rank > 0 else float(np.max(np.abs(fin)))
        eb_ = float(np.max(np.abs(bin_ - Bw) / np.maximum(np.abs(Bw), 1e-300))) if rank < world - 1 else float(np.max(np.abs(bin_)))
        q.put((rank, ef_, eb_))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("l,N,world", [(3, 31, 2), (4, 40, 2), (5, 21, 3)])
def test_rank_affine_composition_gloo(l, N, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_affine_worker, args=(r, world, port, l, N, 0.91, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, ef, eb in res:
        assert ef <= 1e-12 and eb <= 1e-12, (r, ef, eb)
