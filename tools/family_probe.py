"""Small invocation of every kernel family (written for compute-sanitizer, which is closed on this
GPU pool; kept as a quick all-families smoke run): single-walk (k_sw_ops, k_sw_apply incl. the restricted next-update scan, k_rx_*,
k_sw_guard), two-walk (k_chunk_ops*, k_chunk_apply*, TMEM checkpoints, NB>=4 scans), persistent /
batched (k_bat_sinkhorn, k_bat_product), virtual shards (k_compose, k_rx_compose, k_vreduce),
non-uniform grids.

    python tools/family_probe.py
"""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402

DEV = "cuda:0"


def dev(vs):
    return [torch.from_numpy(np.ascontiguousarray(v)).to(DEV) for v in vs]


def solve(ctx, l, N, T=2, tol=0.0, batch=None):
    shape = (N,) if batch is None else (batch, N)
    mus = np.stack(mmot_inputs.random_marginals(5 + l, l, N))
    if batch is not None:
        mus = np.stack([np.stack([mus[q]] * batch) for q in range(l)])
    u = [torch.empty(shape, dtype=torch.float64, device=DEV) for _ in range(l)]
    ctx.init_uniform(u)
    ctx.sinkhorn(dev(mus), T, tol, u)
    for k in range(l):
        ctx.marginal(k, u)
    ctx.cost(u)
    torch.cuda.synchronize()


def main():
    N_sw = 64 * 8 * 40 + 13
    for l in (2, 3, 4, 5):
        ctx = mm.Context(l, N_sw, 2.0, chunk=40, kernel="single_walk")
        solve(ctx, l, N_sw, T=2)
        solve(ctx, l, N_sw, T=2, tol=1e-300)
        ctx.close()
    for l in (3, 4, 5, 6):
        N = 3000
        ctx = mm.Context(l, N, 0.05, kernel="two_walk")
        solve(ctx, l, N, T=2, tol=1e-300)
        ctx.close()
    for l in (3, 4, 5):
        ctx = mm.Context(l, 300, [0.05, 0.002], batch=2)
        solve(ctx, l, 300, T=3, tol=1e-300, batch=2)
        ctx.close()
    x = np.sort(np.random.default_rng(3).uniform(0, 1, 500))
    ctx = mm.Context(4, 500, 0.05, points=x)
    solve(ctx, 4, 500, T=2)
    ctx.close()
    # virtual shards: 2 ranks, single-walk (restricted scan) and two-walk
    for kern, chunk in (("single_walk", 40), ("two_walk", 0)):
        G, l, N = 2, 4, 2 * 64 * 40 * 4
        grp = mm.VirtualGroup(G)
        mus = np.stack(mmot_inputs.random_marginals(9, l, N))

        def rank(r):
            with torch.cuda.stream(torch.cuda.Stream(device=DEV)):
                lo, hi = mm.shard_range(N, r, G)
                c = mm.Context(l, N, 2.0, shard=(r, G, grp), kernel=kern, chunk=chunk)
                u = [torch.empty(hi - lo, dtype=torch.float64, device=DEV) for _ in range(l)]
                c.init_uniform(u)
                c.sinkhorn(dev([m[lo:hi] for m in mus]), 2, 1e-300, u)
                c.cost(u)
                torch.cuda.synchronize()
                c.close()

        ts = [threading.Thread(target=rank, args=(r,)) for r in range(G)]
        [t.start() for t in ts]
        [t.join() for t in ts]
        grp.close()
    print("sanitize probe done")


if __name__ == "__main__":
    main()
