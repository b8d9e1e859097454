"""The paper's 1-D random-distribution experiment (§5.1; Table 1 and Fig. 1a):
three U[0,1] vectors normalised to probability vectors on N uniform grid points of [0,1], eps = 0.1,
100 Sinkhorn iterations; the fast tensor-vector-product Sinkhorn (here: the B200 library) against
the dense O(N^l) Sinkhorn (here: the fp64 CPU oracle O1, oracle/dense.py), with the Frobenius norm
of the difference of the two transport plans and the empirical complexity slopes by linear
regression of log time on log N (paper: O(N^1.01) fast, O(N^3.01) dense, on MATLAB / i5-1135G7).

The paper's grid N = 10..160 is latency-bound on a GPU (a whole 100-sweep solve is one persistent
launch), so the GPU slope is also fitted on large N (3e7..3e8), where the product is HBM-bound.

    python examples/slope_study.py [--out profiles/r02_slope_study.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import mmot_inputs  # noqa: E402

EPS, T, L = 0.1, 100, 3
PAPER_N = [10, 20, 40, 80, 160]
LARGE_N = [1_000_000, 30_000_000, 100_000_000, 300_000_000]


def u01_marginals(N: int, seed: int) -> np.ndarray:
    """Three U[0,1] vectors normalised by their l1 norms, seeded."""
    rng = np.random.default_rng(51_000 + seed)
    u = rng.uniform(0.0, 1.0, (L, N))
    return u / u.sum(axis=1, keepdims=True)


def gpu_solve(mus: np.ndarray, repeats: int = 3):
    """100 sweeps through mmot_sinkhorn from phi = 1/N; returns (phis, median seconds per solve)."""
    import torch

    import paper_2405_19246_b200 as mm
    N = mus.shape[1]
    dev = "cuda:0"
    ctx = mm.Context(L, N, EPS, repr="log")
    mu_d = [torch.from_numpy(m).to(dev) for m in mus]
    u = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(L)]
    times = []
    for i in range(repeats + 1):
        ctx.init_uniform(u)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = ctx.sinkhorn(mu_d, T, 0.0, u)
        torch.cuda.synchronize()
        if i > 0:
            times.append(time.perf_counter() - t0)
        assert rep["status"] == 0
    phis = np.exp(np.stack([x.cpu().numpy() for x in u]))
    kernel = ctx.info["kernel"]
    ctx.close()
    return phis, float(np.median(times)), kernel


def dense_solve(mus: np.ndarray):
    from oracle import dense
    N = mus.shape[1]
    h = mmot_inputs.grid_h(N)
    t0 = time.perf_counter()
    phis, _, _ = dense.sinkhorn(mus, h, EPS, T)
    return phis, time.perf_counter() - t0


def plan(phis: np.ndarray) -> np.ndarray:
    from oracle import dense
    N = phis.shape[1]
    K = dense.kernel_tensor(L, N, mmot_inputs.grid_h(N), EPS)
    return dense.plan(K, list(phis))


def slope(ns, ts) -> float:
    return float(np.polyfit(np.log(ns), np.log(ts), 1)[0])


def run(paper_n=PAPER_N, large_n=LARGE_N):
    rows = []
    for N in paper_n:
        mus = u01_marginals(N, N)
        pf, tf, kern = gpu_solve(mus)
        pd, td = dense_solve(mus)
        diff = float(np.linalg.norm(plan(pf) - plan(pd)))
        rows.append({"N": N, "gpu_s": tf, "dense_cpu_s": td, "speedup": td / tf, "plan_diff_F": diff, "kernel": kern})
    large = []
    for N in large_n:
        mus = u01_marginals(N, N)
        _, tf, kern = gpu_solve(mus, repeats=2)
        large.append({"N": N, "gpu_s": tf, "kernel": kern, "ns_per_point_sweep": tf / (T * N) * 1e9})
    out = {
        "experiment": "PAPER.md §5.1 (Table 1, Fig. 1a): l=3, eps=0.1, 100 iterations, U[0,1] marginals",
        "paper": {"fast_slope": 1.01, "dense_slope": 3.01, "hardware": "MATLAB R2020a, i5-1135G7 (P:1133)"},
        "rows": rows,
        "dense_slope": slope([r["N"] for r in rows if r["N"] >= 40], [r["dense_cpu_s"] for r in rows if r["N"] >= 40]),
        "gpu_slope_paper_grid": slope([r["N"] for r in rows], [r["gpu_s"] for r in rows]),
        "large_n": large,
        "gpu_slope_large_n": slope([r["N"] for r in large[1:]], [r["gpu_s"] for r in large[1:]]),
        "note": ("dense = the fp64 CPU oracle O1 (numpy contraction of the N^3 kernel tensor, one host "
                 "thread); the GPU solve on the paper grid is one persistent launch (latency-bound, slope ~0); "
                 "the large-N slope is the O(N) claim on the HBM-bound path"),
    }
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = run()
    txt = json.dumps(res, indent=1)
    print(txt)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt + "\n")
