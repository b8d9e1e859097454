"""The paper's Ricker-wavelet problem (§5.2) on the GPU path: three shifted
Ricker wavelets on [-2, 2], N = 100, epsilon = 1e-3 (h/eta = 40.4), W_epsilon of the three
normalised wavelets.  The paper's unstabilised recursion stops at iteration 89 (Fig. 2b); the
library keeps the scalings as mantissas with per-chain binary exponents and runs on.

    python examples/ricker_stabilisation.py [sweeps]

(The plain-domain breakdown itself is pinned against the CPU oracle in tests/test_ricker.py.)"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
N, ETA = 100, 1e-3
mus = mmot_inputs.ricker_marginals(N)
dev = "cuda:0"
mu_d = [torch.from_numpy(m).to(dev) for m in mus]
ctx = mm.Context(3, N, ETA, grid=(-2.0, 2.0), repr="log", check_every=1)
u = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(3)]
ctx.init_uniform(u)
done = 0
for target in (50, 89, 100, 200, 500, 1000, T):
    if target > T or target <= done:
        continue
    t0 = time.perf_counter()
    rep = ctx.sinkhorn(mu_d, target - done, 1e-300, u)  # continue from the current scalings
    dt = time.perf_counter() - t0
    done = target
    gmax = max(float(x.abs().max()) for x in u)
    print(f"sweep {done:5d}: status {rep['status']}, residual {rep['residual']:.3e}, max|log phi| {gmax:8.1f}, "
          f"{dt * 1e3:7.2f} ms for the segment")
print(f"W_eps = {ctx.cost(u):.6f}")
m = [ctx.marginal(k, u).cpu().numpy() for k in range(3)]
print("marginal L1 errors:", ["%.2e" % np.abs(m[k] - mus[k]).sum() for k in range(3)])
ctx.close()
