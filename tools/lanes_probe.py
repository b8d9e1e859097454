"""Probe of the l = 6 lane-state family: a few update products at C3 size (for ncu launch lists)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import mmot_inputs
import paper_2405_19246_b200 as mm

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mus = mmot_inputs.c3_marginals(0, N, 6)
mu_d = [torch.from_numpy(m).to('cuda') for m in mus]
ctx = mm.Context(6, N, 1e-3)
u = [torch.empty(N, dtype=torch.float64, device='cuda') for _ in range(6)]
for rep in range(2):
    ctx.init_uniform(u)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = ctx.sinkhorn(mu_d, T, 0.0, u)
    e.record()
    torch.cuda.synchronize()
    print(f"N={N} T={T}: {s.elapsed_time(e):.3f} ms ({s.elapsed_time(e)/T/6*1e3:.1f} us/update) {ctx.info}", flush=True)
