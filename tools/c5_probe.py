"""Reduced C5 run for profiling the batched kernel (not the bench): B instances, T sweeps."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import mmot_inputs
import paper_2405_19246_b200 as mm

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
T = int(sys.argv[2]) if len(sys.argv) > 2 else 10
l, N = 5, 4096
etas = [float(e) for e in mmot_inputs.c5_etas(B)]
mus = mmot_inputs.c5_batch_marginals(0, B, N, l)
dev = 'cuda:0'
mu_d = [torch.from_numpy(mus[q]).to(dev) for q in range(l)]
ctx = mm.Context(l, N, etas, batch=B)
u = [torch.empty((B, N), dtype=torch.float64, device=dev) for _ in range(l)]
for rep in range(2):
    ctx.init_uniform(u)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = ctx.sinkhorn(mu_d, T, 0.0, u)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(f"B={B} T={T}: {ms:.1f} ms, {ms/T/l*1e3:.1f} us/update-wave, status {r['status']}", flush=True)
ctx.close()
