"""Reduced C5 run for profiling the batched kernel (not the bench): B instances, T sweeps."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import mmot_inputs
import paper_2405_19246_b200 as mm

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
T = int(sys.argv[2]) if len(sys.argv) > 2 else 10
DT = sys.argv[3] if len(sys.argv) > 3 else 'f64'
l, N = 5, 4096
etas = [float(e) for e in mmot_inputs.c5_etas(B)]
mus = mmot_inputs.c5_batch_marginals(0, B, N, l)
dev = 'cuda:0'
mu_d = [torch.from_numpy(mus[q].astype(np.float32) if DT == 'f32' else mus[q]).to(dev) for q in range(l)]
ctx = mm.Context(l, N, etas, batch=B, dtype=DT)
u = [torch.empty((B, N), dtype=torch.float64, device=dev) for _ in range(l)]
REPS = int(sys.argv[4]) if len(sys.argv) > 4 else 2
best = 1e30
for rep in range(REPS):
    ctx.init_uniform(u)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = ctx.sinkhorn(mu_d, T, 0.0, u)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    best = min(best, ms) if rep > 0 else best
    print(f"B={B} T={T}: {ms:.1f} ms, {ms/T/l*1e3:.1f} us/update-wave, status {r['status']} pair {ctx.pair_solves}", flush=True)
print(f'best of {REPS - 1}: {best:.2f} ms')
ctx.close()
