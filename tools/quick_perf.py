"""Scratch timing of one Sinkhorn sweep at a config size (CUDA events). Not the bench."""
import sys, time, math
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2405_19246_b200 as mm

def run(l, N, eta, sweeps=2, chunk=0):
    dev = 'cuda:0'
    rng = np.random.default_rng(0)
    mus = [torch.rand(N, dtype=torch.float64, device=dev) + 0.5 for _ in range(l)]
    mus = [m / m.sum() for m in mus]
    ctx = mm.Context(l, N, eta, repr='linear', chunk=chunk)
    u = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(l)]
    ctx.init_uniform(u)
    ctx.sinkhorn(mus, 1, 0.0, u)  # warm
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = ctx.launches
    s.record(); rep = ctx.sinkhorn(mus, sweeps, 0.0, u); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / sweeps
    nl = (ctx.launches - n0) / sweeps
    alg = (l + 1) * N * 8 * l  # bytes per sweep
    print(f"l={l} N={N:.0e} chunk={ctx_chunk(ctx)}: {ms:.3f} ms/sweep, {ms/l:.3f} ms/update, launches/sweep {nl:.0f}, "
          f"alg BW {alg/ms/1e6:.1f} GB/s, status {rep['status']}", flush=True)
    ctx.close()

def ctx_chunk(ctx):
    return '?'

if __name__ == '__main__':
    for spec in sys.argv[1:]:
        l, N, eta = spec.split(',')[:3]
        run(int(l), int(float(N)), float(eta))
