import sys, torch
sys.path.insert(0, '.')
import mmot_inputs
import paper_2405_19246_b200 as mm
cfg = mmot_inputs.CONFIGS["C4"]
l, N, eta = cfg.l, cfg.N, cfg.eta
mus = mmot_inputs.make_marginals("C4", 0)
mu_d = [torch.from_numpy(m).cuda() for m in mus]
del mus
for chunk in [0, 880, 1056, 1320, 1584, 1760, 2200]:
    ctx = mm.Context(l, N, eta, chunk=chunk, kernel="single_walk")
    u = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(l)]
    T = 10
    for rep in range(2):
        ctx.init_uniform(u)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(ctx.stream)
        ctx.sinkhorn(mu_d, T, 0.0, u)
        e.record(ctx.stream)
        torch.cuda.synchronize()
    print(f"chunk {chunk} (P={ctx.info['chain_len']}): {s.elapsed_time(e)/T/l:.4f} ms/update", flush=True)
    ctx.close()
    del u
