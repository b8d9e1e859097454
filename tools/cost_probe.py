import sys, torch
sys.path.insert(0, '.')
import mmot_inputs
import paper_2405_19246_b200 as mm
cfg = mmot_inputs.CONFIGS["C4"]
l, N, eta = cfg.l, cfg.N, cfg.eta
ctx = mm.Context(l, N, eta)
u = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(l)]
ctx.init_uniform(u)
for rep in range(3):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(ctx.stream)
    W = ctx.cost(u)
    e.record(ctx.stream)
    torch.cuda.synchronize()
    t_cost = s.elapsed_time(e)
    s.record(ctx.stream)
    m = ctx.marginal(0, u)
    e.record(ctx.stream)
    torch.cuda.synchronize()
    t_marg = s.elapsed_time(e)
print(f"C4 size: mmot_cost {t_cost:.2f} ms, mmot_marginal {t_marg:.2f} ms (algorithmic l*N*8 B: {l*N*8/1e9:.1f} GB)")
