"""Non-uniform vs uniform grid cost of one Sinkhorn solve (profiling only, not the bench)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import mmot_inputs
import paper_2405_19246_b200 as mm

dev = 'cuda:0'
for (l, N, eta, T, B) in [(4, 1000, 0.01, 200, None), (4, 1_000_000, 1e-3, 20, None), (5, 4096, 0.01, 30, 1184)]:
    rng = np.random.default_rng(1)
    x = np.concatenate([[0.0], np.cumsum(rng.uniform(1.0, 3.0, N - 1))])
    x /= x[-1]
    if B is None:
        mus = np.stack(mmot_inputs.random_marginals(3, l, N))
        mu_d = [torch.from_numpy(m).to(dev) for m in mus]
        shape = (N,)
    else:
        mus = mmot_inputs.c5_batch_marginals(0, B, N, l)
        mu_d = [torch.from_numpy(mus[q]).to(dev) for q in range(l)]
        shape = (B, N)
    res = {}
    for name, kw in (("uniform", {}), ("points", {"points": x})):
        ctx = mm.Context(l, N, eta if B is None else [eta] * B, batch=B, **kw)
        u = [torch.empty(shape, dtype=torch.float64, device=dev) for _ in range(l)]
        for rep in range(2):
            ctx.init_uniform(u)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            ctx.sinkhorn(mu_d, T, 0.0, u)
            e.record()
            torch.cuda.synchronize()
        res[name] = (s.elapsed_time(e), ctx.info["kernel"])
        ctx.close()
    print(f"l={l} N={N} T={T} batch={B}: uniform {res['uniform'][0]:.2f} ms ({res['uniform'][1]}), "
          f"points {res['points'][0]:.2f} ms ({res['points'][1]}), ratio {res['points'][0] / res['uniform'][0]:.2f}")
