"""C5 in an MMOT_F32 context (pair family, fp32 arithmetic): how many instances leave the fp32 range
(MMOT_DEBUG_FAIL=1 prints them; MMOT_NO_STABLE=1 skips the stabilised redo).  Usage:
  python tools/c5_f32_probe.py [T] [B]      (B: the first B instances, e.g. 1024 = one rank of 8)"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mmot_inputs  # noqa: E402
import paper_2405_19246_b200 as mm  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 300
cfg = mmot_inputs.CONFIGS["C5"]
l, N, B = cfg.l, cfg.N, cfg.batch
B = int(sys.argv[2]) if len(sys.argv) > 2 else B
etas = [float(e) for e in mmot_inputs.c5_etas(cfg.batch)[:B]]
mus = mmot_inputs.c5_batch_marginals(0, B, N, l).astype(np.float32)
dev = torch.device("cuda:0")
mu_d = [torch.from_numpy(np.ascontiguousarray(mus[q])).to(dev) for q in range(l)]
ctx = mm.Context(l, N, etas, batch=B, dtype="f32")
u = [torch.empty((B, N), dtype=torch.float64, device=dev) for _ in range(l)]
ctx.init_uniform(u)
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = ctx.sinkhorn(mu_d, T, 0.0, u)
torch.cuda.synchronize()
print(f"T={T} status={rep['status']} {time.perf_counter() - t0:.3f} s pair={ctx.pair_solves} f32={ctx.pair_f32_solves} "
      f"stable_redo={ctx.stable_fallbacks} B={B} kernel={ctx.info['kernel']}", flush=True)
