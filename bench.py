#!/usr/bin/env python
"""bench.py -- B200 benchmark of the fast tensor-vector product inside multi-marginal Sinkhorn.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl mmot|reference]

A *step* is one pass of the whole hot path over the config's synthetic batch: the paper's
initialisation, ``mmot_sinkhorn`` for the config's T sweeps of l fused updates
(residual + tolerance when the config has one) and ``mmot_cost``
(P:1037-1040).  Metric (BASELINE.json): fast marginal evaluations, reported as l*N elements
per second (one eval = one J_k, T*l evals per step), plus Sinkhorn iters/s and the HBM
roofline fraction of the update.

Prints ONE JSON line on rank 0.  See DESIGN.md §5 for every field's definition.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import mmot_inputs  # noqa: E402

METRIC = "fast marginal evals throughput (l*N elements/s)"
UNIT = "elem/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C3f", "C4", "C5"])
    ap.add_argument("--impl", default="mmot", choices=["mmot", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="use the sharded (multi-GPU) context even at one rank (exercises the NCCL exchange)")
    return ap.parse_args()


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _workload(cfg):
    return (f"{cfg.name}: l={cfg.l} N={cfg.N} eta={cfg.eta} {cfg.dtype} T={cfg.iters}"
            + (f" tol={cfg.tol}" if cfg.tol > 0 else ""))


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms.  Started before the warm-up so the
    sampler is running when the timed region starts; begin() marks the start of the timed region and
    stop() keeps the rows taken after it.  A timed region shorter than the sampling period (C1) may
    hold no row: then the last row before it (taken under the warm-up's load) is reported and
    "window" says so."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(dev_index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        self.mark = 0

    def _rows(self):
        self.f.flush()
        rows = []
        try:
            for ln in open(self.f.name):
                parts = [x.strip() for x in ln.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        return rows

    def begin(self):
        """Mark the start of the timed region (waits up to 2 s for the sampler's first row)."""
        t0 = time.time()
        while self.p is not None and not self._rows() and time.time() - t0 < 2.0:
            time.sleep(0.02)
        self.mark = len(self._rows())

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        all_rows = self._rows()
        os.unlink(self.f.name)
        rows = all_rows[self.mark:]
        window = "timed region"
        if not rows and all_rows:
            rows = all_rows[self.mark - 1:self.mark] if self.mark > 0 else all_rows[:1]
            window = "last sample before the timed region (region shorter than the 200 ms period)"
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows), "window": window}


# ------------------------------------------------------------------------------------------
def oracle_update_rate(cfg, mus, n_sample: int):
    """The CPU oracle as it stands (O4, oracle/subset.c subset-lattice DP, gcc -O3, single thread:
    the recurrence is sequential -- BASELINE.md §3): one Sinkhorn update phi_0 <- mu_0 / J_0 on the
    first n_sample grid points of the config's marginals, at the config's lambda."""
    from oracle import regions, subset
    l = cfg.l
    N = n_sample
    h = mmot_inputs.grid_h(cfg.N)  # keep the config's grid spacing (lambda)
    w = regions.edge_weights(l, h, cfg.eta)
    phis = [np.full(N, 1.0 / cfg.N) for _ in range(l)]
    t0 = time.perf_counter()
    J = subset.marginal_product(phis, 0, w)
    phi0 = mus[0][:N] / J
    dt = time.perf_counter() - t0
    assert np.all(np.isfinite(phi0))
    return l * N / dt, dt


def oracle_batched_rate(cfg, n_inst: int, sweeps: int = 2, threads: int = 0):
    """The CPU oracle as it stands (oracle/sinkhorn.py log-domain driver over O4 products) on
    `n_inst` C5 instances x `sweeps` sweeps, instances spread over `threads` host threads (0 = all
    cores; C5 runs instance-parallel): elements/s in the metric's unit."""
    import concurrent.futures as cf

    from oracle import sinkhorn as osk
    threads = threads or os.cpu_count() or 1
    etas = mmot_inputs.c5_etas(n_inst)
    h = mmot_inputs.grid_h(cfg.N)
    inputs = []
    for b in range(n_inst):
        mus = mmot_inputs.c5_marginals(b, cfg.N, cfg.l)
        if cfg.dtype == "f32":
            mus = mus.astype(np.float32).astype(np.float64)  # the fp32-rounded inputs of the GPU run
        inputs.append(mus)

    def one(b):
        osk.sinkhorn(inputs[b], h, float(etas[b]), sweeps, domain="log", engine="subset")

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:   # ctypes releases the GIL
        list(ex.map(one, range(n_inst)))
    dt = time.perf_counter() - t0
    elems = n_inst * sweeps * cfg.l * cfg.l * cfg.N
    return elems / dt, dt, min(threads, n_inst)


def run_reference(args, cfg):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    rates = []
    cores = 1
    if cfg.batch > 1:
        nthr = os.cpu_count() or 1
        for i in range(min(args.warmup, 1) + args.steps):
            r, dt, cores = oracle_batched_rate(cfg, nthr, 2, nthr)
            if i >= min(args.warmup, 1):
                rates.append((r, dt))
        sample = (f"2 log-domain Sinkhorn sweeps (O4 subset-DP products) of {nthr} {cfg.name} instances "
                  f"(l={cfg.l}, N={cfg.N}), one per host thread")
    else:
        n_sample = min(cfg.N, 10_000_000)
        mus = mmot_inputs.make_marginals(cfg.name, 0, None if cfg.N <= 2_000_000 else n_sample)
        if cfg.dtype == "f32":
            mus = mus.astype(np.float32).astype(np.float64)  # the fp32-rounded inputs of the GPU run
        for i in range(args.warmup + args.steps):
            r, dt = oracle_update_rate(cfg, mus, n_sample)
            if i >= args.warmup:
                rates.append((r, dt))
        sample = (f"one Sinkhorn update (J_0 by the O4 subset-DP oracle + division) on the first {n_sample} "
                  f"grid points of {cfg.name}'s marginals, config lambda")
    value = statistics.median(r for r, _ in rates)
    ms = statistics.median(dt for _, dt in rates) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": _workload(cfg), "parallelism": f"oracle, {cores} host thread(s)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    _emit(line)


# ------------------------------------------------------------------------------------------
FP64_PEAK = 148 * 64 * 2 * 1.965e9 / 1e12  # TFLOP/s: SMs x FP64 FMA/clk x 2 x max SM clock
FP32_PEAK = 148 * 128 * 2 * 1.965e9 / 1e12  # TFLOP/s: SMs x FP32 FMA/clk x 2 x max SM clock


def run_batched(args, cfg):
    """C5: `cfg.batch` independent instances sharded contiguously over the ranks, one batched
    context per rank (no collective in the loop)."""
    import torch
    import torch.distributed as dist

    import paper_2405_19246_b200 as mm

    ws, rank, local = _dist()
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    l, N, T = cfg.l, cfg.N, cfg.iters
    b0, b1 = rank * cfg.batch // ws, (rank + 1) * cfg.batch // ws
    B = b1 - b0
    etas = [float(e) for e in mmot_inputs.c5_etas(cfg.batch)[b0:b1]]
    mus_h = mmot_inputs.c5_batch_marginals(b0, B, N, l)            # [l][B][N] fp64, seeded
    io32 = cfg.dtype == "f32"  # C5 is an fp32 config: MMOT_F32 context (fp32 marginals, storage, arithmetic)
    if io32:
        mus_h = mus_h.astype(np.float32)
    mus_d = [torch.from_numpy(np.ascontiguousarray(mus_h[q])).to(dev) for q in range(l)]
    ctx = mm.Context(l, N, etas, batch=B, repr="log", dtype="f32" if io32 else "f64")
    u = [torch.empty((B, N), dtype=torch.float64, device=dev) for _ in range(l)]
    state = {}
    stream = ctx.stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * max(args.steps, 1))]
    sk_ms = []

    def step(i=None):
        ctx.init_uniform(u)
        if i is not None:
            ev[2 * i].record(stream)
        state["rep"] = ctx.sinkhorn(mus_d, T, 0.0, u)
        if i is not None:
            ev[2 * i + 1].record(stream)
        state["W"] = ctx.cost(u)

    def barrier():
        if ws > 1:
            dist.barrier()

    clocks = ClockSampler(local)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks.begin()
    launches0 = ctx.launches
    barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(args.steps):
        step(i)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms_local = e0.elapsed_time(e1) / args.steps
    sk_ms = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(args.steps)]
    launches = (ctx.launches - launches0) // args.steps
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    evals_all = cfg.batch * T * l            # every rank's share, whole job
    value = evals_all * l * N / (ms / 1e3)
    # roofline of the dominant kernel (k_bat_sinkhorn, one launch per step): algorithmic FLOPs
    # = 2 * 2^(l-1) (l+3) per grid point per update, FP64 ALU peak
    flop = B * T * l * N * 2 * (2 ** (l - 1)) * (l + 3)
    sk = statistics.median(sk_ms)
    achieved = flop / (sk / 1e3) / 1e12
    f32c = ctx.pair_f32_solves > 0            # the pair family computed in fp32 (MMOT_F32 context)
    peak = FP32_PEAK if f32c else FP64_PEAK
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": ("k_pair_sinkhorn (pair family: all sweeps of all instances of the rank, one launch, "
                           "plus the layout conversions)" if ctx.pair_solves else
                           "k_bat_sinkhorn (all sweeps of all instances of the rank, one launch)"),
                "alg_flop_per_launch": flop, "ms_per_launch": sk,
                "peak_source": ("derived: 148 SMs x 128 FP32 FMA/clk x 2 x 1.965 GHz (DESIGN.md §5)" if f32c else
                                "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz (DESIGN.md §5)")}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        nthr = os.cpu_count() or 1
        r, dt, cores = oracle_batched_rate(cfg, 2 * nthr, 20, nthr)
        cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"20 log-domain sweeps (O4 subset-DP products) of {2 * nthr} C5 instances on {cores} host "
                         f"threads ({os.cpu_count()} cores), {dt:.1f} s"}
    e2e = None
    if not args.no_e2e:
        # through the C ABI with host buffers: H2D of marginals + initial scalings, D2H of the
        # final scalings and W, every step
        mh = [torch.from_numpy(mus_h[q]).pin_memory() for q in range(l)]
        uh = [torch.empty((B, N), dtype=torch.float64).pin_memory() for _ in range(l)]
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            md = [x.to(dev, non_blocking=True) for x in mh]
            ctx.init_uniform(u)
            ctx.sinkhorn(md, T, 0.0, u)
            W = ctx.cost(u)
            for q in range(l):
                uh[q].copy_(u[q], non_blocking=True)
            torch.cuda.synchronize()
        barrier()
        e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        te = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_ms = float(te.item())
        e2e = {"value": evals_all * l * N / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": l * B * N * mus_h.itemsize, "d2h_bytes_per_step": l * B * N * 8 + B * 8}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32" if f32c else "f64", "data": "synthetic",
            "config": {"workload": f"C5: {cfg.batch} instances x (l={l}, N={N}), eta_b ~ logU[1e-3,1e-1], "
                                   f"T={T}, " + ("f32" if f32c else "f64") + " arithmetic", "l": l, "N": N,
                       "family": ("pair (two threads per instance, no chain operators; mantissas with one "
                                  "exponent per 8 points, " + ("fp32" if io32 else "fp64") + " storage, " +
                                  ("fp32" if f32c else "fp64") + " arithmetic)")
                       if ctx.pair_solves else "persistent (warp per instance, 32 chains, per-chain exponents)",
                       "io_dtype": "f32 marginals (MMOT_F32 context), fp64 u[]" if io32 else "f64",
                       "batch": cfg.batch, "iters": T, "parallelism": f"instances sharded over {ws} GPU(s)",
                       "l2": "per-instance working set L2/SMEM resident; no flush (ALU-bound)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": int(launches), "iters_per_s": cfg.batch * T / (ms / 1e3),
            "W_first": state["W"][0], "impl": "mmot",
        }
        _emit(line)
    ctx.close()
    if ws > 1:
        dist.destroy_process_group()


def run_mmot(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2405_19246_b200 as mm

    ws, rank, local = _dist()
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    l, N, T, tol = cfg.l, cfg.N, cfg.iters, cfg.tol

    mus_h = mmot_inputs.make_marginals(cfg.name, 0)  # fp64 host, seeded (the one global instance)
    shard = None
    if ws > 1 or args.shard:
        # one instance sharded by contiguous grid chunks; the NCCL id travels over torch.distributed
        obj = [mm.nccl_unique_id() if rank == 0 else None]
        if ws > 1:
            dist.broadcast_object_list(obj, src=0)
        shard = (rank, ws, obj[0])
        lo, hi = mm.shard_range(N, rank, ws)
        mus_h = np.ascontiguousarray(mus_h[:, lo:hi])
    io32 = cfg.dtype == "f32"  # C3f: fp32 marginals in (MMOT_F32 I/O), fp64 scans
    if io32:
        mus_h = mus_h.astype(np.float32)
    mus_d = [torch.from_numpy(np.ascontiguousarray(m)).to(dev) for m in mus_h]
    ctx = mm.Context(l, N, cfg.eta, repr="log", check_every=1 if tol > 0 else 0, shard=shard,
                     dtype="f32" if io32 else "f64")
    Nl = ctx.N  # this rank's grid points
    u = [torch.empty(Nl, dtype=torch.float64, device=dev) for _ in range(l)]
    state = {}

    def step():
        ctx.init_uniform(u)
        rep = ctx.sinkhorn(mus_d, T, tol, u)
        state["rep"] = rep
        state["W"] = ctx.cost(u)

    def barrier():
        if ws > 1:
            dist.barrier()

    clocks = ClockSampler(local)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = ctx.stream
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    clocks.begin()
    launches0 = ctx.launches
    graphs0 = ctx.graph_solves
    barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    launches = (ctx.launches - launches0) // args.steps
    graph_solves = ctx.graph_solves - graphs0
    # per-update kernel time: one more step with CUDA events around every product on the context
    # stream (profiling switches the solve to the host-issued launch sequence: the same kernels)
    ctx.profile(True)
    ctx.profile_read()
    step()
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    iters_done = state["rep"]["iters_done"]
    evals = iters_done * l
    value = evals * l * N / (ms / 1e3)  # one global instance of N points (sharded when ws > 1)

    # roofline of the dominant kernel group: the fused Sinkhorn update (one product of mode
    # "update" = operator pass + scan + apply).  Algorithmic bytes per update = (l+1) N 8.
    n_upd = prof["mode_n"]["update"]
    if n_upd > 0:
        upd_ms = prof["mode_ms"]["update"] / n_upd
    else:
        # persistent kernel (small instances): all sweeps in one launch, no per-update events;
        # the step time per update is an upper bound of the update time
        upd_ms = ms / max(iters_done * l, 1)
    alg_bytes = (l + 1) * Nl * 8
    peak, peak_src = _peaks()
    achieved = alg_bytes / (upd_ms / 1e3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf) and shard is None:
        try:
            traffic = json.load(open(tf)).get(cfg.name)
        except Exception:
            traffic = None
    step_frac = alg_bytes * iters_done * l / (ms / 1e3) / 1e9 / peak
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic,
                "kernel": ("k_cta_sinkhorn (whole solve in one launch; per-update time = step / updates)"
                           if ctx.cta_solves else "fused update (ops + scan + apply of one J_k)"),
                "alg_bytes_per_launch": alg_bytes, "ms_per_launch": upd_ms, "peak_source": peak_src,
                "ms_per_launch_source": "CUDA events around each update of one profiled step after the timed region",
                "step_level_frac": step_frac,
                "phase_ms_per_update": {k: v / max(sum(prof["mode_n"].values()), 1) for k, v in prof["phase_ms"].items()}}

    # end-to-end through the C ABI with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        mh = [torch.from_numpy(m).pin_memory() for m in mus_h]
        uh = [torch.empty(Nl, dtype=torch.float64).pin_memory() for _ in range(l)]
        for x in uh:
            x.fill_(-math.log(N))
        ctx.sinkhorn_host(mh, T, tol, uh)  # warm (allocates staging once)
        ctx.cost_staged()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            for x in uh:
                x.fill_(-math.log(N))
            ctx.sinkhorn_host(mh, T, tol, uh)
            state["W_e2e"] = ctx.cost_staged()  # the step's W, from the scalings still on the device
        torch.cuda.synchronize()
        barrier()
        e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        te = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_ms = float(te.item())
        e2e = {"value": evals * l * N / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": l * Nl * (mus_h.itemsize + 8), "d2h_bytes_per_step": l * Nl * 8 + 8}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        n_sample = min(N, 100_000_000)
        r, dt = oracle_update_rate(cfg, mus_h, n_sample)
        cpu = {"value": r, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"one update (O4 subset-DP J_0 + division) over {n_sample} grid points of {cfg.name}, "
                         f"{dt:.1f} s single-thread of {os.cpu_count()} host cores"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload(cfg), "l": l, "N": N, "eta": cfg.eta, "iters": T, "tol": tol,
                       "io_dtype": "f32 marginals (MMOT_F32 context), fp64 u[]" if io32 else "f64",
                       "global_batch": 1,
                       "parallelism": (f"grid sharded over {ws} GPUs (contiguous chunks, NCCL all-gather of "
                                       f"whole-shard operators per update)") if ws > 1 else "single GPU",
                       "kernel": "cta" if ctx.cta_solves else ctx.info["kernel"],
                       "chain_len": ctx.info["chain_len"],
                       "l2": "inputs (l*N*8*2 B) exceed the 126 MB L2; no flush needed" if N >= 5_000_000 else
                             "working set L2-resident (latency-bound config)"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "gpu_launches": int(launches),
            "device_loop": ("CUDA graph, conditional WHILE node (one graph launch per solve)" if graph_solves
                            else "CTA family: one thread block per instance, the whole solve in one launch"
                            if ctx.cta_solves
                            else "persistent kernel" if ctx.info["kernel"] == "persistent" else "host-issued launches"),
            "iters_per_s": iters_done / (ms / 1e3),
            "iters_done": iters_done,
            "W": state["W"],
            "impl": "mmot",
        }
        _emit(line)
    ctx.close()
    if ws > 1:
        dist.destroy_process_group()


_JSON_OUT = None


def _guard_stdout():
    """The contract is ONE JSON line on stdout: native libraries (NCCL's version banner under
    NCCL_DEBUG) write to fd 1 too, so fd 1 is pointed at stderr and the line goes to a duplicate of
    the original stdout."""
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def _emit(line):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    args = _args()
    _guard_stdout()
    cfg = mmot_inputs.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    elif cfg.batch > 1:
        run_batched(args, cfg)
    else:
        run_mmot(args, cfg)


if __name__ == "__main__":
    main()
