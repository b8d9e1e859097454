#!/bin/bash
# full GPU check: all GPU tests, the default bench (C4), C4 through the sharded context, C3, C5
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?"
timeout 600 python bench.py --shard --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_shard.json 2> gpurun_out/bench_c4_shard.err; echo "bench c4 shard rc=$?"
timeout 900 python bench.py --config C3 --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench c3 rc=$?"
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
for f in c4 c4_shard c3 c5; do echo "== $f"; cut -c1-600 gpurun_out/bench_$f.json; tail -2 gpurun_out/bench_$f.err; done
