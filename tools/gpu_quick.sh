#!/bin/bash
# quick loop: selected GPU tests ($1 = pytest -k expr or "all"), bench, launch list, ncu of $2 kernel regex
mkdir -p gpurun_out
if [ "$1" = "all" ]; then K=""; else K="-k $1"; fi
timeout 1200 python -m pytest tests -m gpu -x -q $K > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ -n "$2" ]; then
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 20 -c 1 -o gpurun_out/prof_$2 $CMD > gpurun_out/ncu_full.log 2>&1
fi
echo done
