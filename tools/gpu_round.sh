#!/bin/bash
# full GPU suite + bench lines of the given configs (default C4); logs under gpurun_out/r2/
mkdir -p gpurun_out/r2
O=gpurun_out/r2
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout ${TMO:-2400} python -m pytest tests -m gpu -q -rf --durations=20 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -25 $O/pytest_gpu.log
fi
for c in ${CONFIGS:-C4}; do
  timeout 900 python bench.py --config $c ${BENCH_ARGS} > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
  head -c 1500 $O/bench_$c.json; echo; tail -2 $O/bench_$c.err
done
