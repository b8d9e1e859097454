#!/bin/bash
# GPU test pass: $1 = pytest -k expression (or "all"); logs under gpurun_out/
mkdir -p gpurun_out
if [ "$1" = "all" ] || [ -z "$1" ]; then
  timeout ${TMO:-2400} python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1
else
  timeout ${TMO:-2400} python -m pytest tests -m gpu -q -rf --durations=15 -k "$1" > gpurun_out/pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
