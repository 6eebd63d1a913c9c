#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_generic.py tests/test_outputs.py tests/test_golden.py tests/test_gpu_precond.py -q -m gpu --durations=25 -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
: > gpurun_out/bench_c1.log
for c in C1 C2; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/bench_c1.log 2>&1
done
