#!/bin/bash
# single-pass sweep tile product: parity subset, then C2 / C1 / C3 short benches
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -m gpu -x --durations=8 -p no:cacheprovider > gpurun_out/pytest_sweep.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_sweep.log
: > gpurun_out/bench_sweep.log
for c in C2 C1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/bench_sweep.log 2>&1
done
