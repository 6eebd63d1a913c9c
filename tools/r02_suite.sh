#!/bin/bash
# full GPU suite (no -x: every failure), then the default bench
set -u
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.ncu-rep
timeout 3000 python -m pytest tests -q -m gpu --durations=30 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err
echo "bench rc=$?" >> gpurun_out/bench_full.err
