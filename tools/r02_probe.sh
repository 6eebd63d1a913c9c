#!/bin/bash
# Round-2 first GPU call: host resources, FP64 peak, GPU test suite.
set -u
mkdir -p gpurun_out tools/bin
{ nproc; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; } > gpurun_out/host_probe.txt 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/bench_fp64 tools/bench_fp64.cu && \
  timeout 300 tools/bin/bench_fp64 > gpurun_out/fp64_peak.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
