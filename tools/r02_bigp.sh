#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "large_block" > gpurun_out/pytest_bigp.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_bigp.log
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -s --durations=0 -k "large_basis or l16" >> gpurun_out/pytest_bigp.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_bigp.log
