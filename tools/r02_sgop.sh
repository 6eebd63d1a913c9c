#!/bin/bash
# SG operator: parity (apply_block, golden, trajectories) and standalone timings
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -m gpu -x --durations=5 \
  -k "apply_block or golden or trajectory or drivers or ragged or reduced" > gpurun_out/pytest_sgop.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_sgop.log
: > gpurun_out/sgop_bench.log
for c in C1 C2 C3 C5L8; do
  timeout 600 python tools/sgop_bench.py $c 20 >> gpurun_out/sgop_bench.log 2>&1
done
for v in ${SGOP_VARIANTS:-"SGW_SGOP_NIL=2" "SGW_SGOP_IC=6" "SGW_SGOP_IC=12" "SGW_SGOP_S=3"}; do
  echo "== $v" >> gpurun_out/sgop_bench.log
  env $v timeout 300 python tools/sgop_bench.py C2 20 >> gpurun_out/sgop_bench.log 2>&1
done
