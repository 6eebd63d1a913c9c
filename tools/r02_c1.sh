#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/bench_c1.log
for v in "X=1" "SGW_SWEEP_CS=8" "SGW_PCG_GRID=148" "SGW_PCG_GRID=64" "SGW_PCG_GRID=32"; do
  echo "== $v" >> gpurun_out/bench_c1.log
  env $v timeout 600 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/bench_c1.log 2>&1
done
for v in "X=1" "SGW_PCG_GRID=148"; do
  echo "== C2 $v" >> gpurun_out/bench_c1.log
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/bench_c1.log 2>&1
done
: > gpurun_out/sgop_bench.log
for v in "X=1" "SGW_SGOP_RP=4 SGW_SGOP_CPS=2" "SGW_SGOP_RP=4 SGW_SGOP_CPS=2 SGW_SGOP_IC=12" "SGW_SGOP_RP=16 SGW_SGOP_G=1"; do
  echo "== $v" >> gpurun_out/sgop_bench.log
  env $v timeout 300 python tools/sgop_bench.py C2 20 >> gpurun_out/sgop_bench.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_generic.py tests/test_outputs.py -q -m gpu --durations=20 -p no:cacheprovider > gpurun_out/pytest_parity.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
