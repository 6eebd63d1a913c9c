#!/bin/bash
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
SGW_PCG=phase SGW_PHASE_NOGRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_phase.csv $CMD > gpurun_out/ncu_phase.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_phase.log
SGW_PCG=phase timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_phase.log 2>&1
SGW_PCG=phase SGW_PHASE_NOGRAPH=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/bench_phase.log 2>&1
timeout 3000 python -m pytest tests/test_gpu_fullsize.py -q -m gpu --durations=0 -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_full.log
