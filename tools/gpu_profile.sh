#!/bin/bash
# One gpurun call: GPU tests, default bench, launch list of the timed region
# (ncu --profile-from-start off; cold-cache, serialised), and one --set full
# capture each of the interior sweep and of the persistent PCG kernel.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?" >> gpurun_out/plain.log
timeout 900 ncu --set full -f --clock-control none --import-source on --profile-from-start off \
    -k regex:sweep_kernel -c 2 -o gpurun_out/prof_sweep $CMD > gpurun_out/ncu_sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/plain.log
timeout 900 ncu --set full -f --clock-control none --import-source on --profile-from-start off \
    -k regex:pcg_fused -c 1 -o gpurun_out/prof_pcg $CMD > gpurun_out/ncu_pcg.log 2>&1
echo "pcg rc=$?" >> gpurun_out/plain.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err
echo "bench rc=$?" >> gpurun_out/bench_full.err
