#!/bin/bash
# One gpurun call: default bench, launch list (ncu, cold-cache serialised), and
# one --set full capture of the PCG tile-SYMV and of the sweep GEMV.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err
echo "bench rc=$?" >> gpurun_out/bench_full.err
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?" >> gpurun_out/plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:symv_tiles -s 4 -c 2 \
    -o gpurun_out/prof_symv $CMD > gpurun_out/ncu_symv.log 2>&1
echo "symv rc=$?" >> gpurun_out/plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_n_sub -s 200 -c 2 \
    -o gpurun_out/prof_sweep $CMD > gpurun_out/ncu_sweep.log 2>&1
echo "sweep rc=$?" >> gpurun_out/plain.log
