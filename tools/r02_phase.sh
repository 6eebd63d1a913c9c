#!/bin/bash
# phase-split PCG: the multi-rank bug, overhead (launch list), C1 L2-keep on/off
set -u
mkdir -p gpurun_out
: > gpurun_out/shard_pcg_dbg.log
for c in "24 24 4 4 4" "24 24 3 2 2" "16 16 2 2 4"; do
  echo "== $c" >> gpurun_out/shard_pcg_dbg.log
  timeout 300 python tools/shard_pcg_dbg.py $c >> gpurun_out/shard_pcg_dbg.log 2>&1
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
SGW_PCG=phase timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_phase.csv $CMD > gpurun_out/ncu_phase.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_phase.log
: > gpurun_out/bench_c1.log
for k in 1 0; do
  SGW_PCG_L2KEEP=$k timeout 600 python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/bench_c1.log 2>&1
done
SGW_PCG=phase timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_phase.log 2>&1
