#!/bin/bash
# One gpurun call: GPU tests, the default bench, a launch list of the timed
# region and --set full captures of the sweep and persistent PCG kernels.
set -u
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.ncu-rep  # stale captures must not feed summarize_ncu
# (the GPU test suite runs in its own call: tools/r02_suite.sh, ~50 min with the full-size parity tests)
timeout 900 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err
echo "bench rc=$?" >> gpurun_out/bench_full.err
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
echo "rc=$?" >> gpurun_out/plain.log
timeout 600 python tools/sgop_bench.py C2 5 > gpurun_out/sgop_plain.log 2>&1 && \
timeout 900 ncu --set full -f --clock-control none --import-source on -k regex:sgop_kernel -s 2 -c 1 \
    -o gpurun_out/prof_sgop python tools/sgop_bench.py C2 5 > gpurun_out/ncu_sgop.log 2>&1
echo "rc=$?" >> gpurun_out/plain.log
timeout 900 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3.log 2> gpurun_out/bench_C3.err
echo "C3 rc=$?" >> gpurun_out/bench_C3.err
timeout 600 python bench.py --config C1 > gpurun_out/bench_C1.log 2> gpurun_out/bench_C1.err
echo "C1 rc=$?" >> gpurun_out/bench_C1.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err
echo "ref rc=$?" >> gpurun_out/bench_ref.err
timeout 900 python bench.py --config C5L8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C5L8.log 2> gpurun_out/bench_C5L8.err
echo "C5L8 rc=$?" >> gpurun_out/bench_C5L8.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --force-shard > gpurun_out/bench_C2_shard1.log 2> gpurun_out/bench_C2_shard1.err
echo "shard1 rc=$?" >> gpurun_out/bench_C2_shard1.err
for W in 8 4; do
  timeout 900 python bench.py --config C4 --solo-rank 0 --solo-world $W --steps 20 > gpurun_out/solo_C4_w$W.log 2>&1
  echo "rc=$?" >> gpurun_out/solo_C4_w$W.log
done
