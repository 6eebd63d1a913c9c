#!/bin/bash
# Sharded path: GPU parity suite, C3 two-rank cross-check, phase-split vs
# persistent PCG at C2, 1-rank NCCL (torchrun) and a C4 solo-rank loopback.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --durations=15 > gpurun_out/pytest_parity.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/bench_fused.log 2>&1; echo "rc=$?" >> gpurun_out/bench_fused.log
SGW_PCG=phase timeout 600 $B > gpurun_out/bench_phase.log 2>&1; echo "rc=$?" >> gpurun_out/bench_phase.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --force-shard > gpurun_out/bench_nccl1.log 2>&1
echo "rc=$?" >> gpurun_out/bench_nccl1.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "two_rank" > gpurun_out/pytest_c3w2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_c3w2.log
for W in 8 4; do
  timeout 900 python bench.py --config C4 --solo-rank 0 --solo-world $W --steps 20 > gpurun_out/solo_c4_w$W.log 2>&1
  echo "rc=$?" >> gpurun_out/solo_c4_w$W.log
done
