#!/bin/bash
# gpurun_out/ of one tools/gpu_round.sh (+ r02_suite.sh) call -> profiles/<tag>_*: the JSON line of every bench
# log, the GPU test log, the reduced-memory comparison, then the ncu summaries (summarize_ncu.py).
set -u
tag=${1:?usage: tools/collect_round.sh <tag>}
o=gpurun_out
json() {  # <log> <profiles name>: last JSON line of a bench log
  [ -f "$o/$1" ] || return 0
  grep '^{' "$o/$1" | tail -1 > "profiles/${tag}_$2.json"
  [ -s "profiles/${tag}_$2.json" ] || rm -f "profiles/${tag}_$2.json"
}
json bench_full.log bench_C2
json bench_C1.log bench_C1
json bench_C3.log bench_C3
json bench_C5L8.log bench_C5L8
json bench_ref.log bench_C2_reference
json bench_C2_shard1.log bench_C2_shard1
json solo_C4_w4.log solo_C4_w4
json solo_C4_w8.log solo_C4_w8
[ -f $o/pytest_gpu.log ] && cp $o/pytest_gpu.log profiles/${tag}_gpu_tests.log
[ -f $o/implicit_c2.txt ] && cp $o/implicit_c2.txt profiles/${tag}_implicit_c2.txt
python tools/summarize_ncu.py "$tag"
python tools/results_table.py "$tag"
