#!/bin/bash
# SG operator variants (JIT tuning hooks) at the configs given in $CFGS
set -u
mkdir -p gpurun_out
: > gpurun_out/sgop_var.log
for c in ${CFGS:-C2}; do
  for v in "$@"; do
    if [ "$v" = "-" ]; then e=""; else e="$v"; fi
    echo "== $c $v" >> gpurun_out/sgop_var.log
    env $e timeout 600 python tools/sgop_bench.py $c 20 2>&1 | tail -1 | cut -c1-400 >> gpurun_out/sgop_var.log
  done
done
