#!/bin/bash
# SG-operator shape sweep (standalone apply at C2): one line per environment
# assignment given as an argument ("-" = defaults) in gpurun_out/sgop_tune.log
set -u
mkdir -p gpurun_out
: > gpurun_out/sgop_tune.log
for cfg in "$@"; do
  echo "== $cfg" >> gpurun_out/sgop_tune.log
  if [ "$cfg" = "-" ]; then cfg=""; fi
  env $cfg timeout 300 python tools/sgop_bench.py ${SGOP_CONFIG:-C2} 20 2>&1 | tail -1 >> gpurun_out/sgop_tune.log
done
