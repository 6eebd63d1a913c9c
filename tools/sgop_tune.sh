#!/bin/bash
# SG-operator shape sweep (standalone apply at C2); one line per config in gpurun_out/sgop_tune.log
set -u
mkdir -p gpurun_out
: > gpurun_out/sgop_tune.log
while read -r cfg; do
  [ -z "$cfg" ] && continue
  echo "== $cfg" >> gpurun_out/sgop_tune.log
  env $cfg timeout 300 python tools/sgop_bench.py C2 20 2>&1 | tail -1 >> gpurun_out/sgop_tune.log
done <<'CFGS'
SGW_SGOP_X=0
SGW_SGOP_LA=0
SGW_SGOP_IC=12
SGW_SGOP_IC=8
SGW_SGOP_IC=6
SGW_SGOP_DBG=1
SGW_SGOP_IC=8 SGW_SGOP_DBG=1
SGOP_WHICH=3
CFGS
