#!/bin/bash
# usage: tools/ncu_one.sh <kernel-regex> <skip> <name> [bench args...]
set -u
K=$1; SKIP=$2; NAME=$3; shift 3
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $*"
mkdir -p gpurun_out
timeout 600 $CMD > gpurun_out/plain_$NAME.log 2>&1 && \
timeout 900 ncu --set full -f --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 \
    -o gpurun_out/prof_$NAME $CMD > gpurun_out/ncu_$NAME.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$NAME.log
