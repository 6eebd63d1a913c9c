#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/shard_dbg.log
for m in host phase; do
  for c in "26 26 4 4 4" "16 16 2 2 4" "24 24 4 4 4" "26 26 4 4 2"; do
    echo "== $m $c" >> gpurun_out/shard_dbg.log
    SGW_PCG=$m timeout 300 python tools/shard_dbg.py $c >> gpurun_out/shard_dbg.log 2>&1
  done
done
