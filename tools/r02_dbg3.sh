#!/bin/bash
set -u
mkdir -p gpurun_out
: > gpurun_out/shard_dbg.log
for off in 1 0; do
  echo "== SGOP_OFF=$off host 26 26 4 4 2" >> gpurun_out/shard_dbg.log
  SGW_SGOP_OFF=$off SGW_PCG=host timeout 300 python tools/shard_dbg.py 26 26 4 4 2 >> gpurun_out/shard_dbg.log 2>&1
done
