#!/bin/bash
# ncu --set full captures of the SG operator at C2: default, math only (DBG=2), stream only (DBG=1);
# raw metric pages as CSV in gpurun_out/
set -u
mkdir -p gpurun_out
for v in "" "SGW_SGOP_DBG=2" "SGW_SGOP_DBG=1"; do
  tag=${v##*=}; [ -z "$v" ] && tag=def
  env $v timeout 600 ncu --set full -f --clock-control none --import-source on -k regex:sgop_kernel -s 2 -c 1 \
    -o gpurun_out/prof_sgop_$tag python tools/sgop_bench.py ${SGOP_CONFIG:-C2} 3 > gpurun_out/ncu_sgop_$tag.log 2>&1
  ncu -i gpurun_out/prof_sgop_$tag.ncu-rep --page raw --csv > gpurun_out/sgop_raw_$tag.csv 2>/dev/null
done
