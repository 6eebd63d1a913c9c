set -u
for cfg in "0 1 0" "0 0 0" "4 0 0" "0 0 4"; do
  set -- $cfg
  env="SGW_SGOP_PF=$3"
  [ "$1" != "0" ] && env="$env SGW_SGOP_IC=$1"
  [ "$2" != "0" ] && env="$env SGW_SGOP_DBG=$2"
  echo "== IC=$1 DBG=$2 PF=$3" >> gpurun_out/sgop_tune.log
  env $env timeout 300 python tools/sgop_bench.py C2 20 >> gpurun_out/sgop_tune.log 2>&1
done
timeout 300 python tools/sgop_bench.py C1 20 >> gpurun_out/sgop_tune.log 2>&1
