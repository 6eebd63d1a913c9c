set -u
for cfg in "0 0" "1 7" "2 3" "3 3" "4 2" "4 3" "5 2"; do
  set -- $cfg
  env="SGW_SGOP_PF=0"
  [ "$1" != "0" ] && env="$env SGW_SGOP_G=$1"
  [ "$2" != "0" ] && env="$env SGW_SGOP_R=$2"
  echo "== G=$1 R=$2" >> gpurun_out/sgop_tune.log
  env $env timeout 300 python tools/sgop_bench.py C2 20 >> gpurun_out/sgop_tune.log 2>&1
done
