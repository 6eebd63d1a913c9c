set -u
for cfg in "0 0 0" "0 1 0" "1 4 2" "2 2 3" "1 2 4" "2 4 1"; do
  set -- $cfg
  env="SGW_SGOP_PF=0"
  [ "$1" != "0" ] && env="$env SGW_SGOP_G=$1"
  [ "$2" != "0" ] && env="$env SGW_SGOP_GI=$2"
  [ "$3" != "0" ] && env="$env SGW_SGOP_R=$3"
  echo "== GJ=$1 GI=$2 R=$3" >> gpurun_out/sgop_tune.log
  env $env timeout 300 python tools/sgop_bench.py C2 20 >> gpurun_out/sgop_tune.log 2>&1
done
