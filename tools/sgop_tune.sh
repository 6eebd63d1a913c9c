set -u
for cfg in "jout 0 0 0" "jout 4 0 0" "jout 2 6 0" "jout 2 4 0" "xres 0 0 0"; do
  set -- $cfg
  env="SGW_SGOP_MODE=$1"
  [ "$2" != "0" ] && env="$env SGW_SGOP_R=$2"
  [ "$3" != "0" ] && env="$env SGW_SGOP_IC=$3"
  echo "== $cfg" >> gpurun_out/sgop_tune.log
  env $env timeout 300 python tools/sgop_bench.py C2 20 >> gpurun_out/sgop_tune.log 2>&1
done
