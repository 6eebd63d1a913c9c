mkdir -p gpurun_out; : > gpurun_out/sgop_size.log
for cfg in "3 6 3" "3 4 3" "3 3 3" "3 2 3" "2 6 3" "3 6 2" "3 4 2" "3 2 2"; do
  set -- $cfg
  echo "== L=$1 pin=$2 pout=$3" >> gpurun_out/sgop_size.log
  SGW_SGOP_G=4 SGW_SGOP_R=4 timeout 300 python tools/sgop_bench.py custom 20 256 8 $1 $2 $3 2>&1 | tail -1 >> gpurun_out/sgop_size.log
done
