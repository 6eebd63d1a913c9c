: > gpurun_out/sgop_bench.log
for v in "SGW_SGOP_IC=12" "SGW_SGOP_G=2 SGW_SGOP_RP=6" "SGW_SGOP_G=2 SGW_SGOP_RP=6 SGW_SGOP_DBG=2" "SGW_SGOP_G=2 SGW_SGOP_RP=4" "SGW_SGOP_G=2 SGW_SGOP_RP=6 SGW_SGOP_IC=16" "SGW_SGOP_IC=12 SGW_SGOP_NIL=6" "SGW_SGOP_G=4 SGW_SGOP_RP=4" "SGW_SGOP_G=4 SGW_SGOP_RP=3"; do
  echo "== $v" >> gpurun_out/sgop_bench.log
  env $v timeout 300 python tools/sgop_bench.py C2 20 >> gpurun_out/sgop_bench.log 2>&1
done
for v in "SGW_SGOP_G=4" "SGW_SGOP_G=4 SGW_SGOP_RP=3" "SGW_SGOP_G=8 SGW_SGOP_RP=2" "SGW_SGOP_G=2 SGW_SGOP_RP=4"; do
  echo "== C3 $v" >> gpurun_out/sgop_bench.log
  env $v timeout 300 python tools/sgop_bench.py C3 10 >> gpurun_out/sgop_bench.log 2>&1
done
