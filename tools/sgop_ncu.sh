set -u
mkdir -p gpurun_out
env ${SGOP_ENV:-} timeout 300 python tools/sgop_bench.py C2 20 > gpurun_out/sgop_plain.log 2>&1 && \
env ${SGOP_ENV:-} timeout 600 ncu --set full -f --clock-control none --import-source on -k regex:sgop_kernel -s 2 -c 1 -o gpurun_out/prof_sgop${SGOP_TAG:-0} python tools/sgop_bench.py C2 3 > gpurun_out/ncu_sgop${SGOP_TAG:-0}.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_sgop${SGOP_TAG:-0}.log
