: > gpurun_out/bench_phase.log
for i in 1 2; do for pf in 1 0; do
  echo "== pf=$pf" >> gpurun_out/bench_phase.log
  SGW_PHASE_PREFETCH=$pf SGW_PCG=phase python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/bench_phase.log 2>&1
done; done
echo "== fused" >> gpurun_out/bench_phase.log
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/bench_phase.log 2>&1
