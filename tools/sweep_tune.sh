set -u
for st in 4 5 6; do
  echo "== stages $st" >> gpurun_out/sweep_tune.log
  SGW_SWEEP_STAGES=$st timeout 300 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python3 -c "
import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])" >> gpurun_out/sweep_tune.log
done
