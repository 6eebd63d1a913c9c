#!/bin/bash
# Quick GPU check: optional GPU tests (-k filter in $TESTS), then one short
# bench per environment assignment given as arguments ("-" = defaults), e.g.
#   TESTS="pcg or golden" bash tools/quick.sh - SGW_PCG_L2PF=4
set -u
mkdir -p gpurun_out
if [ -n "${TESTS:-}" ]; then
  if [ "$TESTS" = all ]; then timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/quick_test.log 2>&1
  else timeout 900 python -m pytest tests -q -m gpu -x -k "$TESTS" > gpurun_out/quick_test.log 2>&1; fi
  echo "rc=$?" >> gpurun_out/quick_test.log
fi
i=0
for v in "$@"; do
  if [ "$v" = "-" ]; then e=""; else e="$v"; fi
  env $e timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/quick_$i.log 2>&1
  echo "# $v" >> gpurun_out/quick_$i.log
  i=$((i+1))
done
