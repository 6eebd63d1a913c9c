#!/bin/bash
# Full-size parity tests (C2 100 steps, C3 / C5L8 per-subdomain + cross-checks)
set -u
mkdir -p gpurun_out
timeout 3000 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py::test_pcg_matches_oracle_iterations \
  -q -m gpu -s --durations=0 ${EXTRA:-} > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_full.log
