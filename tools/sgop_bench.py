"""Standalone SG-operator apply at a BASELINE config (for ncu captures):
   python tools/sgop_bench.py [C1|C2] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import bench  # noqa: E402
import paper_2512_23027_b200 as sg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
c = bench.CONFIGS[name]
nx = c["nx"]
coeff = sg.lognormal_coeff(nx, nx, c["sigma"], c["b"], c["b"], c["L"], c["p_in"])
t = sg.triple_products(c["L"], c["p_in"], c["p_out"])
s = sg.SgSolver(nx, nx, c["px"], c["px"], coeff, t, params=sg.NewmarkParams(dt=c["dt"]))
ms = s.bench_kernel(2, reps=reps)
print(f"{name}: sg operator {ms * 1e3:.1f} us/launch, {151898400 / (ms / 1e3) / 1e9:.0f} GB/s (C2 bytes)")
