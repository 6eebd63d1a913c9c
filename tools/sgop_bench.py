"""Standalone SG-operator apply (for ncu captures and scaling experiments):
   python tools/sgop_bench.py [C1|C2|C3] [reps]
   python tools/sgop_bench.py custom <reps> <nx> <px> <L> <p_in> <p_out>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import bench  # noqa: E402
import paper_2512_23027_b200 as sg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if name == "custom":
    nx, px, L, pin, pout = (int(v) for v in sys.argv[3:8])
    c = dict(nx=nx, px=px, L=L, p_in=pin, p_out=pout, sigma=0.3, b=0.5, dt=1e-3)
else:
    c = bench.CONFIGS[name]
nx = c["nx"]
coeff = sg.lognormal_coeff(nx, nx, c["sigma"], c["b"], c["b"], c["L"], c["p_in"])
t = sg.triple_products(c["L"], c["p_in"], c["p_out"])
s = sg.SgSolver(nx, nx, c["px"], c["px"], coeff, t, params=sg.NewmarkParams(dt=c["dt"]))
which = int(os.environ.get("SGOP_WHICH", "2"))  # 3: the step's form with the M x2 term
ms = s.bench_kernel(which, reps=reps)
n = (nx - 1) ** 2
pairs = len({(i, j) for i, j, k in zip(t.i, t.j, t.k)} | {(i, k) for i, j, k in zip(t.i, t.j, t.k)})
nbytes = 8.0 * n * (3 * t.n_input + 2 * t.n_output)
print(f"{name} nx={nx} n_in={t.n_input} P+1={t.n_output} pairs={pairs}: {ms * 1e3:.1f} us/launch, "
      f"{nbytes / (ms / 1e3) / 1e9:.0f} GB/s, {ms * 1e6 / n / pairs * 1e3:.2f} ps per node-pair")
