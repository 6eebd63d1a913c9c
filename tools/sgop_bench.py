"""Standalone SG-operator apply (for ncu captures and scaling experiments):
   python tools/sgop_bench.py [C1|C2|C3|C4|C5L8] [reps]
   python tools/sgop_bench.py custom <reps> <nx> <px> <L> <p_in> <p_out>
Prints one JSON line: time per launch (L2 flushed before each), algorithmic
bytes / flops (kernel_profile) and the roofline fractions."""
import json
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
ms = s.bench_kernel(2, reps=reps)
kp = s.kernel_profile(False)
nbytes, flops = kp["sg_operator"][2], kp["sg_operator_flops"]
peaks = bench.load_peaks() if hasattr(bench, "load_peaks") else {}
bw = peaks.get("hbm_gbs", 6549.8)
fp64 = bench.FP64_TFLOPS if hasattr(bench, "FP64_TFLOPS") else 33.5
t_roof = max(nbytes / (bw * 1e9), flops / (fp64 * 1e12)) * 1e3
print(json.dumps({"config": name, "n_in": t.n_input, "P+1": t.n_output, "us": ms * 1e3, "bytes": nbytes,
                  "flops": flops, "GBs": nbytes / (ms / 1e3) / 1e9, "TFLOPs": flops / (ms / 1e3) / 1e12,
                  "hbm_frac": nbytes / (ms / 1e3) / 1e9 / bw, "roofline_us": t_roof * 1e3,
                  "roofline_frac": t_roof / ms}))
