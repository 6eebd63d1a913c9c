"""Where does sgw_run's wall time go (C2)?  init_state vs steps, repeated."""
import os
import sys
import time

import numpy as np
import torch  # noqa: F401  (before libsgw_b200: torch must bind its own bundled NCCL first)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import bench  # noqa: E402
import paper_2512_23027_b200 as sg  # noqa: E402

c = bench.CONFIGS["C2"]
nx = c["nx"]
coeff = sg.lognormal_coeff(nx, nx, c["sigma"], c["b"], c["b"], c["L"], c["p_in"])
t = sg.triple_products(c["L"], c["p_in"], c["p_out"])
s = sg.SgSolver(nx, nx, c["px"], c["px"], coeff, t, alpha0=bench.ALPHA0, alpha1=bench.ALPHA1,
                params=sg.NewmarkParams(dt=c["dt"]), options=sg.SgOptions(tol=bench.TOL))
node = sg.nearest_node(nx, nx, 0.5, 0.5)
z = np.zeros((nx + 1) ** 2)
f = sg.ForceSpec(node=node, f0=bench.F0, t0=bench.T0)
for rep in range(3):
    w0 = time.perf_counter()
    s.init_state(z, z, f)
    w1 = time.perf_counter()
    s.advance(10)
    w2 = time.perf_counter()
    h = s.run(z, z, 10, f)
    w3 = time.perf_counter()
    print(f"init_state {w1 - w0:.3f} s  advance(10) {w2 - w1:.3f} s  run(10) {w3 - w2:.3f} s  stats {s.stats()}")

# table force (the bench's e2e leg): run(0) = pure API overhead (uploads + initial acceleration)
table = np.zeros((21, (nx + 1) ** 2))
tt = 0.0
for k in range(21):
    table[k, node] = sg.ricker(tt, bench.F0, bench.T0)
    tt += c["dt"]
s.options.probe_nodes = [node]
ft = sg.ForceSpec(table=table)
for rep in range(3):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    s.run(z, z, 0, sg.ForceSpec(table=table[:1].copy()))
    torch.cuda.synchronize()
    w1 = time.perf_counter()
    h = s.run(z, z, 20, ft)
    torch.cuda.synchronize()
    w2 = time.perf_counter()
    h2 = s.run(z, z, 20, f)
    torch.cuda.synchronize()
    w3 = time.perf_counter()
    print(f"run(0) {1e3 * (w1 - w0):.2f} ms  run(20, table) {1e3 * (w2 - w1):.2f} ms  run(20, point) {1e3 * (w3 - w2):.2f} ms  "
          f"iters {int(h.iterations.sum())} {int(h2.iterations.sum())} step_ms {s.stats().get('step_ms')}")
