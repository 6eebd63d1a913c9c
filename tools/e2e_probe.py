"""Where does sgw_run's wall time go (C2)?  init_state vs steps, repeated."""
import os
import sys
import time

import numpy as np

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
