"""Sharded C2 on one GPU through the in-process communicator (LocalGroup):
W ranks vs the single-GPU solver, 8 Newmark steps (correctness at scale)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import bench  # noqa: E402
import paper_2512_23027_b200 as sg  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = bench.CONFIGS["C2"]
nx = c["nx"]
coeff = sg.lognormal_coeff(nx, nx, c["sigma"], c["b"], c["b"], c["L"], c["p_in"])
t = sg.triple_products(c["L"], c["p_in"], c["p_out"])
node = sg.nearest_node(nx, nx, 0.5, 0.5)
kw = dict(alpha0=bench.ALPHA0, alpha1=bench.ALPHA1, params=sg.NewmarkParams(dt=c["dt"]),
          options=sg.SgOptions(tol=bench.TOL, probe_nodes=[node]))
z = np.zeros((nx + 1) ** 2)
f = sg.ForceSpec(node=node, f0=bench.F0, t0=bench.T0)
one = sg.SgSolver(nx, nx, c["px"], c["px"], coeff, t, **kw)
h1 = one.run(z, z, 8, f)
u1 = one.state()
del one
grp = sg.LocalGroup(W)
t0 = time.perf_counter()
ranks = grp.solvers(nx, nx, c["px"], c["px"], coeff, t, **kw)
print(f"W={W}: sharded setup {time.perf_counter() - t0:.1f} s")
hs = grp.map(lambda r: ranks[r].run(z, z, 8, f))
us = grp.map(lambda r: ranks[r].state())
for r in range(W):
    print(f"rank {r}: iterations {hs[r].iterations.tolist()} vs {h1.iterations.tolist()}, "
          f"state rel {np.linalg.norm(us[r] - u1) / np.linalg.norm(u1):.2e}, "
          f"probe rel {np.abs(hs[r].probe_mean - h1.probe_mean).max() / np.abs(h1.probe_mean).max():.2e}")
