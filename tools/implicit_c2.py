"""Reduced-memory mode at C2: device memory and PCG time per iteration vs the
explicit (stored S) path.  python tools/implicit_c2.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2512_23027_b200 as sg  # noqa: E402

c = bench.CONFIGS["C2"]
nx = c["nx"]
coeff = sg.lognormal_coeff(nx, nx, c["sigma"], c["b"], c["b"], c["L"], c["p_in"])
t = sg.triple_products(c["L"], c["p_in"], c["p_out"])
node = sg.nearest_node(nx, nx, 0.5, 0.5)
z = np.zeros((nx + 1) ** 2)
for imp in (False, True):
    s = sg.SgSolver(nx, nx, c["px"], c["px"], coeff, t, params=sg.NewmarkParams(dt=c["dt"]),
                    options=sg.SgOptions(tol=1e-10, implicit_schur=imp))
    s.run(z, z, 3, sg.ForceSpec(node=node))
    s.reset_stats()
    t0 = time.perf_counter()
    h = s.run(z, z, 10, sg.ForceSpec(node=node))
    wall = time.perf_counter() - t0
    st = s.stats()
    print(f"implicit_schur={imp}: device {s.device_bytes / 1e9:.2f} GB, PCG {st['pcg_ms'] / st['iterations']:.3f} ms"
          f"/iteration, {wall / 10 * 1e3:.2f} ms/step (wall), iterations {h.iterations.tolist()}")
    s.close()
