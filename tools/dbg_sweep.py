"""Debug helper: run a few steps at a chosen size and compare with the oracle."""
import sys
import numpy as np
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O
import paper_2512_23027_b200 as sg

nx, px, L, pin, pout, steps = (int(v) for v in sys.argv[1:7])
coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, L, pin)
t = O.triple_products(L, pin, pout)
g = sg.SgSolver(nx, nx, px, px, coeff, t, params=sg.NewmarkParams(dt=1e-3),
                options=sg.SgOptions(tol=1e-10, store_full=True))
node = O.nearest_node(nx, nx, 0.5, 0.5)
z = np.zeros((nx + 1) ** 2)
hg = g.run(z, z, steps, sg.ForceSpec(node=node))
print("gpu iterations", hg.iterations)
if len(sys.argv) > 7:
    c = O.SgSolver(nx, nx, px, px, coeff, t, dt=1e-3, tol=1e-10)
    hc = c.run(z, z, steps, force_node=node, store_full=True)
    print("cpu iterations", hc["iterations"])
    print("rel", np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]))
