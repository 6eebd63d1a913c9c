"""Debug: the W=4 ragged LocalGroup case, per step (mode from SGW_PCG)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O  # noqa: E402
import paper_2512_23027_b200 as sg  # noqa: E402

nx, ny, px, py, W = (int(v) for v in sys.argv[1:6])
coeff = O.lognormal_coeff(nx, ny, 0.3, 0.5, 0.5, 2, 3)
t = O.triple_products(2, 3, 2)
kw = dict(params=sg.NewmarkParams(dt=2e-3), options=sg.SgOptions(tol=1e-10, store_full=True))
one = sg.SgSolver(nx, ny, px, py, coeff, t, **kw)
u0 = np.zeros((nx + 1) * (ny + 1))
force = sg.ForceSpec(node=O.nearest_node(nx, ny, 0.5, 0.5))
h1 = one.run(u0, u0, 8, force)
grp = sg.LocalGroup(W)
ranks = grp.solvers(nx, ny, px, py, coeff, t, **kw)
for r, h in enumerate(grp.map(lambda r: ranks[r].run(u0, u0, 8, force))):
    err = [np.linalg.norm(h.full_state[s] - h1.full_state[s]) / max(np.linalg.norm(h1.full_state[s]), 1e-300)
           for s in range(h1.full_state.shape[0])]
    print(os.environ.get("SGW_PCG", "default"), "rank", r, "its", h.iterations.tolist(), h1.iterations.tolist(),
          "err per step", ["%.1e" % e for e in err], flush=True)
grp.close()
