"""Debug: one interface PCG solve on a W-rank LocalGroup, host vs phase drivers vs one GPU."""
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
os.environ["SGW_PCG"] = "host"
one = sg.SgSolver(nx, ny, px, py, coeff, t, **kw)
b = np.sin(0.37 * np.arange(one.n_global) + 0.1)
x1, r1 = one.pcg(b)
print("single", r1["iterations"], np.round(r1["residual_history"][:8], 6).tolist(), flush=True)
for mode in ["host", "phase"]:
    os.environ["SGW_PCG"] = mode
    grp = sg.LocalGroup(W)
    ranks = grp.solvers(nx, ny, px, py, coeff, t, **kw)
    res = grp.map(lambda r: ranks[r].pcg(b))
    for r, (x, rep) in enumerate(res):
        print(mode, "rank", r, rep["iterations"], np.round(rep["residual_history"][:8], 6).tolist(),
              "x err %.2e" % (np.abs(x - x1).max() / np.abs(x1).max()), flush=True)
    z = grp.map(lambda r: ranks[r].schur().apply_nn2(b))
    print(mode, "nn2 err", ["%.1e" % (np.abs(zz - one.schur().apply_nn2(b)).max()) for zz in z], flush=True)
    del ranks
    grp.close()
