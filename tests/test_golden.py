"""Golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py).

CPU: the oracle still reproduces every fixture, so the fixtures and the pinned
oracle cannot drift apart.  GPU: the sm_100a path, called through the C ABI,
reproduces every fixture without the oracle in the loop.  Tolerances follow
the reference tests: block apply 1e-12 (test_sg.cpp:51-73), Schur/NN2 1e-10,
trajectory 1e-8 relative L2 with PCG iterations within +-1 per step
(BASELINE parity contract)."""
import glob
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
IDS = [os.path.basename(p)[:-4] for p in GOLDEN]


def load(path):
    z = np.load(path)
    nx, ny, px, py, L, pin, pout, steps, node = (int(v) for v in z["spec"])
    sigma, b, dt, tol, a0, a1 = (float(v) for v in z["params"])
    return z, dict(nx=nx, ny=ny, px=px, py=py, steps=steps, node=node, dt=dt, tol=tol, a0=a0, a1=a1)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_fixtures_present():
    assert len(GOLDEN) >= 4


@pytest.mark.parametrize("path", GOLDEN, ids=IDS)
def test_oracle_reproduces_golden(path):
    z, c = load(path)
    t = O.Tensor(int(z["coeff"].shape[0]), int(z["n_output"]), z["ti"], z["tj"], z["tk"], z["tv"])
    s = O.SgSolver(c["nx"], c["ny"], c["px"], c["py"], z["coeff"], t, alpha0=c["a0"], alpha1=c["a1"],
                   dt=c["dt"], tol=c["tol"])
    for op in ("transient", "mass", "stiffness"):
        assert rel(s.apply_block(z["x_block"], op), z["y_" + op]) <= 1e-14
    assert rel(s.schur_matvec(z["x_iface"]), z["schur_x"]) <= 1e-13
    assert rel(s.apply_nn2(z["x_iface"]), z["nn2_x"]) <= 1e-12
    if "coarse" in z:
        assert rel(s.coarse_operator(), z["coarse"]) <= 1e-13
    u0 = z["u0"]
    if c["node"] >= 0:
        h = s.run(u0, 0 * u0, c["steps"], force_node=c["node"], f0=10.0, t0=0.1, store_full=True)
    else:
        h = s.run(u0, 0 * u0, c["steps"], store_full=True)
    assert np.array_equal(h["iterations"], z["iterations"])
    assert rel(h["full"], z["full"]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLDEN, ids=IDS)
def test_gpu_reproduces_golden(gpu, path):
    import paper_2512_23027_b200 as sg
    z, c = load(path)
    t = sg.TripleTensor(int(z["coeff"].shape[0]), int(z["n_output"]), z["ti"], z["tj"], z["tk"], z["tv"])
    g = sg.SgSolver(c["nx"], c["ny"], c["px"], c["py"], z["coeff"], t, alpha0=c["a0"], alpha1=c["a1"],
                    params=sg.NewmarkParams(dt=c["dt"]), options=sg.SgOptions(tol=c["tol"], store_full=True))
    assert rel(g.apply_block_transient(z["x_block"]), z["y_transient"]) <= 1e-12
    assert rel(g.apply_block_mass(z["x_block"]), z["y_mass"]) <= 1e-12
    assert rel(g.apply_block_stiffness(z["x_block"]), z["y_stiffness"]) <= 1e-12
    assert rel(g.schur().matvec(z["x_iface"]), z["schur_x"]) <= 1e-10
    assert rel(g.schur().apply_nn2(z["x_iface"]), z["nn2_x"]) <= 1e-10
    if "coarse" in z:
        assert rel(g.schur().coarse_operator(), z["coarse"]) <= 1e-10
    u0 = z["u0"]
    force = sg.ForceSpec(node=c["node"], f0=10.0, t0=0.1) if c["node"] >= 0 else None
    h = g.run(u0, 0 * u0, c["steps"], force)
    assert np.all(np.abs(h.iterations - z["iterations"]) <= 1)
    assert rel(h.full_state, z["full"]) <= 1e-8
