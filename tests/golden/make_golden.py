"""Generate the committed golden fixtures under tests/golden/ from the CPU oracle.

The reference (C++20 + Eigen, `proj/`) cannot be built in this image, so these
fixtures come from the oracle (`oracle/`).  The oracle is pinned to the
reference's recorded answers by tests/test_oracle.py (proj/test_output.txt,
proj/tests/*.cpp known-answer checks).  The fixtures freeze its outputs on small
seeded problems.  The GPU tests can then check parity without the oracle, and
the CPU suite checks that the oracle still reproduces them bit-for-bit.

    python tests/golden/make_golden.py       # rewrites tests/golden/*.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))

import oracle as O  # noqa: E402

# name: (nx, ny, px, py, sigma, b, L, p_in, p_out, dt, tol, alpha0, alpha1, source, n_steps)
#   source "ricker": Ricker point source f0=10 Hz, t0=0.1 at (0.5, 0.5), zero initial state
#   source "pulse":  Gaussian initial displacement (test_sg.cpp:218-272), no forcing
CASES = {
    "g1_ricker_12x12_2x2": (12, 12, 2, 2, 0.3, 0.5, 2, 2, 2, 1e-3, 1e-10, 0.5445, 0.0174, "ricker", 10),
    "g2_pulse_16x12_4x2": (16, 12, 4, 2, 0.25, 1.0, 3, 2, 3, 1e-2, 1e-10, 0.5445, 0.0174, "pulse", 8),
    "g3_ragged_14x10_4x3": (14, 10, 4, 3, 0.3, 0.5, 2, 3, 2, 5e-3, 1e-10, 0.5445, 0.0174, "pulse", 6),
    "g4_undamped_8x8_1x2": (8, 8, 1, 2, 0.2, 1.0, 1, 2, 2, 2e-2, 1e-12, 0.0, 0.0, "pulse", 6),
}


def make(name, spec):
    nx, ny, px, py, sigma, b, L, pin, pout, dt, tol, a0, a1, source, steps = spec
    coeff = O.lognormal_coeff(nx, ny, sigma, b, b, L, pin)
    t = O.triple_products(L, pin, pout)
    s = O.SgSolver(nx, ny, px, py, coeff, t, alpha0=a0, alpha1=a1, dt=dt, tol=tol)
    rng = np.random.default_rng(sum(map(ord, name)))
    x_block = rng.uniform(-1, 1, s.n_terms * s.n_dofs)
    x_iface = rng.uniform(-1, 1, s.n_global)
    nodes = (nx + 1) * (ny + 1)
    if source == "ricker":
        u0 = np.zeros(nodes)
        node = O.nearest_node(nx, ny, 0.5, 0.5)
        h = s.run(u0, u0, steps, force_node=node, f0=10.0, t0=0.1, store_full=True)
    else:
        u0 = O.gaussian_pulse(nx, ny)
        node = -1
        h = s.run(u0, 0 * u0, steps, store_full=True)
    out = dict(
        spec=np.array([nx, ny, px, py, L, pin, pout, steps, node]),
        params=np.array([sigma, b, dt, tol, a0, a1]),
        coeff=coeff, ti=t.i, tj=t.j, tk=t.k, tv=t.v, n_output=np.array(t.n_output),
        u0=u0,
        x_block=x_block, y_transient=s.apply_block(x_block, "transient"),
        y_mass=s.apply_block(x_block, "mass"), y_stiffness=s.apply_block(x_block, "stiffness"),
        x_iface=x_iface, schur_x=s.schur_matvec(x_iface), nn2_x=s.apply_nn2(x_iface),
        iterations=h["iterations"], full=h["full"],
    )
    if s.n_corner:
        out["coarse"] = s.coarse_operator()
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: n_global={s.n_global} n_corner={s.n_corner} iterations={list(h['iterations'])}")


if __name__ == "__main__":
    for k, v in CASES.items():
        make(k, v)
