"""Pins the CPU oracle to the reference's own tests and recorded numbers.

Each test cites the reference test (proj/tests/...) or recorded output
(proj/test_output.txt) it reproduces.  CPU only.
"""
import math

import numpy as np
import pytest

import oracle as O
import refmodel as R


def rand(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


# --------------------------------------------------------------- inputs ----
def test_multi_index_counts_and_guard_lifted():
    # test_pce.cpp: sizes C(L+p, p); p_in > p_out accepted (guard src/pce.cpp:97-99 lifted)
    t = O.triple_products(3, 6, 3)
    assert (t.n_input, t.n_output) == (math.comb(9, 6), math.comb(6, 3))
    g = t.dense()
    assert np.allclose(g, np.transpose(g, (0, 2, 1)))


@pytest.mark.parametrize("L,pin,pout", [(2, 2, 2), (3, 2, 3), (2, 4, 2), (3, 6, 3), (1, 1, 1)])
def test_triple_products_closed_form_vs_quadrature(L, pin, pout):
    # test_pce.cpp:79-130 / acceptance criterion 9 (tensor diff <= 1e-10; recorded 4.17e-14)
    a = O.triple_products(L, pin, pout).dense()
    b = O.triple_products(L, pin, pout, quadrature=True).dense()
    assert np.abs(a - b).max() <= 1e-10


def test_triple_products_zero_index_is_identity():
    # <psi_0 psi_j psi_k> = delta_jk (orthonormal basis)
    g = O.triple_products(3, 2, 3).dense()
    assert np.allclose(g[0], np.eye(g.shape[1]), atol=1e-14)


def test_kle_roots_satisfy_characteristic_equations():
    # src/kle.cpp:40-68: even tan(wT) = c/w, odd tan(wT) = -w/c on T = 1/2
    lam = O.kle_lambdas(8, 8, 1.0, 0.5, 0.5, 6)
    assert np.all(np.diff(lam) <= 0) and np.all(lam > 0)
    assert lam.sum() < 1.0  # truncated variance fraction of a unit-variance field


def test_lognormal_mean_term_closed_form():
    # src/lognormal.cpp:19-24: c_0 = exp(g0 + 1/2 sum g_v^2) >= exp(g0); sigma = 0 -> constant
    c = O.lognormal_coeff(6, 6, 0.0, 1.0, 1.0, 3, 2, g0=0.1)
    assert np.allclose(c[0], math.exp(0.1)) and np.abs(c[1:]).max() == 0.0
    c = O.lognormal_coeff(6, 6, 0.3, 0.5, 0.5, 2, 4)
    assert np.all(c[0] > 1.0)


# --------------------------------------------------------- operators -------
def test_block_stiffness_matches_explicit_tensor_sum():
    # test_sg.cpp:51-73 (<= 1e-12 relative)
    nx, L = 6, 2
    c = O.lognormal_coeff(nx, nx, 0.2, 1.0, 1.0, L, 2)
    t = O.triple_products(L, 2, 2)
    s = O.SgSolver(nx, nx, 2, 1, c, t, alpha0=0.1, alpha1=0.01, dt=0.05, threads=2)
    bigM, bigK = R.sg_blocks(nx, nx, c, t.dense())
    x = rand(s.n_terms * s.n_dofs, 5)
    y = s.apply_block(x, "stiffness")
    exp = bigK @ x
    assert np.abs(y - exp).max() <= 1e-12 * (1 + np.abs(exp).max())
    assert np.abs(s.apply_block(x, "mass") - bigM @ x).max() <= 1e-15


def test_transient_operator_symmetric():
    # test_sg.cpp:75-83
    nx = 6
    c = O.lognormal_coeff(nx, nx, 0.15, 1.0, 1.0, 2, 1)
    s = O.SgSolver(nx, nx, 2, 1, c, O.triple_products(2, 1, 2), alpha0=0.2, alpha1=0.01, dt=0.05, threads=2)
    x, y = rand(s.n_terms * s.n_dofs, 11), rand(s.n_terms * s.n_dofs, 12)
    lhs, rhs = y @ s.apply_block(x), x @ s.apply_block(y)
    assert abs(lhs - rhs) <= 1e-10 * abs(rhs)


def dense_schur(nx, px, py, c, t, alpha0, alpha1, dt, s):
    bigM, bigK = R.sg_blocks(nx, nx, c, t.dense())
    mf, df = 1 / (0.25 * dt * dt), 0.5 / (0.25 * dt)
    kt = mf * bigM + df * (alpha0 * bigM + alpha1 * bigK) + bigK
    n, nt = s.n_dofs, s.n_terms
    interior, iface = R.interface_split(nx, nx, px, py)
    I = np.concatenate([j * n + interior for j in range(nt)])
    G = np.concatenate([j * n + iface for j in range(nt)])
    return kt[np.ix_(G, G)] - kt[np.ix_(I, G)].T @ np.linalg.solve(kt[np.ix_(I, I)], kt[np.ix_(I, G)])


@pytest.mark.parametrize("px,py", [(2, 1), (2, 2)])
def test_stochastic_schur_matches_dense_block_elimination(px, py):
    # test_sg.cpp:107-156 (8x8 mesh, L=1, p 1/1; <= 1e-10) and test_dd.cpp:77-96
    nx = 8
    c = O.lognormal_coeff(nx, nx, 0.25, 1.0, 1.0, 1, 1)
    t = O.triple_products(1, 1, 1)
    s = O.SgSolver(nx, nx, px, py, c, t, alpha0=0.3, alpha1=0.02, dt=0.04, threads=2)
    S = dense_schur(nx, px, py, c, t, 0.3, 0.02, 0.04, s)
    x = rand(s.n_global, 21)
    sx = s.schur_matvec(x)
    assert np.abs(sx - S @ x).max() <= 1e-10 * (1 + np.abs(S).max())
    assert x @ sx > 0
    r1, r2 = rand(s.n_global, 31), rand(s.n_global, 32)
    a, b = r2 @ s.apply_nn2(r1), r1 @ s.apply_nn2(r2)
    assert abs(a - b) <= 1e-10 * abs(b)
    for sub in range(px * py):
        Sl, _ = s.local_schur(sub)
        assert np.abs(Sl - Sl.T).max() <= 1e-12 * (1 + np.abs(Sl).max())


def test_two_level_without_corners_is_exact_inverse():
    # test_dd.cpp:123-151: one block, no corners -> NN2 = S^{-1}, PCG in 1 iteration
    rng = np.random.default_rng(0)
    n = 7
    a = rng.uniform(-1, 1, (n, n))
    a = a @ a.T + n * np.eye(n)
    r = rand(n, 3)
    z, it = O.single_block_nn2(a, r)
    assert np.abs(a @ z - r).max() <= 1e-10
    assert it == 1


def test_coarse_operator_symmetric_single_cross_point():
    # test_dd.cpp:153-170: 8x8, 2x2 -> one interior cross point (times P+1 terms)
    nx = 8
    c = O.lognormal_coeff(nx, nx, 0.2, 1.0, 1.0, 2, 1)
    s = O.SgSolver(nx, nx, 2, 2, c, O.triple_products(2, 1, 1), alpha0=0.1, alpha1=0.0, dt=0.05, threads=2)
    assert s.n_corner == 1
    F = s.coarse_operator()
    assert F.shape == (s.n_terms, s.n_terms)
    assert np.abs(F - F.T).max() <= 1e-12 * (1 + np.abs(F).max())
    assert np.all(np.linalg.eigvalsh(F) > 0)


# -------------------------------------------------------- trajectories -----
def test_matrix_free_trajectory_matches_dense_newmark():
    # test_sg.cpp:218-272 (<= 1e-8); acceptance criterion 8 recorded 1.57e-15
    nx, dt, steps = 8, 0.04, 10
    c = O.lognormal_coeff(nx, nx, 0.25, 1.0, 1.0, 1, 1)
    t = O.triple_products(1, 1, 1)
    s = O.SgSolver(nx, nx, 2, 1, c, t, dt=dt, tol=1e-12, threads=2)
    u0 = O.gaussian_pulse(nx, nx)
    out = s.run(u0, np.zeros_like(u0), steps, store_full=True)
    bigM, bigK = R.sg_blocks(nx, nx, c, t.dense())
    _, _, _, n2d, free = R.mesh(nx, nx)
    U0 = np.zeros(s.n_terms * s.n_dofs)
    U0[: s.n_dofs] = u0[free]
    ref = R.newmark_dense(bigM, bigK, 0.5445, 0.0174, dt, U0, steps)
    assert max(np.abs(a - b).max() for a, b in zip(out["full"], ref)) <= 1e-8


def test_sigma_zero_reproduces_deterministic_trajectory():
    # test_sg.cpp:180-216 / acceptance criterion 7 (<= 1e-10; recorded 2.05e-15)
    nx, dt, steps = 10, 0.03, 10
    c = O.lognormal_coeff(nx, nx, 0.0, 1.0, 1.0, 3, 2, g0=0.1)
    sg = O.SgSolver(nx, nx, 2, 2, c, O.triple_products(3, 2, 3), dt=dt, tol=1e-12, threads=2)
    det = O.SgSolver(nx, nx, 2, 2, c[:1], O.triple_products(1, 0, 0), dt=dt, tol=1e-12, threads=2)
    u0 = O.gaussian_pulse(nx, nx)
    a = sg.run(u0, 0 * u0, steps, store_full=True)["full"]
    b = det.run(u0, 0 * u0, steps, store_full=True)["full"]
    n = sg.n_dofs
    assert np.abs(a[:, :n] - b).max() <= 1e-10
    assert np.abs(a[:, n:]).max() <= 1e-10


def test_dd_trajectory_matches_direct_solve():
    # test_dd.cpp:248-270 with the NN2 preconditioner (<= 1e-8)
    nx, dt, steps = 16, 0.02, 12
    one = np.ones((1, (nx + 1) ** 2))
    t = O.triple_products(1, 0, 0)
    direct = O.SgSolver(nx, nx, 1, 1, one, t, dt=dt, tol=1e-10, threads=2)
    dd = O.SgSolver(nx, nx, 2, 2, one, t, dt=dt, tol=1e-12, threads=2)
    assert direct.uses_direct and not dd.uses_direct
    u0 = O.gaussian_pulse(nx, nx)
    a = direct.run(u0, 0 * u0, steps, store_full=True)["full"]
    b = dd.run(u0, 0 * u0, steps, store_full=True)["full"]
    assert np.abs(a - b).max() <= 1e-8


def test_zero_data_stays_zero():
    # test_dd.cpp:272-279
    nx = 8
    c = O.lognormal_coeff(nx, nx, 0.2, 1.0, 1.0, 2, 1)
    s = O.SgSolver(nx, nx, 2, 2, c, O.triple_products(2, 1, 2), dt=0.05, threads=2)
    z = np.zeros((nx + 1) ** 2)
    out = s.run(z, z, 5, store_full=True)
    assert np.abs(out["full"]).max() == 0.0 and np.all(out["iterations"] == 0)


def test_thread_count_bitwise_reproducible_and_monotone_residuals():
    # test_dd.cpp:281-308
    nx = 16
    c = O.lognormal_coeff(nx, nx, 0.2, 1.0, 1.0, 2, 1)
    t = O.triple_products(2, 1, 2)
    u0 = O.gaussian_pulse(nx, nx)
    hist = []
    for th in (1, 4):
        s = O.SgSolver(nx, nx, 4, 2, c, t, dt=0.01, tol=1e-10, threads=th)
        s.run(u0, 0 * u0, 8)
        hist.append([s.residual_history(k) for k in range(8)])
    for ra, rb in zip(*hist):
        assert np.array_equal(ra, rb)
        assert np.all(ra[1:] <= ra[:-1] * (1 + 1e-9))


# ------------------------------------------------- recorded known answers ---
def test_recorded_sg_nn2_iteration_flatness():
    # acceptance.cpp:492-529, recorded proj/test_output.txt:52:
    # "mean iters L={3,4,5}: 3.00/3.00/3.00, p_out={2,3,4}: 3.00/3.00/3.00"
    nx = 24
    got = []
    for L, pin, pout in [(3, 2, 3), (4, 2, 3), (5, 2, 3), (3, 2, 2), (3, 2, 4)]:
        c = O.lognormal_coeff(nx, nx, 0.1, 1.0, 1.0, L, pin)
        dt = O.cfl_dt(nx, c[0].max(), 0.1)
        s = O.SgSolver(nx, nx, 4, 4, c, O.triple_products(L, pin, pout), dt=dt, tol=1e-8)
        u0 = O.gaussian_pulse(nx, nx)
        got.append(s.run(u0, 0 * u0, math.ceil(0.3 / dt))["mean_iterations"])
    assert [f"{g:.2f}" for g in got] == ["3.00"] * 5


def test_recorded_deterministic_nn2_iterations():
    # acceptance.cpp:156-177 (run_precond_comparison(40, 0.01, 0.5, ...)), recorded
    # proj/test_output.txt:44: "nn2: 3.0/3.0/3.0" for 4/8/16 subdomains.  The
    # deterministic solver equals the SG solver with one PCE term (test_sg.cpp:158-178).
    nx = 40
    one = np.ones((1, (nx + 1) ** 2))
    t = O.triple_products(1, 0, 0)
    got = []
    for px, py in [(2, 2), (4, 2), (4, 4)]:
        s = O.SgSolver(nx, nx, px, py, one, t, dt=0.01, tol=1e-8)
        u0 = O.gaussian_pulse(nx, nx)
        got.append(s.run(u0, 0 * u0, math.ceil(0.5 / 0.01 - 1e-12))["mean_iterations"])
    assert [f"{g:.1f}" for g in got] == ["3.0"] * 3


# ------------------------------------- lumped / NN1 / NN2 ---
def _det(nx, px, py, dt, precond, tol=1e-10, alpha0=0.5445, alpha1=0.0174):
    """DetSolver(mesh, part, ones, 1, alpha0, alpha1, params, opt) of test_dd.cpp:54-66:
    the SG solver with one PCE term (test_sg.cpp:158-178) and the chosen preconditioner."""
    one = np.ones((1, (nx + 1) ** 2))
    return O.SgSolver(nx, nx, px, py, one, O.triple_products(1, 0, 0), dt=dt, tol=tol, threads=2,
                      alpha0=alpha0, alpha1=alpha1, precond=precond)


@pytest.mark.parametrize("kind", ["lumped", "nn1", "nn2"])
def test_preconditioners_are_symmetric(kind):
    # test_dd.cpp:109-121 (epsilon 1e-10)
    s = _det(8, 2, 2, 0.05, kind, alpha0=0.2, alpha1=0.01)
    r1, r2 = rand(s.n_global, 1), rand(s.n_global, 2)
    a, b = r2 @ s.apply_precond(kind, r1), r1 @ s.apply_precond(kind, r2)
    assert abs(a - b) <= 1e-10 * max(abs(a), abs(b))


@pytest.mark.parametrize("kind", ["lumped", "nn1", "nn2"])
def test_dd_trajectory_matches_direct_for_every_preconditioner(kind):
    # test_dd.cpp:248-270 (<= 1e-8); recorded proj/test_output.txt:43 (criterion 4):
    # "nn2: 8.76e-14  nn1: 4.49e-13  lumped: 1.91e-15"
    nx, dt, steps = 16, 0.02, 12
    direct = _det(nx, 1, 1, dt, "nn2")
    dd = _det(nx, 2, 2, dt, kind, tol=1e-12)
    assert direct.uses_direct and not dd.uses_direct
    u0 = O.gaussian_pulse(nx, nx)
    a = direct.run(u0, 0 * u0, steps, store_full=True)["full"]
    b = dd.run(u0, 0 * u0, steps, store_full=True)["full"]
    assert np.abs(a - b).max() <= 1e-8


def test_recorded_preconditioner_comparison():
    # acceptance.cpp:156-177 (run_precond_comparison(40, 0.01, 0.5, {2x2, 4x2, 4x4}, 2, 1e-8, 500),
    # experiments.cpp:82-111), recorded proj/test_output.txt:44:
    # "lumped: 11.2/11.5/12.0 nn1: 3.7/3.9/4.0 nn2: 3.0/3.0/3.0"
    nx, dt = 40, 0.01
    steps = math.ceil(0.5 / dt - 1e-12)
    u0 = O.gaussian_pulse(nx, nx)
    got = {}
    for kind in ("lumped", "nn1", "nn2"):
        got[kind] = [f"{_det(nx, px, py, dt, kind, tol=1e-8).run(u0, 0 * u0, steps)['mean_iterations']:.1f}"
                     for px, py in [(2, 2), (4, 2), (4, 4)]]
    assert got == {"lumped": ["11.2", "11.5", "12.0"], "nn1": ["3.7", "3.9", "4.0"], "nn2": ["3.0", "3.0", "3.0"]}
