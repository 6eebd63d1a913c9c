"""GPU parity of the lumped / NN1 preconditioners and the deterministic
solver (det_loop.cpp, dd.cpp:159-197) against the CPU
oracle, and the reference's recorded preconditioner comparison."""
import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_2512_23027_b200")

KINDS = ["lumped", "nn1", "nn2"]


def rand(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def relerr(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def det_pair(nx, px, py, dt, kind, tol=1e-10, alpha0=0.5445, alpha1=0.0174):
    """DetSolver(mesh, part, ones, 1, alpha0, alpha1, params, opt) (test_dd.cpp:54-66) on both sides."""
    one = np.ones((nx + 1) ** 2)
    gpu = sg.DetSolver(nx, nx, px, py, one, 1.0, alpha0, alpha1, sg.NewmarkParams(dt=dt),
                       sg.SolveOptions(precond=kind, tol=tol, store_full=True))
    cpu = O.SgSolver(nx, nx, px, py, one[None, :], O.triple_products(1, 0, 0), dt=dt, tol=tol, threads=2,
                     alpha0=alpha0, alpha1=alpha1, precond=kind)
    return gpu, cpu


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("cfg", [(8, 2, 2), (16, 4, 2), (14, 4, 3)])
def test_preconditioner_matches_oracle_and_is_symmetric(gpu, kind, cfg):
    # dd.cpp:159-253 vs the oracle (1e-10); symmetry as test_dd.cpp:109-121 (1e-10)
    nx, px, py = cfg
    g, c = det_pair(nx, px, py, 0.05, kind, alpha0=0.2, alpha1=0.01)
    r1, r2 = rand(c.n_global, 1), rand(c.n_global, 2)
    z1 = g.schur().apply_precond(kind, r1)
    assert relerr(z1, c.apply_precond(kind, r1)) <= 1e-10
    a, b = r2 @ z1, r1 @ g.schur().apply_precond(kind, r2)
    assert abs(a - b) <= 1e-10 * max(abs(a), abs(b))


def test_unbuilt_preconditioner_rejected(gpu):
    g, c = det_pair(8, 2, 2, 0.05, "nn2")
    with pytest.raises(sg.SgInvalidArgument):
        g.schur().apply_precond("nn1", rand(c.n_global, 1))
    with pytest.raises(sg.SgInvalidArgument):
        sg.precond_from_string("jacobi")  # test_cli_io.cpp:65


@pytest.mark.parametrize("kind", KINDS)
def test_dd_trajectory_matches_direct_for_every_preconditioner(gpu, kind):
    # test_dd.cpp:248-270: the 2x2 DD run against the single-domain direct
    # solve (the oracle's direct path) within 1e-8
    nx, dt, steps = 16, 0.02, 12
    g, _ = det_pair(nx, 2, 2, dt, kind, tol=1e-12)
    direct = O.SgSolver(nx, nx, 1, 1, np.ones((1, (nx + 1) ** 2)), O.triple_products(1, 0, 0), dt=dt, tol=1e-10)
    assert direct.uses_direct
    u0 = sg.gaussian_pulse(nx, nx)
    a = g.run(u0, 0 * u0, steps).full_u
    b = direct.run(u0, 0 * u0, steps, store_full=True)["full"]
    assert np.abs(a - b).max() <= 1e-8


@pytest.mark.parametrize("kind", ["lumped", "nn1"])
def test_iterations_match_oracle(gpu, kind):
    nx, dt, steps = 24, 0.01, 10
    g, c = det_pair(nx, 4, 2, dt, kind, tol=1e-10)
    u0 = sg.gaussian_pulse(nx, nx)
    hg = g.run(u0, 0 * u0, steps)
    hc = c.run(u0, 0 * u0, steps, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_u - hc["full"]) <= 1e-8 * np.linalg.norm(hc["full"])


def test_recorded_preconditioner_comparison_on_gpu(gpu):
    # acceptance.cpp:156-177 via run_precond_comparison (experiments.cpp:82-111);
    # recorded proj/test_output.txt:44:
    # "lumped: 11.2/11.5/12.0 nn1: 3.7/3.9/4.0 nn2: 3.0/3.0/3.0, nn2 growth 0%"
    cmp = sg.run_precond_comparison(40, 0.01, 0.5, [(2, 2), (4, 2), (4, 4)], tol=1e-8)
    got = {k: [f"{v:.1f}" for v in cmp[k]] for k in KINDS}
    assert got == {"lumped": ["11.2", "11.5", "12.0"], "nn1": ["3.7", "3.9", "4.0"], "nn2": ["3.0", "3.0", "3.0"]}


def test_stochastic_solver_with_nn1_matches_oracle(gpu):
    # the SG system with the one-level preconditioner (an extension of the
    # reference, whose SG path hard-wires NN2): same iterations and trajectory
    nx, L, pin, pout, dt = 16, 2, 2, 2, 2e-3
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, L, pin)
    t = O.triple_products(L, pin, pout)
    g = sg.SgSolver(nx, nx, 4, 2, coeff, t, params=sg.NewmarkParams(dt=dt),
                    options=sg.SgOptions(precond="nn1", tol=1e-10, store_full=True))
    c = O.SgSolver(nx, nx, 4, 2, coeff, t, dt=dt, tol=1e-10, precond="nn1")
    x = rand(c.n_global, 3)
    assert relerr(g.schur().apply_nn1(x), c.apply_nn1(x)) <= 1e-10
    node = sg.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(z, z, 6, sg.ForceSpec(node=node))
    hc = c.run(z, z, 6, force_node=node, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) <= 1e-8 * np.linalg.norm(hc["full"])


def test_subdomain_without_interior_dofs_keeps_schur_equal_to_k_gg(gpu):
    # test_dd.cpp:98-107: one cell per subdomain, the only free node is the
    # shared centre, so S = K~_GG (the oracle's dense restatement)
    g, c = det_pair(2, 2, 2, 0.1, "nn2", alpha0=0.0, alpha1=0.0)
    assert c.n_global == 1
    one = np.ones(1)
    assert relerr(g.schur().matvec(one), c.schur_matvec(one)) <= 1e-12


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("cfg", [(4, 4, 4), (6, 6, 2), (5, 4, 3)])
def test_one_cell_subdomains_match_oracle(gpu, kind, cfg):
    # blocks one cell wide (all of them, one direction only, or mixed with
    # two-cell blocks by the floor-division split): Schur, preconditioner and
    # a short trajectory against the oracle
    nx, px, py = cfg
    g, c = det_pair(nx, px, py, 0.05, kind, alpha0=0.2, alpha1=0.01)
    r = rand(c.n_global, 3)
    assert relerr(g.schur().matvec(r), c.schur_matvec(r)) <= 1e-11
    assert relerr(g.schur().apply_precond(kind, r), c.apply_precond(kind, r)) <= 1e-10
    u0 = O.gaussian_pulse(nx, nx)
    hg = g.run(u0, 0 * u0, 3)
    hc = c.run(u0, 0 * u0, 3, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_u - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-9
