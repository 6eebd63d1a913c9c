"""GPU parity at the sizes where numbers are claimed (BASELINE configs[1],
[2] and [4]; SURVEY 8c parity contract: PCG iterations within +-1 per step and
the PCE solution within 1e-8 relative L2 at CG tolerance 1e-10).

* C2 (configs[1]): the whole 100-step benchmark configuration against the
  oracle run in the same process (oracle setup ~1 min + ~0.5 s per step on the
  box's host cores, ~1 GB of full-state history per side).
* C3 (configs[2]) and C5 L=8 (configs[4]): the oracle's whole solver needs
  more than the host has at C5 L=8 and ~20 min of setup at C3, so each
  subdomain class (interior, edge, corner) is checked on its own: the oracle
  builds that one subdomain's S_s, S_rr^-1 and Psi_s (SgSolver::local_blocks,
  src/sg.cpp:186-246, src/dd.cpp:112-120) and the GPU exports the same
  operators from its tiles (sgw_local_block).  The full-size trajectory is then
  cross-checked between three independent GPU constructions: the explicit
  Schur tiles, the reduced-memory implicit Schur (S_s never formed) and the
  sharded two-rank decomposition.  The full C3 oracle trajectory runs with
  SGW_FULL_ORACLE=1 (tests/test_gpu_fullsize.py::test_c3_full_oracle_trajectory).
"""
import gc
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_2512_23027_b200")
bench = pytest.importorskip("bench")


def relerr(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def cfg_inputs(name):
    c = bench.CONFIGS[name]
    nx = c["nx"]
    coeff = O.lognormal_coeff(nx, nx, c["sigma"], c["b"], c["b"], c["L"], c["p_in"])
    t = O.triple_products(c["L"], c["p_in"], c["p_out"])
    return c, nx, coeff, t


def gpu_solver(name, coeff, t, **opt):
    c = bench.CONFIGS[name]
    return sg.SgSolver(c["nx"], c["nx"], c["px"], c["px"], coeff, t, alpha0=bench.ALPHA0, alpha1=bench.ALPHA1,
                       params=sg.NewmarkParams(dt=c["dt"]), options=sg.SgOptions(tol=bench.TOL, **opt))


def ricker_run(solver, nx, steps):
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    return solver.run(z, z, steps, sg.ForceSpec(node=node, f0=bench.F0, t0=bench.T0))


def subdomain_classes(px):
    """one interior, one edge and one corner subdomain (row-major ids)"""
    return [px + 1, 1, 0] if px > 2 else [0, 1]


def check_local_blocks(g, name, coeff, t, subs):
    c = bench.CONFIGS[name]
    nx = c["nx"]
    rng = np.random.default_rng(5)
    for s in subs:
        lb = O.LocalBlocks(nx, nx, c["px"], c["px"], coeff, t, s, alpha0=bench.ALPHA0, alpha1=bench.ALPHA1,
                           dt=c["dt"])
        S_o, gm_o = lb.schur()
        S_g, gm_g = g.schur().local_block(s, "S")
        assert np.array_equal(gm_o, gm_g), f"subdomain {s}: flat maps differ"
        assert relerr(S_g, S_o) <= 1e-10, f"subdomain {s}: S_s"
        del S_o, S_g
        Q_g, _ = g.schur().local_block(s, "Q")
        V = rng.uniform(-1.0, 1.0, (lb.r, 4))
        assert relerr(Q_g @ V, lb.srr_solve(V)) <= 1e-9, f"subdomain {s}: S_rr^-1"
        del Q_g
        if lb.c:
            P_g, _ = g.schur().local_block(s, "Psi")
            assert relerr(P_g, lb.psi()) <= 1e-9, f"subdomain {s}: Psi_s"
        del lb
        gc.collect()


@pytest.mark.timeout(2400)
def test_c2_full_benchmark_trajectory_against_oracle(gpu):
    # BASELINE configs[1] as benchmarked: 256x256, 8x8, P+1 = 20, 100 steps
    c, nx, coeff, t = cfg_inputs("C2")
    steps = 100
    g = gpu_solver("C2", coeff, t, store_full=True)
    hg = ricker_run(g, nx, steps)
    g.close()
    del g
    gc.collect()
    cpu = O.SgSolver(nx, nx, c["px"], c["px"], coeff, t, alpha0=bench.ALPHA0, alpha1=bench.ALPHA1, dt=c["dt"],
                     tol=bench.TOL)
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hc = cpu.run(z, z, steps, force_node=node, f0=bench.F0, t0=bench.T0, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    full_g, full_c = hg.full_state, hc["full"]
    assert np.linalg.norm(full_g - full_c) / np.linalg.norm(full_c) <= 1e-8
    per_step = np.linalg.norm(full_g - full_c, axis=1) / np.maximum(np.linalg.norm(full_c, axis=1), 1e-300)
    assert per_step[1:].max() <= 1e-8
    print(f"C2 100 steps: iterations GPU {int(hg.iterations.sum())} oracle {int(hc['iterations'].sum())}, "
          f"max per-step rel L2 {per_step[1:].max():.2e}")


class _Traj:
    pass


@pytest.fixture(scope="module")
def c3_explicit(gpu):
    """C3 with the explicit Schur tiles: per-subdomain blocks against the
    oracle, plus a 5-step trajectory kept for the cross-checks below."""
    c, nx, coeff, t = cfg_inputs("C3")
    g = gpu_solver("C3", coeff, t, store_full=True)
    check_local_blocks(g, "C3", coeff, t, subdomain_classes(c["px"]))
    tr = _Traj()
    h = ricker_run(g, nx, 5)
    tr.iterations, tr.full = h.iterations.copy(), h.full_state.copy()
    x = np.random.default_rng(3).uniform(-1, 1, g.n_global)
    tr.x, tr.Sx, tr.Nx = x, g.schur().matvec(x), g.schur().apply_nn2(x)
    g.close()
    del g, h
    gc.collect()
    return tr


@pytest.mark.timeout(2400)
def test_c3_subdomain_blocks_and_reduced_memory_trajectory(c3_explicit):
    # reduced-memory mode never forms S_s: same Schur products and trajectory
    c, nx, coeff, t = cfg_inputs("C3")
    g = gpu_solver("C3", coeff, t, store_full=True, implicit_schur=True)
    assert relerr(g.schur().matvec(c3_explicit.x), c3_explicit.Sx) <= 1e-10
    assert relerr(g.schur().apply_nn2(c3_explicit.x), c3_explicit.Nx) <= 1e-12
    h = ricker_run(g, nx, 5)
    assert np.all(np.abs(h.iterations - c3_explicit.iterations) <= 1)
    assert np.linalg.norm(h.full_state - c3_explicit.full) / np.linalg.norm(c3_explicit.full) <= 1e-10
    g.close()


@pytest.mark.timeout(2400)
def test_c3_two_rank_decomposition_trajectory(c3_explicit):
    # the sharded code path (two ranks on one device) at full size
    c, nx, coeff, t = cfg_inputs("C3")
    grp = sg.LocalGroup(2)
    kw = dict(alpha0=bench.ALPHA0, alpha1=bench.ALPHA1, params=sg.NewmarkParams(dt=c["dt"]),
              options=sg.SgOptions(tol=bench.TOL, store_full=True))
    ranks = grp.solvers(nx, nx, c["px"], c["px"], coeff, t, **kw)
    for y in grp.map(lambda r: ranks[r].schur().matvec(c3_explicit.x)):
        assert relerr(y, c3_explicit.Sx) <= 1e-12
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    force = sg.ForceSpec(node=node, f0=bench.F0, t0=bench.T0)
    for h in grp.map(lambda r: ranks[r].run(z, z, 5, force)):
        assert np.all(np.abs(h.iterations - c3_explicit.iterations) <= 1)
        assert np.linalg.norm(h.full_state - c3_explicit.full) / np.linalg.norm(c3_explicit.full) <= 1e-10
    for r in ranks:
        r.close()
    grp.close()


@pytest.mark.timeout(2400)
def test_c5_l8_subdomain_blocks_against_oracle(gpu):
    # BASELINE configs[4] at L = 8 (P+1 = 45, 495 input terms, p_in = 4)
    c, nx, coeff, t = cfg_inputs("C5L8")
    g = gpu_solver("C5L8", coeff, t)
    assert g.n_terms == 45
    check_local_blocks(g, "C5L8", coeff, t, subdomain_classes(c["px"]))
    h = ricker_run(g, nx, 2)
    assert np.all(h.iterations >= 1) and np.all(h.iterations <= 6)
    g.close()


@pytest.mark.timeout(7200)
@pytest.mark.skipif(os.environ.get("SGW_FULL_ORACLE") != "1", reason="full C3 oracle: ~130 GB host RAM, ~20 min")
def test_c3_full_oracle_trajectory(c3_explicit):
    c, nx, coeff, t = cfg_inputs("C3")
    cpu = O.SgSolver(nx, nx, c["px"], c["px"], coeff, t, alpha0=bench.ALPHA0, alpha1=bench.ALPHA1, dt=c["dt"],
                     tol=bench.TOL)
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hc = cpu.run(z, z, 5, force_node=node, f0=bench.F0, t0=bench.T0, store_full=True)
    assert np.all(np.abs(c3_explicit.iterations - hc["iterations"]) <= 1)
    rel = np.linalg.norm(c3_explicit.full - hc["full"]) / np.linalg.norm(hc["full"])
    print(f"C3 5 steps vs oracle: rel L2 {rel:.2e}, setup {hc['t_setup']:.0f} s")
    assert rel <= 1e-8


# ---------------------------------------------------------- large bases ----
# The P+1 caps of round 1: interior blocks B = W (P+1) >
# 1536 (the large-block sweep), P+1 beyond the JIT operator's register budget
# (table-driven operator) and local vectors beyond one CTA's shared memory
# (host-driven PCG).  configs[4]'s L = 12 basis (P+1 = 91, n_in = 1820).
def large_pair(nx, px, L, pin, pout, implicit=False, oracle=True):
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, L, pin)
    t = O.triple_products(L, pin, pout)
    g = sg.SgSolver(nx, nx, px, px, coeff, t, alpha0=bench.ALPHA0, alpha1=bench.ALPHA1,
                    params=sg.NewmarkParams(dt=1e-3),
                    options=sg.SgOptions(tol=1e-10, store_full=True, implicit_schur=implicit))
    c = O.SgSolver(nx, nx, px, px, coeff, t, alpha0=bench.ALPHA0, alpha1=bench.ALPHA1, dt=1e-3, tol=1e-10,
                   threads=os.cpu_count() or 4) if oracle else None
    return g, c


@pytest.mark.timeout(1500)
def test_large_basis_p91_trajectory_against_oracle(gpu):
    # nx = 40 on 2 x 2 (m = 20, B = 19 x 91 = 1729 > 1536): the large-block
    # sweep, the table-driven SG operator (n_in = 1820), the oracle's setup
    # takes ~3 min on 8 host cores
    nx = 40
    g, c = large_pair(nx, 2, 12, 4, 2)
    assert g.n_terms == 91
    x = np.random.default_rng(3).uniform(-1, 1, g.n_terms * g.n_dofs)
    assert relerr(g.apply_block_transient(x), c.apply_block(x, "transient")) <= 1e-12
    xi = np.random.default_rng(4).uniform(-1, 1, g.n_global)
    assert relerr(g.schur().matvec(xi), c.schur_matvec(xi)) <= 1e-10
    assert relerr(g.schur().apply_nn2(xi), c.apply_nn2(xi)) <= 1e-10
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(z, z, 3, sg.ForceSpec(node=node, f0=bench.F0, t0=bench.T0))
    hc = c.run(z, z, 3, force_node=node, f0=bench.F0, t0=bench.T0, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    rel = np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"])
    assert rel <= 1e-8, rel


@pytest.mark.timeout(1500)
def test_large_basis_p91_m32_explicit_vs_reduced_memory(gpu):
    # the VERDICT r1 case: nx = 64 on 2 x 2 (m = 32, B = 31 x 91 = 2821), GPU
    # only (the oracle's setup alone would take ~20 min here): the explicit
    # Schur tiles and the reduced-memory implicit Schur, two independent
    # constructions, agree step by step; the PCG's true residual meets the
    # tolerance (sgw_pcg report)
    nx = 64
    runs = []
    for implicit in (False, True):
        g, _ = large_pair(nx, 2, 12, 4, 2, implicit=implicit, oracle=False)
        node = O.nearest_node(nx, nx, 0.5, 0.5)
        z = np.zeros((nx + 1) ** 2)
        runs.append(g.run(z, z, 2, sg.ForceSpec(node=node, f0=bench.F0, t0=bench.T0)))
        if not implicit:
            b = np.random.default_rng(5).uniform(-1, 1, g.n_global)
            x, rep = g.pcg(b)
            assert rep["converged"] and rep["residual_history"][-1] <= 1e-10
        del g
        gc.collect()
    a, b = runs
    assert np.all(np.abs(a.iterations - b.iterations) <= 1)
    assert np.linalg.norm(a.full_state - b.full_state) / np.linalg.norm(b.full_state) <= 1e-8


@pytest.mark.timeout(1500)
def test_c5_l16_shaped_subdomains_reduced_memory(gpu):
    # configs[4]'s L = 16 basis (P+1 = 153, n_in = 4845) on 32 x 32 subdomains
    # (B = 31 x 153 = 4743) in reduced-memory mode: constructs, and a step's
    # interface solve converges (true residual <= tol)
    nx = 64
    g, _ = large_pair(nx, 2, 16, 4, 2, implicit=True, oracle=False)
    assert g.n_terms == 153
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    h = g.run(z, z, 1, sg.ForceSpec(node=node, f0=bench.F0, t0=bench.T0))
    assert h.iterations[0] >= 1 and np.isfinite(h.full_state).all()
