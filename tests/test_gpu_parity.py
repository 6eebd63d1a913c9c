"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle on
identical seeded inputs.  Tolerances follow the reference tests and the
BASELINE parity contract (PCG iterations within +-1 per step, PCE solution
within 1e-8 relative L2 at CG tolerance 1e-10)."""
import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

sg = pytest.importorskip("paper_2512_23027_b200")


def rand(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def pair(nx, px, py, sigma, b, L, pin, pout, dt, tol=1e-10, alpha0=0.5445, alpha1=0.0174, g0=0.0):
    coeff = O.lognormal_coeff(nx, nx, sigma, b, b, L, pin, g0=g0)
    t = O.triple_products(L, pin, pout)
    gpu = sg.SgSolver(nx, nx, px, py, coeff, t, alpha0=alpha0, alpha1=alpha1, params=sg.NewmarkParams(dt=dt),
                      options=sg.SgOptions(tol=tol, store_full=True))
    cpu = O.SgSolver(nx, nx, px, py, coeff, t, alpha0=alpha0, alpha1=alpha1, dt=dt, tol=tol)
    return gpu, cpu


def relerr(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("op", ["mass", "stiffness", "transient"])
@pytest.mark.parametrize("cfg", [(12, 2, 4, 2), (40, 3, 2, 3), (70, 3, 3, 3), (20, 4, 2, 3), (34, 4, 6, 3),
                                 (14, 6, 4, 2), (11, 8, 4, 2), (3, 2, 4, 2), (4, 3, 6, 3), (5, 5, 4, 2)])
def test_apply_block_matches_oracle(gpu, op, cfg):
    # sg.cpp:425-447 vs the oracle; test_sg.cpp:51-73 tolerance 1e-12.  The
    # JIT-specialised operator (sgop.cu) with 1, 2 and 4 thread groups per node
    # (P+1 = 6, 20 / 21, 28 / 35, 45), grids that are not multiples of the
    # 32-column strip (W = 33 leaves a 1-column strip), and the 1x1 / 2x2 dof
    # grids where every boundary-coupling slot is used.
    nx, L, pin, pout = cfg
    g, c = pair(nx, 2, 2, 0.3, 0.5, L, pin, pout, 1e-3)
    x = rand(g.n_terms * g.n_dofs, 1)
    a = getattr(g, f"apply_block_{op}")(x)
    b = c.apply_block(x, op)
    assert relerr(a, b) <= 1e-12


@pytest.mark.parametrize("case", [(20, 2, 2, 3, 4, 2), (17, 3, 2, 2, 4, 2)])
def test_large_block_sweep_matches_oracle(gpu, monkeypatch, case):
    # the large-block interior sweep (sweep.cu sweep_generic_kernel, used when
    # B = W (P+1) > 1536), forced here on small blocks: Schur products (which
    # stand on the setup only) and the trajectory (two sweeps per step)
    monkeypatch.setenv("SGW_SWEEP_GENERIC", "1")
    nx, px, py, L, pin, pout = case
    g, c = pair(nx, px, py, 0.3, 0.5, L, pin, pout, 1e-3)
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(z, z, 6, sg.ForceSpec(node=node))
    hc = c.run(z, z, 6, force_node=node, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10


@pytest.mark.parametrize("cfg", [(8, 2, 1, 1, 1, 1), (12, 2, 2, 2, 2, 2), (16, 4, 4, 2, 4, 2), (24, 3, 2, 3, 2, 3),
                                 (22, 4, 3, 2, 2, 2), (13, 5, 2, 1, 2, 2)])
def test_schur_and_nn2_match_oracle(gpu, cfg):
    nx, px, py, L, pin, pout = cfg
    g, c = pair(nx, px, py, 0.3, 0.5, L, pin, pout, 1e-3)
    assert (g.n_global, g.n_terms) == (c.n_global, c.n_terms)
    x = rand(g.n_global, 7)
    assert relerr(g.schur().matvec(x), c.schur_matvec(x)) <= 1e-10
    assert relerr(g.schur().apply_nn2(x), c.apply_nn2(x)) <= 1e-10
    if c.n_corner:
        F = g.schur().coarse_operator()
        assert relerr(F, c.coarse_operator()) <= 1e-10


def test_nn2_symmetric_and_schur_spd(gpu):
    g, _ = pair(16, 4, 4, 0.3, 0.5, 2, 4, 2, 1e-3)
    r1, r2 = rand(g.n_global, 31), rand(g.n_global, 32)
    a, b = r2 @ g.schur().apply_nn2(r1), r1 @ g.schur().apply_nn2(r2)
    assert abs(a - b) <= 1e-10 * abs(b)
    assert r1 @ g.schur().matvec(r1) > 0


@pytest.mark.parametrize("cfg", [(16, 4, 4, 2, 4, 2), (24, 3, 2, 3, 2, 3), (26, 4, 3, 2, 3, 2)])
def test_pcg_matches_oracle_iterations(gpu, cfg):
    # pcg(matvec, apply_nn2) (src/pcg.cpp:7-50) on the same right-hand side:
    # iteration count within +-1, residual history and solution against the
    # oracle's own pcg
    nx, px, py, L, pin, pout = cfg
    g, c = pair(nx, px, py, 0.3, 0.5, L, pin, pout, 1e-3)
    b = c.schur_matvec(rand(g.n_global, 3))
    x, rep = g.pcg(b)
    xc, repc = c.pcg(b)
    assert rep["converged"] and repc["converged"]
    assert abs(rep["iterations"] - repc["iterations"]) <= 1
    if rep["iterations"] == repc["iterations"]:
        h, hc = np.asarray(rep["residual_history"]), repc["residual_history"]
        assert len(h) == len(hc) and np.allclose(h, hc, rtol=1e-6, atol=1e-14)
    res = np.linalg.norm(c.schur_matvec(x) - b) / np.linalg.norm(b)
    assert res <= 1e-10
    assert np.linalg.norm(x - xc) / np.linalg.norm(xc) <= 1e-8


@pytest.mark.parametrize("mode", ["fused", "host", "phase"])
def test_pcg_drivers_agree_with_oracle(gpu, monkeypatch, mode):
    # persistent cooperative PCG kernel (default), the host-driven loop, and the
    # phase-split kernels of the sharded path (CUDA graph, WHILE conditional node)
    if mode != "fused":
        monkeypatch.setenv("SGW_PCG", mode)
    nx = 32
    g, c = pair(nx, 4, 2, 0.3, 0.5, 2, 4, 2, 1e-3)
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(z, z, 30, sg.ForceSpec(node=node))
    hc = c.run(z, z, 30, force_node=node, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10
    b = c.schur_matvec(rand(g.n_global, 9))
    x, rep = g.pcg(b)
    assert rep["converged"] and len(rep["residual_history"]) == rep["iterations"] + 1
    assert np.linalg.norm(c.schur_matvec(x) - b) / np.linalg.norm(b) <= 1e-10


@pytest.mark.parametrize("cfg", [(18, 3, 3, 1, 2, 2), (30, 5, 4, 1, 4, 4), (40, 4, 4, 3, 2, 3)])
def test_fused_pcg_odd_term_counts(gpu, cfg):
    # odd P+1 (3, 5): odd r_s / c_s / n_C in the persistent kernel's Psi tiles
    # (column chunks of < 64, rows past r_s), the F_cc^-1 rows' 16-byte
    # alignment, and ranges that split subdomains across CTAs; 3x3 / 5x4
    # partitions with cross points; (40, 4x4, P+1 = 10) has full 64-wide chunks
    nx, px, py, L, pin, pout = cfg
    g, c = pair(nx, px, py, 0.3, 0.5, L, pin, pout, 1e-3)
    assert c.n_corner > 0
    x = rand(g.n_global, 5)
    assert relerr(g.schur().apply_nn2(x), c.apply_nn2(x)) <= 1e-10
    b = c.schur_matvec(rand(g.n_global, 6))
    xg, rep = g.pcg(b)
    assert rep["converged"]
    assert np.linalg.norm(c.schur_matvec(xg) - b) / np.linalg.norm(b) <= 1e-10
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(z, z, 8, sg.ForceSpec(node=node))
    hc = c.run(z, z, 8, force_node=node, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10


def test_c5_l8_basis_small_mesh(gpu):
    # the C5 L = 8 basis (P+1 = 45, p_in = 4: 495 input terms) on a small mesh:
    # the JIT operator at 5 threads per node, odd P+1 everywhere in the PCG
    nx = 12
    g, c = pair(nx, 2, 2, 0.3, 0.5, 8, 4, 2, 1e-3)
    assert g.n_terms == 45
    x = rand(g.n_terms * g.n_dofs, 2)
    assert relerr(g.apply_block_transient(x), c.apply_block(x, "transient")) <= 1e-12
    r = rand(g.n_global, 3)
    assert relerr(g.schur().apply_nn2(r), c.apply_nn2(r)) <= 1e-10
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(z, z, 4, sg.ForceSpec(node=node))
    hc = c.run(z, z, 4, force_node=node, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10


def test_c1_trajectory_parity(gpu):
    # BASELINE configs[0] (C1): 64x64, 4x4, L=2, p_in 4, p_out 2, sigma 0.3, b 0.5,
    # dt 1e-3, 50 steps, tol 1e-10, Ricker f0 = 10 Hz at (0.5, 0.5)
    nx = 64
    g, c = pair(nx, 4, 4, 0.3, 0.5, 2, 4, 2, 1e-3)
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(z, z, 50, sg.ForceSpec(node=node, f0=10.0, t0=0.1))
    hc = c.run(z, z, 50, force_node=node, f0=10.0, t0=0.1, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    rel = np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"])
    assert rel <= 1e-8
    per_step = np.linalg.norm(hg.full_state - hc["full"], axis=1) / np.maximum(np.linalg.norm(hc["full"], axis=1), 1e-300)
    assert per_step[1:].max() <= 1e-8


def test_recorded_sg_nn2_iterations_on_gpu(gpu):
    # acceptance criterion 13, recorded proj/test_output.txt:52 (mean 3.00)
    nx = 24
    for L, pin, pout in [(3, 2, 3), (5, 2, 3), (3, 2, 4)]:
        coeff = O.lognormal_coeff(nx, nx, 0.1, 1.0, 1.0, L, pin)
        dt = O.cfl_dt(nx, coeff[0].max(), 0.1)
        g = sg.SgSolver(nx, nx, 4, 4, coeff, O.triple_products(L, pin, pout), params=sg.NewmarkParams(dt=dt),
                        options=sg.SgOptions(tol=1e-8))
        u0 = O.gaussian_pulse(nx, nx)
        h = g.run(u0, 0 * u0, math.ceil(0.3 / dt))
        assert f"{h.mean_iterations():.2f}" == "3.00"


def test_gaussian_pulse_trajectory_matches_oracle(gpu):
    # test_sg.cpp:218-272-style trajectory (initial displacement, damping on)
    nx = 16
    g, c = pair(nx, 2, 2, 0.25, 1.0, 2, 2, 3, 0.01)
    u0 = O.gaussian_pulse(nx, nx)
    hg = g.run(u0, 0 * u0, 12)
    hc = c.run(u0, 0 * u0, 12, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-8


@pytest.mark.parametrize("case", [(8, 2, 2, 1, 1, 1), (16, 2, 2, 2, 2, 2), (24, 2, 2, 2, 4, 2), (32, 2, 2, 2, 2, 2),
                                  (26, 4, 3, 2, 3, 2), (9, 3, 3, 1, 2, 2)])
def test_small_block_sweep_matches_tiled_and_oracle(gpu, monkeypatch, case):
    # sweep_small_kernel (B = W (P+1) <= 96: one consumer warp per subdomain,
    # rows lane, lane + 32, lane + 64 in registers) for B = 6 .. 90 (one to three
    # rows per lane), ragged frames and 2-row interiors: oracle trajectory, and
    # the tiled kernel (SGW_SWEEP_SMALL=0) on the same problem
    nx, px, py, L, pin, pout = case
    g, c = pair(nx, px, py, 0.3, 0.5, L, pin, pout, 2e-3)
    u0 = O.gaussian_pulse(nx, nx)
    hg = g.run(u0, 0 * u0, 6)
    hc = c.run(u0, 0 * u0, 6, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10
    assert np.array_equal(hg.full_state, g.run(u0, 0 * u0, 6).full_state)  # bitwise reproducible
    monkeypatch.setenv("SGW_SWEEP_SMALL", "0")
    g2, _ = pair(nx, px, py, 0.3, 0.5, L, pin, pout, 2e-3)
    ht = g2.run(u0, 0 * u0, 6)
    assert np.linalg.norm(hg.full_state - ht.full_state) / np.linalg.norm(ht.full_state) <= 1e-11


@pytest.mark.parametrize("cs", ["1", "2", "4", "8", "16"])
def test_interior_sweep_every_cluster_size(gpu, monkeypatch, cs):
    # the batched Dirichlet solve (one thread-block cluster of CS CTAs per
    # subdomain) must give the oracle trajectory for every cluster size
    monkeypatch.setenv("SGW_SWEEP_CS", cs)
    nx = 24
    g, c = pair(nx, 3, 2, 0.3, 0.5, 2, 4, 2, 2e-3)
    u0 = O.gaussian_pulse(nx, nx)
    hg = g.run(u0, 0 * u0, 6)
    hc = c.run(u0, 0 * u0, 6, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10


@pytest.mark.parametrize("batch", ["1", "5"])
def test_setup_in_subdomain_batches(gpu, monkeypatch, batch):
    # the setup processes subdomains in batches (memory bound at C3+); any batch
    # size gives the oracle's operators and trajectory
    monkeypatch.setenv("SGW_SETUP_BATCH", batch)
    nx = 24
    g, c = pair(nx, 4, 3, 0.3, 0.5, 2, 3, 2, 2e-3)
    x = rand(g.n_global, 17)
    assert relerr(g.schur().matvec(x), c.schur_matvec(x)) <= 1e-10
    assert relerr(g.schur().apply_nn2(x), c.apply_nn2(x)) <= 1e-10
    u0 = O.gaussian_pulse(nx, nx)
    hg = g.run(u0, 0 * u0, 5)
    hc = c.run(u0, 0 * u0, 5, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10


@pytest.mark.parametrize("cs", ["2", "4"])
def test_sweep_multi_tile_blocks_reproducible(gpu, monkeypatch, cs):
    # interior blocks of several 64x64 tiles (B = 47 x 6 = 282: 5 tile rows),
    # split over a cluster: oracle parity and bitwise-identical reruns (a race
    # between the ranks' shared-memory pushes would show up as run-to-run noise)
    monkeypatch.setenv("SGW_SWEEP_CS", cs)
    nx = 96
    g, c = pair(nx, 2, 2, 0.3, 0.5, 2, 2, 2, 1e-3)
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    runs = [g.run(z, z, 4, sg.ForceSpec(node=node)).full_state for _ in range(3)]
    hc = c.run(z, z, 4, force_node=node, store_full=True)
    assert np.linalg.norm(runs[0] - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10
    assert all(np.array_equal(runs[0], r) for r in runs[1:])


@pytest.mark.parametrize("cs", ["1", "4"])
def test_ragged_partition_trajectory(gpu, monkeypatch, cs):
    # partition_structured's floor-division ownership (partition.cpp:70-76)
    # with px, py not dividing nx: blocks of two widths in a padded frame
    monkeypatch.setenv("SGW_SWEEP_CS", cs)
    nx = 26
    g, c = pair(nx, 4, 3, 0.3, 0.5, 2, 3, 2, 2e-3)
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(z, z, 8, sg.ForceSpec(node=node))
    hc = c.run(z, z, 8, force_node=node, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10


@pytest.mark.timeout(900)
@pytest.mark.parametrize("world,case", [(2, (24, 24, 3, 2)), (3, (26, 20, 4, 3)), (4, (16, 16, 2, 2)),
                                        (4, (26, 26, 4, 4)), (6, (24, 24, 3, 4)), (8, (32, 32, 4, 4))])
def test_sharded_ranks_match_single_gpu(gpu, world, case):
    # the multi-GPU decomposition (include/sgw.h): ranks own 2D blocks of
    # subdomains, complete the shared interface nodes by point-to-point halo
    # exchanges and sum the coarse vector and CG scalars over the ranks; the
    # PCG runs as the phase-split kernels.  Here the ranks are threads on one
    # device (LocalGroup, host-synchronised exchanges), exercising the same
    # sharded kernels the NCCL communicator drives across GPUs.
    nx, ny, px, py = case
    coeff = O.lognormal_coeff(nx, ny, 0.3, 0.5, 0.5, 2, 3)
    t = O.triple_products(2, 3, 2)
    probes = [O.nearest_node(nx, ny, 0.5, 0.5), O.nearest_node(nx, ny, 0.2, 0.8), O.nearest_node(nx, ny, 0.9, 0.1)]
    kw = dict(params=sg.NewmarkParams(dt=2e-3), options=sg.SgOptions(tol=1e-10, store_full=True, probe_nodes=probes))
    one = sg.SgSolver(nx, ny, px, py, coeff, t, **kw)
    grp = sg.LocalGroup(world)
    ranks = grp.solvers(nx, ny, px, py, coeff, t, **kw)
    x = rand(one.n_global, 5)
    for y in grp.map(lambda r: ranks[r].schur().matvec(x)):
        assert relerr(y, one.schur().matvec(x)) <= 1e-12
    for z in grp.map(lambda r: ranks[r].schur().apply_nn2(x)):
        assert relerr(z, one.schur().apply_nn2(x)) <= 1e-10
    if one.n_corner:
        for f in grp.map(lambda r: ranks[r].schur().coarse_operator()):
            assert relerr(f, one.schur().coarse_operator()) <= 1e-12
    u0 = np.zeros((nx + 1) * (ny + 1))
    force = sg.ForceSpec(node=O.nearest_node(nx, ny, 0.5, 0.5))
    h1 = one.run(u0, u0, 8, force)
    for h in grp.map(lambda r: ranks[r].run(u0, u0, 8, force)):
        assert np.all(np.abs(h.iterations - h1.iterations) <= 1)
        assert np.linalg.norm(h.full_state - h1.full_state) / np.linalg.norm(h1.full_state) <= 1e-10
        assert np.abs(h.probe_mean - h1.probe_mean).max() <= 1e-9 * np.abs(h1.probe_mean).max()
    grp.close()


def test_nccl_one_rank_communicator(gpu):
    # the NCCL transport of the sharded path (ncclCommInitRank + ncclAllReduce on
    # the solver stream, host-driven PCG) on a 1-rank communicator
    nx = 24
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, 2, 3)
    t = O.triple_products(2, 3, 2)
    kw = dict(params=sg.NewmarkParams(dt=2e-3), options=sg.SgOptions(tol=1e-10, store_full=True))
    one = sg.SgSolver(nx, nx, 3, 2, coeff, t, **kw)
    nc = sg.SgSolver(nx, nx, 3, 2, coeff, t, rank=0, world_size=1, nccl_id=sg.nccl_unique_id(), **kw)
    x = rand(one.n_global, 3)
    assert relerr(nc.schur().matvec(x), one.schur().matvec(x)) <= 1e-14
    assert relerr(nc.schur().apply_nn2(x), one.schur().apply_nn2(x)) <= 1e-12
    u0 = O.gaussian_pulse(nx, nx)
    h1, h2 = one.run(u0, 0 * u0, 6), nc.run(u0, 0 * u0, 6)
    assert np.all(np.abs(h1.iterations - h2.iterations) <= 1)
    assert np.linalg.norm(h2.full_state - h1.full_state) / np.linalg.norm(h1.full_state) <= 1e-10


def test_solo_rank_construction(gpu):
    # one rank of a 4-rank decomposition built alone (sgw_create_solo): the
    # per-rank memory and shard kernels of configurations that need several
    # GPUs (bench.py --solo-rank); exchanges deliver zeros
    nx = 32
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, 2, 3)
    t = O.triple_products(2, 3, 2)
    kw = dict(params=sg.NewmarkParams(dt=2e-3), options=sg.SgOptions(tol=1e-10, max_iter=30))
    full = sg.SgSolver(nx, nx, 4, 4, coeff, t, **kw)
    solo = sg.SgSolver(nx, nx, 4, 4, coeff, t, rank=1, world_size=4, solo=True, **kw)
    assert solo.device_bytes < 0.6 * full.device_bytes
    x, rep = solo.pcg(rand(solo.n_global, 2))
    assert 1 <= rep["iterations"] <= 30 and np.all(np.isfinite(x))
    S_g, _ = solo.schur().local_block(2, "S")  # subdomain 2 belongs to rank 1 (2x2 rank grid)
    S_f, _ = full.schur().local_block(2, "S")
    assert np.array_equal(S_g, S_f)


def test_nonconvergence_raises(gpu):
    # sg.cpp:413-416: a step whose interface solve does not converge throws
    coeff = O.lognormal_coeff(16, 16, 0.3, 0.5, 0.5, 2, 2)
    g = sg.SgSolver(16, 16, 4, 4, coeff, O.triple_products(2, 2, 2), params=sg.NewmarkParams(dt=1e-3),
                    options=sg.SgOptions(tol=1e-14, max_iter=1))
    u0 = O.gaussian_pulse(16, 16)
    with pytest.raises(sg.SgError) as e:
        g.run(u0, 0 * u0, 2)
    assert not isinstance(e.value, ValueError)


@pytest.mark.parametrize("cfg", [(4, 2, 2, 1, 1, 0), (6, 3, 2, 1, 2, 0), (8, 1, 4, 2, 2, 1)])
def test_smallest_meshes_and_single_term(gpu, cfg):
    # edge cases: one interior node per subdomain (4x4 on 2x2), P+1 = 1
    # (deterministic limit), strips without cross points (no coarse space)
    nx, px, py, L, pin, pout = cfg
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, L, pin)
    t = O.triple_products(L, pin, pout)
    g = sg.SgSolver(nx, nx, px, py, coeff, t, params=sg.NewmarkParams(dt=1e-2),
                    options=sg.SgOptions(tol=1e-10, store_full=True))
    c = O.SgSolver(nx, nx, px, py, coeff, t, dt=1e-2, tol=1e-10)
    x = rand(g.n_terms * g.n_dofs, 4)
    assert relerr(g.apply_block_transient(x), c.apply_block(x, "transient")) <= 1e-12
    u0 = O.gaussian_pulse(nx, nx)
    hg = g.run(u0, 0 * u0, 4)
    hc = c.run(u0, 0 * u0, 4, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10


def test_zero_data_stays_zero(gpu):
    g, _ = pair(8, 2, 2, 0.2, 1.0, 2, 1, 2, 0.05)
    z = np.zeros(81)
    h = g.run(z, z, 4)
    assert np.abs(h.full_state).max() == 0.0 and np.all(h.iterations == 0)


def test_bitwise_reproducible_runs(gpu):
    g, _ = pair(16, 4, 2, 0.3, 0.5, 2, 2, 2, 0.01)
    u0 = O.gaussian_pulse(16, 16)
    a = g.run(u0, 0 * u0, 5).full_state
    b = g.run(u0, 0 * u0, 5).full_state
    assert np.array_equal(a, b)


def test_probes_match_full_state(gpu):
    nx = 16
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, 2, 2)
    probes = [O.nearest_node(nx, nx, 0.5, 0.5), O.nearest_node(nx, nx, 0.7, 0.7)]
    g = sg.SgSolver(nx, nx, 2, 2, coeff, O.triple_products(2, 2, 2), params=sg.NewmarkParams(dt=0.01),
                    options=sg.SgOptions(tol=1e-10, store_full=True, probe_nodes=probes))
    u0 = O.gaussian_pulse(nx, nx)
    h = g.run(u0, 0 * u0, 6)
    n = g.n_dofs
    for p, node in enumerate(probes):
        i, j = node % (nx + 1), node // (nx + 1)
        d = (j - 1) * (nx - 1) + (i - 1)
        assert np.array_equal(h.probe_mean[p], h.full_state[:, d])
        std = np.sqrt((h.full_state[:, n + d::n][:, : g.n_terms - 1] ** 2).sum(axis=1))
        assert np.allclose(h.probe_std[p], std, rtol=1e-14, atol=0)


def test_force_table_matches_point_source(gpu):
    # ForceFn as a nodal table (det_loop.hpp:32; rows t_0 .. t_N read straight
    # from the caller's buffer) against the same Ricker source given as a point
    # force, and a table that is too short is rejected
    nx, dt, steps = 16, 2e-3, 8
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, 2, 2)
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    g = sg.SgSolver(nx, nx, 2, 2, coeff, O.triple_products(2, 2, 2), params=sg.NewmarkParams(dt=dt),
                    options=sg.SgOptions(tol=1e-10, store_full=True))
    z = np.zeros((nx + 1) ** 2)
    table = np.zeros((steps + 1, (nx + 1) ** 2))
    t = 0.0
    for k in range(steps + 1):  # the solver's own time accumulation (t += dt)
        table[k, node] = sg.ricker(t, 10.0, 0.1)
        t += dt
    hp = g.run(z, z, steps, sg.ForceSpec(node=node, f0=10.0, t0=0.1))
    ht = g.run(z, z, steps, sg.ForceSpec(table=table))
    assert np.array_equal(hp.iterations, ht.iterations)
    assert np.abs(hp.full_state - ht.full_state).max() <= 1e-14 * np.abs(hp.full_state).max()
    ht2 = g.run(z, z, steps, sg.ForceSpec(table=table))  # rerun from the same buffer: bitwise identical
    assert np.array_equal(ht.full_state, ht2.full_state)
    with pytest.raises(Exception):
        g.run(z, z, steps + 2, sg.ForceSpec(table=table[: steps + 1].copy()))


def test_constrained_probe_rejected(gpu):
    coeff = O.lognormal_coeff(8, 8, 0.2, 1.0, 1.0, 1, 1)
    g = sg.SgSolver(8, 8, 2, 2, coeff, O.triple_products(1, 1, 1), params=sg.NewmarkParams(dt=0.05),
                    options=sg.SgOptions(probe_nodes=[0]))
    with pytest.raises(ValueError):
        g.run(np.zeros(81), np.zeros(81), 1)


@pytest.mark.timeout(1200)
def test_c2_full_size_parity_and_properties(gpu):
    # BASELINE configs[1] (C2) at full size: 256x256, 8x8 subdomains, P+1 = 20,
    # n_in = 84.  Three Newmark steps against the oracle (iterations +-1,
    # trajectory 1e-8), and size-independent properties of the operators:
    # symmetry of S and NN2 (test_dd.cpp:77-96), linearity of the SG operator.
    import bench
    c = bench.CONFIGS["C2"]
    nx = c["nx"]
    coeff = O.lognormal_coeff(nx, nx, c["sigma"], c["b"], c["b"], c["L"], c["p_in"])
    t = O.triple_products(c["L"], c["p_in"], c["p_out"])
    g = sg.SgSolver(nx, nx, c["px"], c["px"], coeff, t, alpha0=bench.ALPHA0, alpha1=bench.ALPHA1,
                    params=sg.NewmarkParams(dt=c["dt"]), options=sg.SgOptions(tol=bench.TOL, store_full=True))
    x, y = rand(g.n_global, 41), rand(g.n_global, 42)
    S = g.schur()
    a, b = y @ S.matvec(x), x @ S.matvec(y)
    assert abs(a - b) <= 1e-11 * abs(b)
    a, b = y @ S.apply_nn2(x), x @ S.apply_nn2(y)
    assert abs(a - b) <= 1e-11 * abs(b)
    u, w = rand(g.n_terms * g.n_dofs, 43), rand(g.n_terms * g.n_dofs, 44)
    lhs = g.apply_block_transient(2.0 * u - 3.0 * w)
    rhs = 2.0 * g.apply_block_transient(u) - 3.0 * g.apply_block_transient(w)
    assert relerr(lhs, rhs) <= 1e-13
    cpu = O.SgSolver(nx, nx, c["px"], c["px"], coeff, t, alpha0=bench.ALPHA0, alpha1=bench.ALPHA1, dt=c["dt"],
                     tol=bench.TOL)
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(z, z, 3, sg.ForceSpec(node=node, f0=bench.F0, t0=bench.T0))
    hc = cpu.run(z, z, 3, force_node=node, f0=bench.F0, t0=bench.T0, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-8


@pytest.mark.parametrize("cfg", [(16, 4, 2, 2, 4, 2), (22, 4, 3, 2, 2, 2)])
def test_reduced_memory_mode_matches_oracle(gpu, cfg):
    # S_s not stored, applied as A_GG - A_GI A_II^-1 A_IG through
    # the local stencils and the interior sweep (include/sgw.h implicit_schur)
    nx, px, py, L, pin, pout = cfg
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, L, pin)
    t = O.triple_products(L, pin, pout)
    mk = lambda imp: sg.SgSolver(nx, nx, px, py, coeff, t, params=sg.NewmarkParams(dt=1e-3),  # noqa: E731
                                 options=sg.SgOptions(tol=1e-10, store_full=True, implicit_schur=imp))
    g, e = mk(True), mk(False)
    c = O.SgSolver(nx, nx, px, py, coeff, t, dt=1e-3, tol=1e-10)
    assert g.device_bytes < e.device_bytes
    x = rand(c.n_global, 4)
    assert relerr(g.schur().matvec(x), c.schur_matvec(x)) <= 1e-10
    b = c.schur_matvec(rand(c.n_global, 8))
    xg, rep = g.pcg(b)
    assert rep["converged"] and np.linalg.norm(c.schur_matvec(xg) - b) / np.linalg.norm(b) <= 1e-10
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(z, z, 8, sg.ForceSpec(node=node))
    hc = c.run(z, z, 8, force_node=node, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10


@pytest.mark.parametrize("mode", ["fused", "host", "phase"])
def test_nonconvergence_leaves_state_unadvanced(gpu, monkeypatch, mode):
    # sg.cpp:412-416: a step whose interface PCG fails throws before
    # newmark_update.  The persistent PCG's verdict is read after the step's
    # update is queued, so the update and the probe row are conditional on the
    # device-side flag: the state, the time and the step index stay put.
    if mode != "fused":
        monkeypatch.setenv("SGW_PCG", mode)
    nx = 16
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, 2, 2)
    t = O.triple_products(2, 2, 2)
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    g = sg.SgSolver(nx, nx, 2, 2, coeff, t, params=sg.NewmarkParams(dt=1e-3),
                    options=sg.SgOptions(tol=1e-14, max_iter=1, probe_nodes=[node]))
    z = np.zeros((nx + 1) ** 2)
    g.init_state(O.gaussian_pulse(nx, nx), z)
    u0 = g.state()
    with pytest.raises(sg.SgError) as e:
        g.advance(1)
    assert e.value.code == sg.SGW_ENOCONV
    assert np.array_equal(g.state(), u0)


def test_nonconvergence_with_next_rhs_launched_ahead(gpu):
    # advance(n > 1) puts the next step's right-hand side on the stream before
    # it reads the current step's verdict (step.cu launch_rhs): a failed solve
    # must still leave the state, the time and the step index untouched, and
    # the dropped right-hand side must not leak into a later step
    nx = 16
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, 2, 2)
    t = O.triple_products(2, 2, 2)
    g = sg.SgSolver(nx, nx, 2, 2, coeff, t, params=sg.NewmarkParams(dt=1e-3),
                    options=sg.SgOptions(tol=1e-14, max_iter=1))
    z = np.zeros((nx + 1) ** 2)
    g.init_state(O.gaussian_pulse(nx, nx), z)
    u0 = g.state()
    for _ in range(2):
        with pytest.raises(sg.SgError) as e:
            g.advance(3)
        assert e.value.code == sg.SGW_ENOCONV
        assert np.array_equal(g.state(), u0)


def test_advance_in_one_call_equals_step_by_step(gpu):
    # the right-hand side launched ahead inside advance(n) is the one a
    # step-by-step caller computes: same iterations, bitwise the same state
    nx = 24
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    runs = []
    for chunks in ([7], [1] * 7, [3, 4]):
        g, _ = pair(nx, 3, 2, 0.3, 0.5, 2, 4, 2, 1e-3)
        g.init_state(O.gaussian_pulse(nx, nx), z, sg.ForceSpec(node=node))
        its = np.concatenate([g.advance(k) for k in chunks])
        runs.append((its, g.state()))
    for its, u in runs[1:]:
        assert np.array_equal(its, runs[0][0])
        assert np.array_equal(u, runs[0][1])


def test_step_without_coupling_blocks_matches_oracle(gpu, monkeypatch):
    # the coupling / interface-force blocks are built at setup only while
    # memory allows; without them the step takes the stencil
    # kernels (coupling_kernel, local_force_kernel): same trajectory
    monkeypatch.setenv("SGW_NO_CPL_BLOCKS", "1")
    nx = 24
    g, c = pair(nx, 3, 2, 0.3, 0.5, 2, 4, 2, 1e-3)
    node = O.nearest_node(nx, nx, 0.5, 0.5)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(z, z, 6, sg.ForceSpec(node=node))
    hc = c.run(z, z, 6, force_node=node, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10


@pytest.mark.parametrize("nx,L,pin,pout", [(12, 2, 2, 2), (17, 2, 4, 2)])
def test_single_subdomain_direct_path(gpu, nx, L, pin, pout):
    # sg.cpp:146 / :158-172 / :301-305: one subdomain, no interface: each step
    # solves the whole stochastic transient system directly (the GPU's
    # interior block-Thomas solve over all dofs), 0 PCG iterations
    g, c = pair(nx, 1, 1, 0.3, 0.5, L, pin, pout, 1e-3)
    assert g.n_global == 0
    u0 = O.gaussian_pulse(nx, nx)
    z = np.zeros((nx + 1) ** 2)
    hg = g.run(u0, z, 5, sg.ForceSpec(node=O.nearest_node(nx, nx, 0.5, 0.5)))
    hc = c.run(u0, z, 5, force_node=O.nearest_node(nx, nx, 0.5, 0.5), store_full=True)
    assert np.all(hg.iterations == 0) and np.all(hc["iterations"] == 0)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10


@pytest.mark.parametrize("cfg", [(8, 8, 4), (7, 4, 7)])
def test_one_cell_subdomains_sg_trajectory(gpu, cfg):
    # SG system (P+1 = 6) on partitions with one-cell blocks (no interior
    # dofs, test_dd.cpp:98-107): S_s = K~_GG, blocks mixed with two-cell ones
    nx, px, py = cfg
    g, c = pair(nx, px, py, 0.3, 0.5, 2, 4, 2, 1e-2)
    x = rand(g.n_global, 5)
    assert relerr(g.schur().matvec(x), c.schur_matvec(x)) <= 1e-11
    assert relerr(g.schur().apply_nn2(x), c.apply_nn2(x)) <= 1e-10
    u0 = O.gaussian_pulse(nx, nx)
    hg = g.run(u0, 0 * u0, 4)
    hc = c.run(u0, 0 * u0, 4, store_full=True)
    assert np.all(np.abs(hg.iterations - hc["iterations"]) <= 1)
    assert np.linalg.norm(hg.full_state - hc["full"]) / np.linalg.norm(hc["full"]) <= 1e-10
