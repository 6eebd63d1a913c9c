"""The reference's generic entry points on the GPU: pcg over arbitrary
operators (include/sgwave/pcg.hpp:15-21, src/pcg.cpp:7-50; test_dd.cpp:215-246)
and a SchurSystem built from hand-made LocalSchur data (dd.hpp:50-96;
test_dd.cpp:123-151), checked against the oracle's SchurSystem on the same
locals (oracle.local_schur) and against dense numpy algebra."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
sg = pytest.importorskip("paper_2512_23027_b200")


def test_pcg_basics(gpu):
    # test_dd.cpp:215-246, the same three subcases
    a = np.array([[4.0, 1, 0], [1, 3, 1], [0, 1, 2]])
    x, rep = sg.pcg(lambda v: a @ v, lambda v: v, np.zeros(3), 1e-12, 10)
    assert rep["converged"] and rep["iterations"] == 0 and np.linalg.norm(x) == 0.0
    b = np.array([1.0, 2, 3])
    x, rep = sg.pcg(lambda v: a @ v, lambda v: v, b, 1e-12, 10)
    assert rep["converged"] and rep["iterations"] <= 3 and np.linalg.norm(a @ x - b) <= 1e-10
    assert len(rep["residual_history"]) == rep["iterations"] + 1 and rep["residual_history"][0] == 1.0
    ainv = np.linalg.inv(a)
    x, rep = sg.pcg(lambda v: a @ v, lambda v: ainv @ v, np.array([-1.0, 0.5, 2]), 1e-12, 10)
    assert rep["converged"] and rep["iterations"] == 1


def test_pcg_nonconvergence_and_identity_precond(gpu):
    rng = np.random.default_rng(1)
    m = rng.normal(size=(40, 40))
    a = m @ m.T + 40 * np.eye(40)
    b = rng.normal(size=40)
    x, rep = sg.pcg(lambda v: a @ v, None, b, 1e-14, 3)  # max_iter reached
    assert not rep["converged"] and rep["iterations"] == 3 and len(rep["residual_history"]) == 4
    x, rep = sg.pcg(lambda v: a @ v, None, b, 1e-12, 200)
    assert rep["converged"] and np.linalg.norm(a @ x - b) <= 1e-10 * np.linalg.norm(b)


def test_pcg_operator_exception_propagates(gpu):
    def bad(v):
        raise ValueError("operator failed")
    with pytest.raises(ValueError, match="operator failed"):
        sg.pcg(bad, None, np.ones(4), 1e-10, 5)


def test_two_level_with_one_block_and_no_corners_is_exact_inverse(gpu):
    # test_dd.cpp:123-151: one local, no corners: apply_nn2 = S^-1, PCG in 1 iteration
    n = 7
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, (n, n))
    a = a @ a.T + n * np.eye(n)
    ls = sg.LocalSchur(S=a, gmap=np.arange(n), weights=np.ones(n), r_idx=np.arange(n))
    sys = sg.SchurFromLocals(n, 0, [ls])
    r = rng.uniform(-1, 1, n)
    z = sys.apply_nn2(r)
    assert np.abs(a @ z - r).max() <= 1e-10
    x, rep = sys.pcg(r, 1e-10, 50)
    assert rep["converged"] and rep["iterations"] == 1


def test_llt_regularized_retry_on_a_floating_block(gpu):
    # dd.cpp:66-76: a singular PSD block (a floating subdomain: constants in the
    # null space) hits an exact zero pivot in the first Cholesky; the retry
    # factors S + 1e-10 trace(S) / n I.  The response to the null-space vector
    # is 1 / shift, so it pins the shift the retry branch applied.
    S = np.array([[1.0, -1.0], [-1.0, 1.0]])
    ls = sg.LocalSchur(S=S, gmap=np.arange(2), weights=np.ones(2), r_idx=np.arange(2))
    sys = sg.SchurFromLocals(2, 0, [ls])
    shift = 1e-10 * np.trace(S) / 2
    for r in (np.array([1.0, 1.0]), np.array([1.0, 0.0])):
        z = sys.apply_nn2(r)
        ref = np.linalg.solve(S + shift * np.eye(2), r)
        assert np.abs(z - ref).max() <= 1e-5 * np.abs(ref).max()
    # an indefinite block still fails after the shift (dd.cpp:72-74)
    bad = sg.LocalSchur(S=np.array([[1.0, 2.0], [2.0, 1.0]]), gmap=np.arange(2), weights=np.ones(2), r_idx=np.arange(2))
    with pytest.raises(Exception, match="regulariz"):
        sg.SchurFromLocals(2, 0, [bad])


def _random_locals(seed=3):
    """three overlapping locals on a 10-node interface whose last 2 nodes are corners"""
    rng = np.random.default_rng(seed)
    specs = [([0, 1, 2, 3, 8], [8]), ([3, 4, 5, 6, 8, 9], [8, 9]), ([6, 7, 0, 9, 2], [9])]
    mult = np.zeros(10)
    for g, _ in specs:
        mult[g] += 1
    out = []
    for g, cs in specs:
        n = len(g)
        m = rng.uniform(-1, 1, (n, n))
        S = m @ m.T + n * np.eye(n)
        c_idx = [g.index(c) for c in cs]
        r_idx = [k for k in range(n) if k not in c_idx]
        out.append(sg.LocalSchur(S=S, gmap=np.array(g), weights=1.0 / mult[g], r_idx=np.array(r_idx),
                                 c_idx=np.array(c_idx), corner_gmap=np.array([c - 8 for c in cs])))
    return out


def test_schur_from_locals_against_dense_algebra(gpu):
    locs = _random_locals()
    sys = sg.SchurFromLocals(10, 2, locs)
    x = np.random.default_rng(9).uniform(-1, 1, 10)
    # matvec: sum_s R_s^T S_s R_s x (dd.cpp:142-157)
    y = np.zeros(10)
    for ls in locs:
        y[ls.gmap] += ls.S @ x[ls.gmap]
    assert np.abs(sys.matvec(x) - y).max() <= 1e-12 * np.abs(y).max()
    # coarse operator: sum_s B_c^T (S_cc - S_rc^T S_rr^-1 S_rc) B_c (dd.cpp:122-137)
    F = np.zeros((2, 2))
    for ls in locs:
        r, c = ls.r_idx, ls.c_idx
        Sc = ls.S[np.ix_(c, c)] - ls.S[np.ix_(r, c)].T @ np.linalg.solve(ls.S[np.ix_(r, r)], ls.S[np.ix_(r, c)])
        F[np.ix_(ls.corner_gmap, ls.corner_gmap)] += Sc
    assert np.abs(sys.coarse_operator() - F).max() <= 1e-12 * np.abs(F).max()
    # NN2 (dd.cpp:199-253) as a dense restatement
    d = np.zeros(2)
    ts = []
    for ls in locs:
        rl = x[ls.gmap] * ls.weights
        t = np.linalg.solve(ls.S[np.ix_(ls.r_idx, ls.r_idx)], rl[ls.r_idx])
        ts.append(t)
        d[ls.corner_gmap] += rl[ls.c_idx] - ls.S[np.ix_(ls.r_idx, ls.c_idx)].T @ t
    uc = np.linalg.solve(F, d)
    z = np.zeros(10)
    for ls, t in zip(locs, ts):
        ucl = uc[ls.corner_gmap]
        ur = t - np.linalg.solve(ls.S[np.ix_(ls.r_idx, ls.r_idx)], ls.S[np.ix_(ls.r_idx, ls.c_idx)] @ ucl)
        zl = np.zeros(len(ls.gmap))
        zl[ls.c_idx], zl[ls.r_idx] = ucl, ur
        z[ls.gmap] += zl * ls.weights
    assert np.abs(sys.apply_nn2(x) - z).max() <= 1e-10 * np.abs(z).max()
    # PCG on S u = b with NN2
    b = sys.matvec(np.linspace(-1, 1, 10))
    u, rep = sys.pcg(b, 1e-12, 100)
    assert rep["converged"] and np.abs(u - np.linspace(-1, 1, 10)).max() <= 1e-9


def test_schur_from_locals_matches_the_structured_solver(gpu):
    # the oracle's own LocalSchur blocks of a real partition, injected: the
    # generic GPU system reproduces the structured GPU solver's matvec / NN2
    nx = 16
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, 2, 2)
    t = O.triple_products(2, 2, 2)
    c = O.SgSolver(nx, nx, 2, 2, coeff, t, dt=1e-3, tol=1e-10)
    g = sg.SgSolver(nx, nx, 2, 2, coeff, t, params=sg.NewmarkParams(dt=1e-3), options=sg.SgOptions(tol=1e-10))
    locs = []
    for s in range(4):
        d = c.local_schur_full(s)
        locs.append(sg.LocalSchur(S=d["S"], gmap=d["gmap"], weights=d["weights"], r_idx=d["r_idx"],
                                  c_idx=d["c_idx"], corner_gmap=d["corner_gmap"]))
    sys = sg.SchurFromLocals(g.n_global, g.schur().n_corner, locs)
    x = np.random.default_rng(2).uniform(-1, 1, g.n_global)
    assert np.abs(sys.matvec(x) - g.schur().matvec(x)).max() <= 1e-10 * np.abs(g.schur().matvec(x)).max()
    z = g.schur().apply_nn2(x)
    assert np.abs(sys.apply_nn2(x) - z).max() <= 1e-9 * np.abs(z).max()
