"""solve-sg data files (experiments.cpp:393-434, docs/outputs.md:19-30) written
from an SgHistory: CsvWriter's %.17g format (io.cpp:15-44), step numbering,
moments (sg.cpp:17-26) and the Dirichlet expansion of snapshots."""
import csv
import os

import numpy as np
import pytest

import oracle as O
from paper_2512_23027_b200.sgwave import SgHistory, moments, write_sg_outputs


def read(path):
    with open(path) as f:
        return list(csv.reader(f))


def synthetic(nx=4, ny=3, nt=3, steps=2):
    n = (nx - 1) * (ny - 1)
    rng = np.random.default_rng(5)
    full = rng.normal(size=(steps + 1, nt * n))
    pc = rng.normal(size=(1, nt, steps + 1))
    return SgHistory(times=np.cumsum(np.r_[0.0, np.full(steps, 0.1)]), iterations=np.array([3, 4], np.int32),
                     residual=np.array([1e-11, 2.5e-11]), probe_mean=pc[:, 0, :].copy(),
                     probe_std=np.sqrt((pc[:, 1:, :] ** 2).sum(axis=1)), full_state=full, probe_coeffs=pc)


def test_writers_format_and_values(tmp_path):
    h = synthetic()
    names = write_sg_outputs(str(tmp_path), h, 4, 3, 0.1, snapshot_times=(0.1, 7.0))
    assert names == ["probe_0.csv", "iterations.csv", "snapshot_0.csv", "snapshot_1.csv"]
    p = read(os.path.join(tmp_path, "probe_0.csv"))
    assert p[0] == ["t", "mean", "std", "u0", "u1", "u2"]
    for s, row in enumerate(p[1:]):  # %.17g round-trips every double exactly
        vals = [float(v) for v in row]
        assert vals[0] == h.times[s] and vals[1] == h.probe_mean[0, s] and vals[2] == h.probe_std[0, s]
        assert vals[3:] == list(h.probe_coeffs[0, :, s])
        assert all(v == "%.17g" % float(v) for v in row)
    it = read(os.path.join(tmp_path, "iterations.csv"))
    assert it[0] == ["step", "iterations", "final_residual"]
    assert it[1] == ["1", "3", "9.9999999999999994e-12"] and it[2][:2] == ["2", "4"]
    snap = read(os.path.join(tmp_path, "snapshot_0.csv"))
    assert snap[0] == ["node_id", "x", "y", "mean", "std"] and len(snap) == 1 + 5 * 4
    mean, sd = moments(h.full_state[1], 6)  # t = 0.1 -> step 1
    node = 1 * 5 + 2  # (gi, gj) = (2, 1) -> dof (0)*3 + 1
    row = [float(v) for v in snap[1 + node]]
    assert row[:3] == [node, 2 / 4, 1 / 3] and row[3] == mean[1] and row[4] == sd[1]
    assert all(float(r[3]) == 0.0 for r in snap[1:] if int(float(r[0])) in (0, 4, 5, 19))  # Dirichlet
    last = read(os.path.join(tmp_path, "snapshot_1.csv"))  # beyond the run: last state (min(...))
    m2, _ = moments(h.full_state[-1], 6)
    assert float(last[1 + node][3]) == m2[1]


@pytest.mark.gpu
def test_gpu_history_outputs_match_oracle(gpu, tmp_path):
    import paper_2512_23027_b200 as sg
    nx = 16
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, 2, 2)
    t = O.triple_products(2, 2, 2)
    probes = [O.nearest_node(nx, nx, 0.5, 0.5), O.nearest_node(nx, nx, 0.25, 0.75)]
    g = sg.SgSolver(nx, nx, 2, 2, coeff, t, params=sg.NewmarkParams(dt=1e-2),
                    options=sg.SgOptions(tol=1e-10, store_full=True, probe_nodes=probes))
    c = O.SgSolver(nx, nx, 2, 2, coeff, t, dt=1e-2, tol=1e-10)
    u0 = O.gaussian_pulse(nx, nx)
    h = g.run(u0, 0 * u0, 6)
    hc = c.run(u0, 0 * u0, 6, store_full=True)
    n = g.n_dofs
    for p, node in enumerate(probes):
        d = (node // (nx + 1) - 1) * (nx - 1) + node % (nx + 1) - 1
        coeffs = hc["full"][:, d::n][:, : g.n_terms].T  # terms x steps from the oracle state
        assert np.abs(h.probe_coeffs[p] - coeffs).max() <= 1e-8 * np.abs(coeffs).max()
        assert np.array_equal(h.probe_coeffs[p][0], h.probe_mean[p])
    names = sg.write_sg_outputs(str(tmp_path), h, nx, nx, 1e-2, snapshot_times=(0.03,))
    assert "snapshot_0.csv" in names and "probe_1.csv" in names
    snap = np.array([[float(v) for v in r] for r in read(os.path.join(tmp_path, "snapshot_0.csv"))[1:]])
    mean, sd = moments(hc["full"][3], n)
    inner = [(j + 1) * (nx + 1) + i + 1 for j in range(nx - 1) for i in range(nx - 1)]
    assert np.abs(snap[inner, 3] - mean).max() <= 1e-8 * np.abs(mean).max()
    assert np.abs(snap[inner, 4] - sd).max() <= 1e-8 * np.abs(sd).max()
