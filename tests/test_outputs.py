"""solve-sg data files (experiments.cpp:393-434, docs/outputs.md:19-30) written
from an SgHistory: CsvWriter's %.17g format (io.cpp:15-44), step numbering,
moments (sg.cpp:17-26) and the Dirichlet expansion of snapshots."""
import csv
import os

import numpy as np
import pytest

import oracle as O
from paper_2512_23027_b200.sgwave import (SgHistory, kle_spectrum, moments, pce_indices, svg_lines,
                                          write_sg_outputs)


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
    assert names == ["probe_0.csv", "iterations.csv", "snapshot_0.csv", "snapshot_1.csv", "probes.svg"]
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


def test_solve_sg_output_set_order_and_contents(tmp_path):
    # driver_solve_sg's file set and order (experiments.cpp:393-449) plus the
    # manifest (run_driver, :741-754; io.cpp:131-140)
    h = synthetic()
    man = {"command": "solve-sg", "config": {"nx": 4, "ny": 3}, "seed": 7, "wall_seconds": 1.5}
    names = write_sg_outputs(str(tmp_path), h, 4, 3, 0.1, snapshot_times=(0.1,), kle=(0.3, 0.5, 0.5, 3),
                             pce=(3, 2), manifest=man)
    assert names == ["probe_0.csv", "kle_spectrum.csv", "pce_indices.csv", "iterations.csv", "snapshot_0.csv",
                     "probes.svg", "manifest.json"]
    # kle_spectrum.csv: KleMode::lambda = sigma^2 lambda_x lambda_y (kle.cpp:80-133, 161-167), vs the oracle
    k = read(os.path.join(tmp_path, "kle_spectrum.csv"))
    assert k[0] == ["n", "lambda"] and [int(r[0]) for r in k[1:]] == [1, 2, 3]
    lam = O.kle_lambdas(4, 3, 0.3, 0.5, 0.5, 3)
    assert np.allclose([float(r[1]) for r in k[1:]], lam, rtol=1e-14, atol=0)
    assert all(r[1] == "%.17g" % float(r[1]) for r in k[1:])
    # pce_indices.csv: graded order, total order, ';'-joined exponents (pce.cpp:19-37, 84-94)
    pi = read(os.path.join(tmp_path, "pce_indices.csv"))
    assert pi[0] == ["term", "total_order", "exponents"] and len(pi) == 1 + 10
    assert pi[1] == ["0", "0", "0;0;0"] and pi[2] == ["1", "1", "1;0;0"] and pi[4] == ["3", "1", "0;0;1"]
    assert pi[5] == ["4", "2", "2;0;0"] and pi[10] == ["9", "2", "0;0;2"]
    assert all(int(r[1]) == sum(int(v) for v in r[2].split(";")) for r in pi[1:])
    # probes.svg: one mean and one std polyline per probe (write_svg_lines)
    svg = open(os.path.join(tmp_path, "probes.svg")).read()
    assert svg.startswith('<svg xmlns="http://www.w3.org/2000/svg" width="720" height="480">')
    assert svg.count("<polyline") == 2 and "mean p0" in svg and "std p0" in svg and svg.endswith("</svg>\n")
    import json
    m = json.load(open(os.path.join(tmp_path, "manifest.json")))
    assert m == {"command": "solve-sg", "config": {"nx": 4, "ny": 3}, "seed": 7, "wall_seconds": 1.5,
                 "version": "0.1.0", "outputs": names[:-1]}


def test_svg_axes_and_points():
    # write_svg_lines geometry (io.cpp:58-123): data range -> plot box [70, 560] x [430, 40]
    svg = svg_lines("T", "x", "y", [("a", [0.0, 1.0, 2.0], [1.0, 3.0, 2.0])])
    assert 'points="70,430 315,40 560,235 "' in svg
    assert '<text x="70" y="446" text-anchor="middle" font-size="10">0</text>' in svg
    assert '<text x="64" y="43" text-anchor="end" font-size="10">3</text>' in svg


def test_pce_indices_and_kle_spectrum_builders():
    ix = pce_indices(2, 3)
    assert ix.tolist() == [[0, 0], [1, 0], [0, 1], [2, 0], [1, 1], [0, 2], [3, 0], [2, 1], [1, 2], [0, 3]]
    assert len(pce_indices(6, 4)) == 210  # C4's input basis
    lam = kle_spectrum(0.4, 0.3, 0.3, 4)
    assert np.allclose(lam, O.kle_lambdas(8, 8, 0.4, 0.3, 0.3, 4), rtol=1e-14, atol=0) and np.all(np.diff(lam) <= 0)


@pytest.mark.gpu
def test_gpu_solve_sg_outputs_byte_identical_reruns(gpu, tmp_path):
    # acceptance criterion 16 (acceptance.cpp:570-606): two runs of the same
    # solve-sg configuration write byte-identical .csv files
    import paper_2512_23027_b200 as sg
    nx = 12
    coeff = O.lognormal_coeff(nx, nx, 0.3, 0.5, 0.5, 2, 2)
    t = O.triple_products(2, 2, 2)
    probes = [O.nearest_node(nx, nx, 0.5, 0.5), O.nearest_node(nx, nx, 0.2, 0.7)]
    outs = []
    for r in range(2):
        g = sg.SgSolver(nx, nx, 2, 2, coeff, t, params=sg.NewmarkParams(dt=1e-2),
                        options=sg.SgOptions(tol=1e-10, store_full=True, probe_nodes=probes))
        h = g.run(O.gaussian_pulse(nx, nx), np.zeros((nx + 1) ** 2), 15)
        d = tmp_path / f"run{r}"
        outs.append((d, sg.write_sg_outputs(str(d), h, nx, nx, 1e-2, snapshot_times=(0.1,), kle=(0.3, 0.5, 0.5, 2),
                                            pce=(2, 2), manifest={"command": "solve-sg", "seed": 0,
                                                                  "wall_seconds": float(r)})))
        del g
    (d1, n1), (d2, n2) = outs
    assert n1 == n2
    csvs = [n for n in n1 if n.endswith(".csv")]
    assert len(csvs) >= 6
    for n in csvs + ["probes.svg"]:
        assert (d1 / n).read_bytes() == (d2 / n).read_bytes(), n


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
