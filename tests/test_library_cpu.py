"""CPU-side checks of the product library: the C ABI loads, exports every
symbol include/sgw.h declares, its host input builders agree with the oracle,
and compute entry points fail loudly without a GPU (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sg = pytest.importorskip("paper_2512_23027_b200")


def header_symbols():
    text = open(os.path.join(ROOT, "include", "sgw.h")).read()
    return sorted(set(re.findall(r"\b(sgw_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = sg.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


@pytest.mark.parametrize("args", [(16, 16, 0.3, 0.5, 0.5, 2, 4), (12, 10, 0.4, 0.3, 0.7, 3, 2), (8, 8, 0.0, 1.0, 1.0, 3, 2)])
def test_lognormal_builder_matches_oracle(args):
    nx, ny, sigma, bx, by, L, pin = args
    a = sg.lognormal_coeff(nx, ny, sigma, bx, by, L, pin)
    b = O.lognormal_coeff(nx, ny, sigma, bx, by, L, pin)
    assert a.shape == b.shape
    assert np.abs(a - b).max() <= 1e-15 * np.abs(b).max()


@pytest.mark.parametrize("args", [(2, 4, 2), (3, 6, 3), (4, 6, 3), (3, 2, 3), (1, 0, 0)])
def test_triple_products_builder_matches_oracle(args):
    a = sg.triple_products(*args)
    b = O.triple_products(*args)
    assert (a.n_input, a.n_output) == (b.n_input, b.n_output)
    assert np.array_equal(a.i, b.i) and np.array_equal(a.j, b.j) and np.array_equal(a.k, b.k)
    assert np.array_equal(a.v, b.v)


def test_nearest_node_matches_oracle():
    for nx, x, y in [(64, 0.5, 0.5), (256, 0.5, 0.5), (24, 0.7, 0.7), (33, 0.2, 0.7)]:
        assert sg.nearest_node(nx, nx, x, y) == O.nearest_node(nx, nx, x, y)


def test_compute_without_gpu_fails_loudly():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    coeff = O.lognormal_coeff(8, 8, 0.2, 1.0, 1.0, 1, 1)
    with pytest.raises(sg.SgError):
        sg.SgSolver(8, 8, 2, 2, coeff, O.triple_products(1, 1, 1))


def test_invalid_arguments_rejected_before_device_work():
    coeff = O.lognormal_coeff(8, 8, 0.2, 1.0, 1.0, 2, 1)
    with pytest.raises(ValueError):  # mismatched tensor (test_sg.cpp "mismatched ... rejected")
        sg.SgSolver(8, 8, 2, 2, coeff, O.triple_products(2, 2, 2))


def test_problem_struct_layout_matches_header(tmp_path):
    # the ctypes mirror of sgw_problem must match the C layout field by field
    import ctypes
    import shutil
    import subprocess

    if not shutil.which("gcc"):
        pytest.skip("no C compiler")
    src = tmp_path / "layout.c"
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "sgw.h"\n'
                   'int main(void) { printf("%zu %zu %zu %zu\\n", sizeof(sgw_problem), '
                   'offsetof(sgw_problem, nccl_id), offsetof(sgw_problem, precond), '
                   'offsetof(sgw_problem, implicit_schur)); return 0; }\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    size, o_id, o_pc, o_imp = (int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                                              check=True).stdout.split())
    P = sg.sgwave._Problem
    assert ctypes.sizeof(P) == size
    assert (P.nccl_id.offset, P.precond.offset, P.implicit_schur.offset) == (o_id, o_pc, o_imp)


def test_preconditioner_names():
    # precond_from_string (dd.hpp:100); test_cli_io.cpp:65 rejects "jacobi"
    assert [sg.precond_from_string(k) for k in ("nn2", "nn1", "lumped")] == [0, 1, 2]
    with pytest.raises(ValueError):
        sg.precond_from_string("jacobi")
    coeff = O.lognormal_coeff(8, 8, 0.2, 1.0, 1.0, 1, 1)
    with pytest.raises(ValueError):  # rejected before any device work
        sg.SgSolver(8, 8, 2, 2, coeff, O.triple_products(1, 1, 1), options=sg.SgOptions(precond="jacobi"))
