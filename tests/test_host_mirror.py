"""The C++ host mirror (include/sgwave_b200.hpp) — the reference's interface in
C++ over the C ABI — built and run as a C++ test program (tests/cpp)."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
CPP = os.path.join(HERE, "cpp")


def build():
    if not shutil.which(os.environ.get("CXX", "g++")):
        pytest.skip("no C++ compiler")
    r = subprocess.run(["make", "-s", "-C", CPP], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return os.path.join(CPP, "build", "test_host_mirror")


def run(mode):
    r = subprocess.run([build(), mode], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


def test_cpp_mirror_builders_and_argument_checking():
    run("cpu")


def test_cpp_mirror_without_gpu_reports_runtime_error():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    run("nogpu")


@pytest.mark.gpu
def test_cpp_mirror_parity_with_oracle(gpu):
    run("gpu")
