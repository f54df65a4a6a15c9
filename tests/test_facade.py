"""The C++ facade (include/mprec_gpu.hpp) compiles against the C ABI and, on a
B200, runs the reference-style checks in tests/cpp/test_facade.cpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1912_04385_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")


def _build(tmp_path):
    exe = str(tmp_path / "test_facade")
    subprocess.run(["g++", "-std=c++17", "-O1", "-o", exe, SRC, "-I", os.path.join(ROOT, "include"),
                    "-L", PKG, "-lmprec_gpu", "-lmprec_gen", f"-Wl,-rpath,{PKG}"], check=True)
    return exe


def test_facade_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_facade_runs_on_gpu(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "all facade checks passed" in out.stdout
