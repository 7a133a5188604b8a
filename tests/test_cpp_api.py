"""The C++ host API (include/hermsim_b200/hermsim.hpp) compiles as documented in INTEGRATION.md and,
on a GPU, runs a reference-style caller end to end (tests/cpp/api_demo.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_15765_b200", "lib")


def _build(tmp_path):
    exe = str(tmp_path / "api_demo")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp", "api_demo.cpp"),
           "-L", LIB, "-lhermsim_b200", f"-Wl,-rpath,{LIB}", "-o", exe]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


def test_cpp_api_compiles(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_cpp_api_runs(tmp_path):
    env = dict(os.environ, API_DEMO_OHRM=str(tmp_path / "rho.ohrm"))
    out = subprocess.run([_build(tmp_path)], capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode == 0, (out.returncode, out.stdout, out.stderr)
    assert "api_demo ok" in out.stdout
