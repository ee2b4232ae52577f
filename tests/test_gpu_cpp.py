"""Compiles and runs the C++ mirror tests (tests/cpp/test_wrapper.cpp,
tests/cpp/test_search_api.cpp) against the in-tree libcmgpu.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = ["test_wrapper", "test_search_api"]


def _build(name):
    pkg = os.path.join(ROOT, "paper_2502_11602_b200")
    out = os.path.join(ROOT, "build", name)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-L", pkg, "-lcmgpu",
                    f"-Wl,-rpath,{pkg}", "-o", out], check=True)
    return out


@pytest.mark.parametrize("name", TESTS)
def test_cpp_mirror_compiles(name):
    assert os.path.exists(_build(name))


@pytest.mark.gpu
@pytest.mark.parametrize("name", TESTS)
def test_cpp_mirror_runs(name):
    r = subprocess.run([_build(name)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "ok" in r.stdout
