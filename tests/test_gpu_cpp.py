"""Compiles and runs the C++ wrapper test (tests/cpp/test_wrapper.cpp)
against the in-tree libcmgpu.so."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build():
    pkg = os.path.join(ROOT, "paper_2502_11602_b200")
    out = os.path.join(ROOT, "build", "test_wrapper")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_wrapper.cpp"), "-L", pkg, "-lcmgpu",
                    f"-Wl,-rpath,{pkg}", "-o", out], check=True)
    return out


def test_cpp_wrapper_compiles():
    assert os.path.exists(_build())


@pytest.mark.gpu
def test_cpp_wrapper_runs():
    r = subprocess.run([_build()], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "cpp wrapper ok" in r.stdout
