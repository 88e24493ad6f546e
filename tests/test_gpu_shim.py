"""Runs the C++ drop-in shim test (tests/cpp/shim_test.cpp over include/csr5g.hpp)."""
import os
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
BIN = os.path.join(ROOT, "build", "shim_test")


@pytest.mark.gpu
def test_cpp_shim():
    subprocess.run(["make", "-C", ROOT, "shim"], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "SHIM OK" in r.stdout, r.stdout + r.stderr
