"""Shared test plumbing.

`-m "not gpu"` tests run in the build container (no GPU): the oracle against
the reference's golden vectors, host logic, the C-ABI symbol table, and the
multi-rank host logic over gloo.  `-m gpu` tests call the CUDA product through
its C ABI and compare with the oracle on the same inputs.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _ensure_oracle():
    lib = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"], check=True)


@pytest.fixture(scope="session")
def orc():
    _ensure_oracle()
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Ref, have_ref
    if not have_ref():
        pytest.skip("oracle/_ref/libcsr5ref.so not built (reference sources absent)")
    return Ref()


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    z = np.load(os.path.join(ROOT, "tests", "golden", "ref_w32.npz"))
    meta = json.loads(str(z["meta"]))
    return z, meta


@pytest.fixture(scope="session")
def edges():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "ref_edges.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cpp_build(tmp_path_factory):
    """The C++ drop-in test programs (tests/cpp) configured through
    find_package(csr5) and built; returns the build directory."""
    import shutil
    if not shutil.which("cmake"):
        pytest.skip("cmake not on PATH")
    if not os.path.exists(os.path.join(ROOT, "paper_1503_05032_b200", "libcsr5g.so")):
        subprocess.run(["make", "-C", ROOT, "lib"], check=True)
    bdir = str(tmp_path_factory.mktemp("csr5pkg") / "cpp")
    gen = ["-G", "Ninja"] if shutil.which("ninja") else []
    subprocess.run(["cmake", "-S", os.path.join(ROOT, "tests", "cpp"), "-B", bdir,
                    f"-Dcsr5_DIR={os.path.join(ROOT, 'cmake')}", *gen],
                   check=True, capture_output=True, text=True)
    r = subprocess.run(["cmake", "--build", bdir, "-j", "4"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    return bdir
