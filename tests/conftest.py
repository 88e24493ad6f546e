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
