"""CPU checks of the drop-in boundary: libcsr5g.so loads and exports every
symbol include/csr5g.h declares; host-only entry points behave like the
reference (no compute calls -- there is no GPU here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "csr5g.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"CSR5G_API\s+[\w\s\*]*?\b(csr5g_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for must in ("csr5g_build", "csr5g_spmv", "csr5g_release", "csr5g_export",
                 "csr5g_build_shard", "csr5g_fixup", "csr5g_to_csr"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_1503_05032_b200 import _lib
    L = _lib.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_host_entry_points(orc):
    from paper_1503_05032_b200 import csr5
    for npr in (0.5, 2.0, 4.0, 4.4, 4.6, 10.0, 31.5, 32.0, 33.0, 100.0, 256.0, 257.0, 1000.0):
        assert csr5.select_sigma(npr) == orc.select_sigma(npr)
    for sigma in range(1, 49):
        assert csr5.layout(32, sigma) == orc.layout(32, sigma)
    with pytest.raises(ValueError, match="smaller sigma"):
        csr5.layout(32, 49)
    with pytest.raises(ValueError, match="r <= s <= t"):
        csr5.select_sigma(3.0, r=10, s=5)


def test_no_cpu_fallback_without_gpu():
    """Every compute entry point must fail loudly when no device is usable."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1503_05032_b200 import _lib
    L = _lib.lib()
    h = C.c_void_p()
    p = _lib.Params(32, 4, 4, 32, 256, 4)
    rc = L.csr5g_build(0, 0, 0, 0, None, None, None, C.byref(p), None, C.byref(h))
    assert rc == _lib.ECUDA
    assert "CUDA" in L.csr5g_last_error().decode() or "device" in L.csr5g_last_error().decode()
    # the multi-GPU exchange: argument errors first (reference-style EINVAL),
    # then no device -> ECUDA, never a host stand-in
    mb = C.c_void_p()
    assert L.csr5g_mailbox_create(0, 0, 0, 0, C.byref(mb)) == _lib.EINVAL
    assert L.csr5g_mailbox_create(0, 2, 2, 0, C.byref(mb)) == _lib.EINVAL
    assert L.csr5g_mailbox_create(0, 2, 0, -1, C.byref(mb)) == _lib.EINVAL
    assert L.csr5g_mailbox_create(0, 2, 0, 16, C.byref(mb)) == _lib.ECUDA
    assert L.csr5g_mg_spmv(None, None, None, None, None, None) == _lib.EINVAL
    assert L.csr5g_mg_iter(None, 0, None, None, None) == _lib.EINVAL


def test_stencil_box_sizes_and_weak_scaling():
    """csr5g_stencil_box_size (host-only) against the oracle's formula and the
    host generator; the weak-scaling workload rule of bench.py."""
    import ctypes as C

    from oracle.oracle import Oracle, stencil, stencil_box_size
    from paper_1503_05032_b200 import _lib
    from paper_1503_05032_b200.synthetic import WORKLOADS, scaled_workload
    L = _lib.lib()
    orc = Oracle()
    for kind in (0, 1):
        for a in (1, 2, 3, 7):
            for layers in (1, 2, a, 3 * a):
                m, nnz = C.c_int64(), C.c_int64()
                assert L.csr5g_stencil_box_size(kind, a, layers, C.byref(m), C.byref(nnz)) == 0
                assert (m.value, nnz.value) == stencil_box_size(kind, a, layers)
                if m.value <= 2000:
                    h = stencil(orc, kind, a, layers)
                    assert (h.m, h.row_ptr[-1]) == (m.value, nnz.value)
    w = scaled_workload(WORKLOADS["st27_200"], 8)
    assert (w["a"], w["layers"]) == (200, 1600)
    assert scaled_workload(WORKLOADS["rmat24"], 8)["scale"] == 27  # BASELINE config 5
    assert scaled_workload(WORKLOADS["mixed23"], 4)["log2_m"] == 25
    with pytest.raises(ValueError, match="power-of-two"):
        scaled_workload(WORKLOADS["rmat24"], 3)


def test_bench_x_matches_the_reference_engine(orc):
    """bench.cpp:103-105 x: the native generator (csr5g_bench_x, host code),
    the numpy restatement and the oracle's mt19937_64 agree bit for bit."""
    import numpy as np

    from paper_1503_05032_b200.synthetic import bench_x, bench_x_numpy, mt19937_64
    assert int(mt19937_64(5489, 10000)[-1]) == 9981545732273789042  # std KAT
    for n in (0, 1, 311, 312, 313, 5000):
        a, b = bench_x(n), bench_x_numpy(n)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert np.array_equal(bench_x(4000, seed=1), orc.rng(1).random_x(4000))
