"""run_benchmark harness API (paper_1503_05032_b200.benchmark) against the
reference's own bench.cpp, called through oracle/_ref (the unmodified
reference library): kernel-list parsing, the iteration-scenario formula and
its errors, and the CSV text byte for byte.  The timing path itself needs a
GPU (tests/test_gpu_benchmark.py)."""
import ctypes as C
import math
import random

import pytest

from oracle.oracle import have_ref
from paper_1503_05032_b200 import benchmark as B

pytestmark = pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Ref
    L = Ref().L
    L.ref_parse_kernels.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.c_int]
    L.ref_parse_kernels.restype = C.c_int
    L.ref_iteration_speedup.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int64,
                                        C.POINTER(C.c_double)]
    L.ref_iteration_speedup.restype = C.c_int
    d = C.POINTER(C.c_double)
    L.ref_emit_csv.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int,
                               C.c_char_p, d, d, d, d, d, d, C.c_char_p, C.c_int64]
    L.ref_emit_csv.restype = C.c_int64
    L.ref_last_error.restype = C.c_char_p
    return L


KINDS = [B.KernelKind.csr_scalar, B.KernelKind.csr_segsum, B.KernelKind.csr5]


@pytest.mark.parametrize("text", ["csr5", "csr-scalar,csr5", "csr5,", "csr-segsum,csr-scalar,csr5",
                                  "", ",", "csr5,,csr5", "csr6", "CSR5", "csr5,csr5", " csr5"])
def test_parse_kernel_list(ref, text):
    out = (C.c_int * 8)()
    n = ref.ref_parse_kernels(text.encode(), out, 8)
    if n < 0:
        with pytest.raises(ValueError) as e:
            B.parse_kernel_list(text)
        assert str(e.value) == ref.ref_last_error().decode()
    else:
        assert B.parse_kernel_list(text) == [KINDS[out[i]] for i in range(n)]


def test_iteration_speedup(ref):
    rng = random.Random(3)
    cases = [(1.0, 0.0, 0.5, 50), (2.0, 30.0, 0.25, 500), (1.0, -1.0, 1.0, 5), (0.0, 1.0, 1.0, 5),
             (1.0, 1.0, 0.0, 5), (1.0, 1.0, 1.0, 0), (3.5, 1e-9, 7.25, 1)]
    cases += [(rng.uniform(1e-3, 10), rng.uniform(0, 100), rng.uniform(1e-3, 10),
               rng.choice([1, 50, 500, 10**6])) for _ in range(200)]
    for t_csr, t_pre, t_new, n in cases:
        out = C.c_double()
        rc = ref.ref_iteration_speedup(t_csr, t_pre, t_new, n, C.byref(out))
        if rc:
            with pytest.raises(ValueError) as e:
                B.iteration_speedup(t_csr, t_pre, t_new, n)
            assert str(e.value) == ref.ref_last_error().decode()
        else:
            assert B.iteration_speedup(t_csr, t_pre, t_new, n) == out.value


def _ref_csv(ref, rep: B.BenchReport) -> str:
    k = rep.kernels
    arr = lambda f: (C.c_double * max(1, len(k)))(*[getattr(x, f) for x in k])  # noqa: E731
    buf = C.create_string_buffer(1 << 16)
    n = ref.ref_emit_csv(rep.matrix.encode(), rep.m, rep.n, rep.nnz, rep.threads, len(k),
                         "\n".join(x.kernel for x in k).encode(), arr("best_ms"), arr("avg_ms"),
                         arr("gflops"), arr("conv_ms"), arr("speedup_n50"), arr("speedup_n500"),
                         buf, len(buf))
    return buf.raw[:n].decode()


def test_emit_csv_matches_reference(ref, tmp_path):
    rng = random.Random(7)
    special = [0.0, 1.0, 0.1, 1e-5, 1.5e-4, 123456789.0, 1234567890123.0, 9.999999999e9,
               1e10, 2.0 ** -30, 1 / 3, 2 / 3, 0.00001234567891234, 5e-324, 1.7976931348623157e308,
               float("inf"), -2.5, 1e16, 12345.678901234]
    for trial in range(60):
        kernels = []
        for name in ("csr-scalar", "csr-segsum", "csr5")[:1 + trial % 3]:
            vals = [rng.choice(special) if rng.random() < 0.4 else
                    10 ** rng.uniform(-8, 12) * rng.choice([1, -1]) for _ in range(6)]
            kernels.append(B.KernelResult(name, [], *vals))
        rep = B.BenchReport(f"mat{trial}", rng.randrange(1 << 40), rng.randrange(1 << 40),
                            rng.randrange(1 << 50), rng.randrange(1, 512), kernels)
        assert B.emit_csv(rep) == _ref_csv(ref, rep)
    p = tmp_path / "r.csv"
    assert B.emit_csv(rep, str(p)) == p.read_text()
    assert p.read_text().splitlines()[0] == B.CSV_HEADER
    with pytest.raises(RuntimeError, match="emit_csv: cannot open"):
        B.emit_csv(rep, str(tmp_path / "missing" / "r.csv"))
    assert not math.isnan(B.relative_error(1.0, 0.0))
