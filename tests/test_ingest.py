"""Matrix Market reader (csr5g_mm_read, host code of libcsr5g) against the
reference's own read_matrix_market (oracle/_ref) on generated files: the same
entries in the same order for every valid file, the same exception text for
every malformed one.  Runs without a GPU."""
import ctypes as C
import random

import numpy as np
import pytest

from oracle.oracle import have_ref

pytestmark = pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Ref
    L = Ref().L
    p64 = C.POINTER(C.c_int64)
    L.ref_mm_read.argtypes = [C.c_char_p, p64, p64, p64, C.POINTER(C.c_void_p)]
    L.ref_mm_read.restype = C.c_int
    L.ref_mm_get.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ref_mm_free.argtypes = [C.c_void_p]
    L.ref_last_error.restype = C.c_char_p
    return L


def ref_read(L, path):
    m, n, k, h = C.c_int64(), C.c_int64(), C.c_int64(), C.c_void_p()
    rc = L.ref_mm_read(str(path).encode(), C.byref(m), C.byref(n), C.byref(k), C.byref(h))
    if rc:
        return rc, L.ref_last_error().decode()
    rows, cols = np.empty(k.value, np.int64), np.empty(k.value, np.int64)
    vals = np.empty(k.value)
    L.ref_mm_get(h, rows.ctypes.data, cols.ctypes.data, vals.ctypes.data)
    L.ref_mm_free(h)
    return 0, (m.value, n.value, rows, cols, vals)


def ours(path):
    from paper_1503_05032_b200 import csr5
    try:
        return 0, csr5.read_matrix_market(str(path))
    except RuntimeError as e:
        return 2, str(e)


def same(a, b):
    assert a[0] == b[0], (a, b)
    if a[0]:
        assert a[1] == b[1]
    else:
        for u, v in zip(a[1], b[1]):
            assert np.array_equal(u, v) if isinstance(u, np.ndarray) else u == v


def _value(rng, field):
    if field == "integer":
        return str(rng.randint(-50, 50))
    return rng.choice([f"{rng.uniform(-5, 5):.17g}", f"{rng.uniform(-5, 5):e}", "1", "-0.5",
                       ".5", "5.", "+3.25", "1e-300", "2E+10"])


def valid_file(rng):
    field = rng.choice(["real", "integer", "pattern"])
    sym = rng.choice(["general", "symmetric"])
    banner = rng.choice(["%%MatrixMarket", "%%matrixmarket", "%%MATRIXMARKET"])
    m = rng.randint(1, 40)
    n = m if sym == "symmetric" else rng.randint(1, 40)
    k = rng.randint(0, 60)
    nl = rng.choice(["\n", "\r\n"])
    lines = [f"{banner} {rng.choice(['matrix', 'MATRIX'])} {rng.choice(['coordinate', 'Coordinate'])}"
             f" {field} {sym}"]
    lines += ["% a comment", "", "   ", "\t% indented comment"][:rng.randint(0, 4)]
    lines.append(f"{m} {n} {k}")
    for _ in range(k):
        r = rng.randint(1, m)
        c = rng.randint(1, r) if sym == "symmetric" else rng.randint(1, n)
        sep = rng.choice([" ", "  ", "\t"])
        e = f"{r}{sep}{c}" + ("" if field == "pattern" else f"{sep}{_value(rng, field)}")
        if rng.random() < 0.1:
            e += " trailing"
        lines.append(e)
        if rng.random() < 0.1:
            lines.append("% interleaved comment")
    return nl.join(lines) + rng.choice([nl, ""])


BAD = [
    "",
    "%%MatrixMarket matrix coordinate real\n2 2 1\n1 1 1.0\n",
    "%%NotMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n",
    "%%MatrixMarket vector coordinate real general\n2 2 1\n1 1 1.0\n",
    "%%MatrixMarket matrix array real general\n2 2\n1.0\n",
    "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1.0 0.0\n",
    "%%MatrixMarket matrix coordinate double general\n2 2 1\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real hermitian\n2 2 1\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "%%MatrixMarket matrix coordinate real general\n2 2\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 -2 1\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\nx 2 1\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 2.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 abc\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 inf\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1.5 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n\n% c\n1 3 1.0\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1\n",
    "%%MatrixMarket matrix coordinate integer symmetric\n3 3 2\n1 1 4\n3 2 -1\n",
    "%%MatrixMarket matrix coordinate real general\r\n2 2 1\r\n2 2 7.5\r\n",
    "%%MatrixMarket matrix coordinate real general\n0 0 0\n",
]


def test_reader_matches_reference(ref, tmp_path):
    rng = random.Random(12)
    files = [valid_file(rng) for _ in range(150)] + BAD
    for i, text in enumerate(files):
        p = tmp_path / f"m{i}.mtx"
        p.write_bytes(text.encode())
        same(ours(p), ref_read(ref, p))
    missing = tmp_path / "nope.mtx"
    same(ours(missing), ref_read(ref, missing))
