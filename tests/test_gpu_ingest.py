"""Device COO -> CSR (csr5g_coo_to_csr) against the reference's coo_to_csr
(oracle/_ref): bit-identical row_ptr, col_idx and summed values, including
duplicate runs whose sums depend on the addition order, and the reference's
error text for out-of-range entries.  Then the file path end to end:
load_matrix_market -> csr_to_csr5 -> SpMV against the oracle."""
import ctypes as C
import random

import numpy as np
import pytest

from oracle.oracle import Csr, have_ref
from tests._util import assert_y_close

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_ref(), reason="oracle/_ref")]


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_1503_05032_b200 import csr5
    return csr5


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Ref
    R = Ref()
    L = R.L
    L.ref_coo_to_csr.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.POINTER(C.c_void_p)]
    L.ref_coo_to_csr.restype = C.c_int
    L.ref_csr_nnz.restype = C.c_int64
    L.ref_csr_nnz.argtypes = [C.c_void_p]
    L.ref_csr_get.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ref_csr_free.argtypes = [C.c_void_p]
    L.ref_last_error.restype = C.c_char_p
    return L


def ref_coo(L, rows, cols, vals, m, n):
    h = C.c_void_p()
    rc = L.ref_coo_to_csr(m, n, len(rows), rows.ctypes.data, cols.ctypes.data, vals.ctypes.data,
                          C.byref(h))
    if rc:
        return rc, L.ref_last_error().decode()
    nz = L.ref_csr_nnz(h)
    rp, ci, va = np.empty(m + 1, np.int64), np.empty(nz, np.int64), np.empty(nz)
    L.ref_csr_get(h, rp.ctypes.data, ci.ctypes.data, va.ctypes.data)
    L.ref_csr_free(h)
    return 0, (rp, ci, va)


def test_coo_to_csr_bit_exact(g, ref):
    rng = np.random.default_rng(5)
    for trial in range(40):
        m, n = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
        k = int(rng.integers(0, 20000))
        if trial % 4 == 0:  # heavy duplication: few distinct keys
            rows = rng.integers(0, min(m, 20), k)
            cols = rng.integers(0, min(n, 20), k)
        else:
            rows, cols = rng.integers(0, m, k), rng.integers(0, n, k)
        vals = rng.standard_normal(k) * 10.0 ** rng.integers(-8, 8, k)
        exp = ref_coo(ref, rows, cols, vals, m, n)
        a = g.coo_to_csr(rows, cols, vals, m, n)
        assert exp[0] == 0
        rp, ci, va = exp[1]
        assert np.array_equal(a.row_ptr.cpu().numpy(), rp), trial
        assert np.array_equal(a.col_idx.cpu().numpy().astype(np.int64), ci), trial
        assert np.array_equal(a.val.cpu().numpy(), va), trial  # bitwise: same summation order
    # high row and column bits of the (row << 31 | col) sort key
    a = g.coo_to_csr(np.array([5, 2**25 - 1, 5]), np.array([2**31 - 2, 1, 2**31 - 2]),
                     np.array([1.0, 2.0, 3.0]), 2**25, 2**31 - 1)
    assert a.nnz == 2 and a.val.cpu().tolist() == [4.0, 2.0]
    assert a.col_idx.cpu().tolist() == [2**31 - 2, 1]


def test_coo_to_csr_errors(g, ref):
    for rows, cols, m, n in (([0, 3, 5], [0, 0, 9], 4, 4), ([0, -1], [0, 0], 2, 2),
                             ([1], [2], 2, 2), ([0], [0], 0, 0)):
        rows, cols = np.array(rows, np.int64), np.array(cols, np.int64)
        vals = np.ones(len(rows))
        exp = ref_coo(ref, rows, cols, vals, m, n)
        assert exp[0] == 1
        with pytest.raises(ValueError) as e:
            g.coo_to_csr(rows, cols, vals, m, n)
        assert str(e.value) == exp[1]
    a = g.coo_to_csr(np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0), 3, 3)
    assert a.nnz == 0 and a.row_ptr.cpu().tolist() == [0, 0, 0, 0]


def test_matrix_market_end_to_end(g, orc, tmp_path):
    rng = random.Random(3)
    m = n = 900
    ent = {}
    for _ in range(12000):
        r = rng.randint(1, m)
        c = rng.randint(1, r)
        ent.setdefault((r, c), []).append(rng.uniform(-2, 2))
    lines = ["%%MatrixMarket matrix coordinate real symmetric", "% test", f"{m} {n} "
             f"{sum(len(v) for v in ent.values())}"]
    for (r, c), vs in ent.items():
        lines += [f"{r} {c} {v:.17g}" for v in vs]
    p = tmp_path / "s.mtx"
    p.write_text("\n".join(lines) + "\n")
    a = g.load_matrix_market(str(p))
    host = Csr(a.m, a.n, a.row_ptr.cpu().numpy(), a.col_idx.cpu().numpy().astype(np.int64),
               a.val.cpu().numpy())
    sigma = orc.select_sigma(host.nnz / host.m)
    a5 = g.csr_to_csr5(a, g.TuningParams(sigma=sigma))
    x = orc.rng(2).random_x(n)
    y = g.spmv_csr5(a5, torch.as_tensor(x).cuda()).cpu().numpy()
    assert_y_close(y, orc.spmv(host, x, 32, sigma), host, x, "mtx")
    A = np.zeros((m, n))
    for (r, c), vs in ent.items():
        s = 0.0
        for v in vs:
            s += v
        A[r - 1, c - 1] = s
        A[c - 1, r - 1] = s
    dense = np.zeros((m, n))
    for r in range(m):
        dense[r, host.col_idx[host.row_ptr[r]:host.row_ptr[r + 1]]] = \
            host.val[host.row_ptr[r]:host.row_ptr[r + 1]]
    assert np.array_equal(dense, A)
