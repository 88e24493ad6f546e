"""Pins the CPU oracle (oracle/csr5_oracle.c) before it is trusted.

1. Known-answer tests restated from the reference's own unit tests
   (proj/tests/test_format.cpp, test_descriptor.cpp, test_tuning.cpp,
   test_segmented_sum.cpp, test_spmv.cpp) -- file:line cited per test.
2. Golden fixtures produced by the unmodified reference (tests/golden/).
3. A randomized sweep against the compiled reference (oracle/_ref) when present.
"""
import numpy as np
import pytest

from oracle.oracle import Csr, OracleError


def small_matrix_with_empty_row(orc):
    # test_format.cpp:17-28: row_ptr = [0, 2, 2, 5, 8]
    return orc.coo_to_csr([0, 0, 2, 2, 2, 3, 3, 3], [0, 1, 0, 1, 2, 0, 1, 3],
                          [1, 2, 3, 4, 5, 6, 7, 8], 4, 4)


def eight_by_eight(orc):
    # test_format.cpp:30-44 / acceptance.cpp:158-166
    cols = [[0, 1, 2, 3, 4, 5], [], [0, 2, 4, 6, 7], [1, 3, 5, 6, 7], [0, 1, 2, 3, 4, 5, 6],
            [1, 2, 3, 5, 6, 7], [0, 3, 6], [2, 5]]
    rows, cc = [], []
    for r, c in enumerate(cols):
        rows += [r] * len(c)
        cc += c
    a = orc.coo_to_csr(rows, cc, np.arange(1, 35, dtype=float), 8, 8)
    assert a.nnz == 34 and a.row_ptr[4] == 16
    return a


def test_mt19937_64_known_answer(orc):
    # std::mt19937_64 default seed: the 10000th output is 9981545732273789042
    g = orc.rng(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042


def test_row_of_nonzero(orc):  # test_format.cpp:48-56
    rp = [0, 2, 2, 5, 8]
    assert [orc.row_of_nonzero(rp, g) for g in (0, 1, 2, 4, 5, 8)] == [0, 0, 2, 2, 3, 3]


def test_tile_ptr_small(orc):  # test_format.cpp:58-68
    a = small_matrix_with_empty_row(orc)
    A = orc.build(a, 2, 2)
    rows = [int(v) & 0x7FFFFFFF for v in A.tile_ptr]
    flags = [bool(int(v) >> 31) for v in A.tile_ptr]
    assert rows == [0, 2, 3] and flags[:2] == [True, False]


def test_tile_ptr_bits(orc):  # test_format.cpp:78-82
    assert orc.L.orc_tile_ptr_bits(100) == 32
    assert orc.L.orc_tile_ptr_bits((1 << 31) - 1) == 32
    assert orc.L.orc_tile_ptr_bits(1 << 31) == 64


def test_bit_flag(orc):  # test_format.cpp:84-102
    a = small_matrix_with_empty_row(orc)
    assert orc.bit_flag(a, 0, 2, 2).tolist() == [1, 0, 1, 0]
    one_row = orc.coo_to_csr([0] * 4, [0, 1, 2, 3], [1.0] * 4, 1, 4)
    assert orc.bit_flag(one_row, 0, 2, 2).tolist() == [1, 0, 0, 0]
    singletons = orc.coo_to_csr([0, 1, 2, 3], [0, 1, 2, 3], [1.0] * 4, 4, 4)
    assert orc.bit_flag(singletons, 0, 2, 2).tolist() == [1, 1, 1, 1]


def test_y_and_seg_offset(orc):  # test_format.cpp:104-131, acceptance.cpp:175-196
    bf = np.zeros(16, np.uint8)
    bf[[0, 1, 2, 9]] = 1
    y, s = orc.y_seg_offset(bf, 4, 4)
    assert y.tolist() == [0, 3, 3, 4] and s.tolist() == [1, 0, 1, 0]
    bf = np.zeros(16, np.uint8)
    bf[[0, 6, 13]] = 1
    assert orc.y_seg_offset(bf, 4, 4)[1].tolist() == [0, 1, 0, 0]
    bf = np.zeros(16, np.uint8)
    bf[[0, 5, 14]] = 1
    assert orc.y_seg_offset(bf, 4, 4)[1].tolist() == [0, 1, 0, 0]
    bf = np.zeros(16, np.uint8)
    bf[[0, 4, 8, 12]] = 1
    assert orc.y_seg_offset(bf, 4, 4)[1].tolist() == [0, 0, 0, 0]


def test_empty_offset(orc):  # test_format.cpp:133-141
    A = orc.build(small_matrix_with_empty_row(orc), 2, 2)
    assert A.eo[A.eo_ptr[0]:A.eo_ptr[1]].tolist() == [0, 2]


def test_transpose_and_roundtrip(orc):  # test_format.cpp:143-161, 185-204
    a = Csr(1, 4, np.array([0, 4], np.int64), np.arange(4, dtype=np.int64),
            np.array([1.0, 2.0, 3.0, 4.0]))
    A = orc.build(a, 2, 2)
    assert A.val.tolist() == [1.0, 3.0, 2.0, 4.0]
    g = orc.rng(23)
    for omega in (1, 2, 4, 8, 32):
        for sigma in (1, 2, 4, 12, 16):
            if omega * sigma < 2:
                continue
            for _ in range(4):
                m, n = 1 + g() % 40, 1 + g() % 40
                a = g.random_csr(m, n, g() % (m * n + 1))
                ci, va = orc.to_csr(a, omega, sigma)
                assert np.array_equal(ci, a.col_idx) and np.array_equal(va, a.val)


def test_eight_by_eight(orc):  # test_format.cpp:163-173
    A = orc.build(eight_by_eight(orc), 4, 4)
    assert (A.p, A.pc, A.tail_len) == (3, 2, 2)
    assert int(A.tile_ptr[1]) & 0x7FFFFFFF == 4
    assert int(A.tile_ptr[0]) >> 31 == 1 and int(A.tile_ptr[1]) >> 31 == 0


def test_exact_tile_multiple(orc):  # test_format.cpp:206-214
    a = orc.generate_synthetic(0, 8, 16, 64, 3)
    A = orc.build(a, 4, 4)
    assert (A.p, A.pc, A.tail_len) == (4, 4, 0)
    assert int(A.tile_ptr[4]) & 0x7FFFFFFF == 7


def test_empty_matrix(orc):  # test_format.cpp:175-183
    a = orc.coo_to_csr([], [], [], 5, 5)
    A = orc.build(a, 4, 16)
    assert A.p == 0 and A.pc == 0 and len(A.tile_desc) == 0 and len(A.col_idx) == 0


def test_invalid_shape_rejected(orc):  # test_format.cpp:229-232, test_tuning.cpp:31-38
    a = orc.coo_to_csr([0], [0], [1.0], 1, 1)
    with pytest.raises(OracleError, match="omega \\* sigma must be >= 2"):
        orc.build(a, 1, 1)
    with pytest.raises(OracleError):
        orc.validate(0, 16)
    with pytest.raises(OracleError):
        orc.validate(4, 16, r=10, s=5)
    with pytest.raises(OracleError):
        orc.validate(4, 16, u=0)
    orc.validate(1, 2)


def test_layout(orc):  # test_descriptor.cpp:26-58, acceptance.cpp:240-246
    assert [orc.ceil_log2(v) for v in (1, 2, 3, 32, 33, 512)] == [0, 1, 2, 5, 6, 9]
    assert orc.layout(32, 16) == (9, 5, 32)
    assert orc.layout(4, 40)[2] == 64
    with pytest.raises(OracleError, match="smaller sigma"):
        orc.layout(4, 60)
    # omega = 32: u32 words up to sigma = 17, u64 from 18, reject above 48
    assert orc.layout(32, 17)[2] == 32 and orc.layout(32, 18)[2] == 64
    assert orc.layout(32, 48)[2] == 64
    with pytest.raises(OracleError):
        orc.layout(32, 49)


def test_pack(orc):  # test_descriptor.cpp:60-98
    bf = np.zeros(8, np.uint8)
    bf[0] = 1
    assert orc.pack([0, 0], [0, 0], bf, 2, 4)[0] == 0x8
    assert not orc.pack([0] * 4, [0] * 4, np.zeros(16, np.uint8), 4, 4).any()
    with pytest.raises(OracleError):
        orc.pack([0, 0, 1 << 10, 0], [0] * 4, np.zeros(16, np.uint8), 4, 4)
    g = orc.rng(17)
    for omega in (1, 2, 4, 8, 32):
        for sigma in (2, 4, 12, 16):
            for _ in range(20):
                bf = np.array([1 if g() % 4 == 0 else 0 for _ in range(omega * sigma)], np.uint8)
                bf[0] = 1
                y, s = orc.y_seg_offset(bf, omega, sigma)
                y2, s2, bf2 = orc.unpack(orc.pack(y, s, bf, omega, sigma), omega, sigma)
                assert np.array_equal(y, y2) and np.array_equal(s, s2) and np.array_equal(bf, bf2)


def test_select_sigma(orc):  # test_tuning.cpp:16-25, acceptance.cpp:269-275
    assert [orc.select_sigma(v) for v in (2.0, 10.0, 100.0, 1000.0)] == [4, 10, 32, 4]
    assert [orc.select_sigma(v) for v in (4.0, 32.0, 256.0)] == [4, 32, 32]


def test_segmented_sums(orc):  # test_segmented_sum.cpp:28-150, acceptance.cpp:200-238
    assert orc.serial_segsum([1, 2, 3, 4], [1, 0, 1, 0]).tolist() == [3, 0, 7, 0]
    assert orc.serial_segsum([1, 2], [0, 0]).tolist() == [0, 0]
    out = orc.fast_segsum([1, 2, 3, 4], [0, 1, 0, 0])
    assert out[0] == 1.0 and out[1] == 5.0
    assert orc.fast_segsum([3.0, 4.0], [1, 0])[0] == 7.0
    with pytest.raises(OracleError):
        orc.fast_segsum([1, 2], [2, 0])
    g = orc.rng(5)
    for _ in range(200):
        n = 1 + g() % 64
        data = [float((g() % (1 << 34)) - (1 << 33)) for _ in range(n)]
        heads = [1 if g() % 4 == 0 else 0 for _ in range(n)]
        off = []
        for i in range(n):
            j = i + 1
            while j < n and not heads[j]:
                j += 1
            off.append(j - i - 1 if heads[i] else 0)
        f = orc.fast_segsum(data, off)
        s = orc.serial_segsum(data, heads)
        assert all(f[i] == s[i] for i in range(n) if heads[i])


def test_tile_contributions(orc):  # test_spmv.cpp:78-143
    a = orc.coo_to_csr([0] * 8, list(range(8)), [float(c + 1) for c in range(8)], 1, 8)
    rows, vals, acc = orc.tile_contrib(a, 4, 2, 0, np.ones(8))
    assert rows.tolist() == [0] and acc.tolist() == [True] and vals[0] == 36.0
    a = orc.coo_to_csr(list(range(8)), [0] * 8, [float(i + 1) for i in range(8)], 8, 1)
    rows, vals, acc = orc.tile_contrib(a, 4, 2, 0, np.ones(1))
    assert len(rows) == 8
    by = {}
    for r, v in zip(rows, vals):
        by[int(r)] = by.get(int(r), 0.0) + v
    assert by == {i: float(i + 1) for i in range(8)}


def test_spmv_matches_dense_oracle(orc):  # test_spmv.cpp:153-171, acceptance.cpp:106-151
    g = orc.rng(53)
    for omega in (1, 2, 4, 8, 32):
        for sigma in (1, 2, 4, 12, 16):
            if omega * sigma < 2:
                continue
            for _ in range(3):
                m, n = 1 + g() % 50, 1 + g() % 50
                a = g.random_csr(m, n, g() % 500)
                x = g.random_x(n)
                y = orc.spmv(a, x, omega, sigma)
                ref = orc.dense_spmv(a, x)
                err = np.abs(y - ref) / np.maximum(1.0, np.abs(ref))
                assert err.max(initial=0) <= 1e-12


def test_golden_w32(orc, golden):
    """Every golden case: oracle arrays bit-exact and y bit-exact vs reference."""
    z, meta = golden
    for c in meta:
        k, mk = c["key"], c["mat"]
        a = Csr(c["m"], c["n"], z[f"{mk}_row_ptr"], z[f"{mk}_col_idx"].astype(np.int64), z[f"{mk}_val"])
        A = orc.build(a, 32, c["sigma"])
        assert (A.p, A.pc, A.tail_len, A.word_bits) == (c["p"], c["pc"], c["tail"], c["word_bits"])
        assert np.array_equal(A.tile_ptr, z[f"{k}_tile_ptr"]), c
        assert np.array_equal(A.tile_desc, z[f"{k}_tile_desc"]), c
        assert np.array_equal(A.eo_ptr, z[f"{k}_eo_ptr"]), c
        assert np.array_equal(A.eo, z[f"{k}_eo"]), c
        assert np.array_equal(A.col_idx, z[f"{k}_tcol"].astype(np.int64)), c
        y = orc.spmv(a, z[f"{mk}_x"], 32, c["sigma"])
        assert np.array_equal(y, z[f"{k}_y"]), c


def test_golden_edges(orc, edges):
    for d in edges:
        rp = np.array(d["row_ptr"], np.int64)
        nnz = int(rp[-1])
        cols = d.get("col_idx")
        if cols is None:
            cols = []
            for i in range(len(rp) - 1):
                cols += list(range(int(rp[i + 1] - rp[i])))
        a = Csr(len(rp) - 1, max(max(cols, default=0) + 1, nnz, 1), rp, np.array(cols, np.int64),
                np.arange(1, nnz + 1, dtype=float))
        A = orc.build(a, d["omega"], d["sigma"])
        assert [int(v) for v in A.tile_ptr] == d["tile_ptr"], d["name"]
        assert [int(v) for v in A.tile_desc] == d["tile_desc"], d["name"]
        assert A.eo.tolist() == d["eo"], d["name"]


def test_generators_match_reference(orc, ref):
    for kind in (0, 1, 2):
        for seed in (1, 42, 77):
            a = orc.generate_synthetic(kind, 60, 80, 700, seed, 0.1)
            b = ref.generate_synthetic(kind, 60, 80, 700, seed, 0.1)
            assert np.array_equal(a.row_ptr, b.row_ptr)
            assert np.array_equal(a.col_idx, b.col_idx)
            assert np.array_equal(a.val, b.val)


def test_oracle_vs_reference_sweep(orc, ref):
    """acceptance.cpp:53-104-style corpus at omega 32 and the CPU shapes."""
    g = orc.rng(7)
    for case in range(40):
        m, n = 1 + g() % 200, 1 + g() % 200
        kind = case % 3
        nnz = min(m * n, g() % 5000)
        try:
            a = orc.generate_synthetic(kind, m, n, nnz, g(), 0.3)
        except OracleError:
            a = g.random_csr(m, n, nnz)
        x = g.random_x(n)
        for omega, sigma in ((32, 1 + g() % 48), (4, 16), (8, 12), (2, 1)):
            A, B = orc.build(a, omega, sigma), ref.build(a, omega, sigma)
            for f in ("tile_ptr", "tile_desc", "eo_ptr", "eo", "col_idx", "val"):
                assert np.array_equal(getattr(A, f), getattr(B, f)), (case, omega, sigma, f)
            assert np.array_equal(orc.spmv(a, x, omega, sigma), ref.spmv(a, x, omega, sigma))
