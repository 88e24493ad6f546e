"""ctypes front-end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two checkers live behind this module:

* ``Oracle``: the C restatement in ``oracle/csr5_oracle.c`` (+ ``testgen.c``),
  built into ``oracle/liboracle.so``.
* ``Ref``: the unmodified reference library (``/root/reference/proj/core/src``)
  compiled by ``oracle/Makefile`` into ``oracle/_ref/libcsr5ref.so``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and only
to check or time the CPU side.  The product (``paper_1503_05032_b200``) never
imports it.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libcsr5ref.so")

_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


@dataclass
class Csr:
    """Canonical CSR on the host (csr.hpp:25-35), int64 indices."""

    m: int
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if len(self.row_ptr) else 0


@dataclass
class Csr5Arrays:
    """Every array of a Csr5Matrix (format.hpp:130-176), widened to 64 bit."""

    m: int
    n: int
    nnz: int
    omega: int
    sigma: int
    p: int
    pc: int
    tail_len: int
    tile_ptr_bits: int
    word_bits: int
    y_bits: int
    seg_bits: int
    tile_ptr: np.ndarray  # uint64 [p+1]
    tile_desc: np.ndarray  # uint64 [pc*omega]
    eo_ptr: np.ndarray  # int64 [pc+1]
    eo: np.ndarray  # int64
    col_idx: np.ndarray  # int64 [nnz] transposed
    val: np.ndarray  # float64 [nnz] transposed


class _OrcCsr5(C.Structure):
    _fields_ = [
        ("m", C.c_int64), ("n", C.c_int64), ("nnz", C.c_int64),
        ("omega", C.c_int64), ("sigma", C.c_int64),
        ("p", C.c_int64), ("pc", C.c_int64), ("tail_len", C.c_int64),
        ("tile_ptr_bits", C.c_int), ("y_bits", C.c_int), ("seg_bits", C.c_int),
        ("word_bits", C.c_int),
        ("tile_ptr", _u64p), ("tile_desc", _u64p), ("eo_ptr", _i64p), ("eo", _i64p),
        ("row_ptr", _i64p), ("col_idx", _i64p), ("val", _f64p),
    ]


class _OrcCsr(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", _i64p), ("col_idx", _i64p), ("val", _f64p)]


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _copy(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


class Oracle:
    """The C restatement (csr5_oracle.c)."""

    def __init__(self, path: str = LIB_ORACLE):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = C.CDLL(path)
        self.L = L
        L.orc_build.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _f64p] + [C.c_int64] * 6 + [
            C.POINTER(_OrcCsr5), C.c_char_p, C.c_size_t]
        L.orc_free.argtypes = [C.POINTER(_OrcCsr5)]
        L.orc_spmv.argtypes = [C.POINTER(_OrcCsr5), _f64p, _f64p]
        L.orc_tile_contrib.argtypes = [C.POINTER(_OrcCsr5), C.c_int64, _f64p, _i64p, _f64p, _u8p,
                                       C.c_int64]
        L.orc_tile_contrib.restype = C.c_int64
        L.orc_dense_spmv.argtypes = [C.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.orc_csr5_to_csr.argtypes = [C.POINTER(_OrcCsr5), _i64p, _f64p]
        L.orc_row_of_nonzero.argtypes = [_i64p, C.c_int64, C.c_int64]
        L.orc_row_of_nonzero.restype = C.c_int64
        L.orc_select_sigma.argtypes = [C.c_double] + [C.c_int64] * 4 + [_i64p, C.c_char_p, C.c_size_t]
        L.orc_layout.argtypes = [C.c_int64, C.c_int64, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                 C.POINTER(C.c_int), C.c_char_p, C.c_size_t]
        L.orc_ceil_log2.argtypes = [C.c_int64]
        L.orc_validate_params.argtypes = [C.c_int64] * 6 + [C.c_char_p, C.c_size_t]
        L.orc_pack_desc.argtypes = [_i64p, _i64p, _u8p, C.c_int64, C.c_int64, C.c_int, C.c_int, _u64p]
        L.orc_unpack_desc.argtypes = [_u64p, C.c_int64, C.c_int64, C.c_int, C.c_int, _i64p, _i64p, _u8p]
        L.orc_bit_flag.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _u8p]
        L.orc_y_seg_offset.argtypes = [_u8p, C.c_int64, C.c_int64, _i64p, _i64p]
        L.orc_serial_segsum.argtypes = [_f64p, _u8p, C.c_int64]
        L.orc_fast_segsum.argtypes = [_f64p, _i64p, C.c_int64]
        L.orc_tile_ptr_bits.argtypes = [C.c_int64]
        # generators
        L.orc_mt64_new.argtypes = [C.c_uint64]
        L.orc_mt64_new.restype = C.c_void_p
        L.orc_mt64_delete.argtypes = [C.c_void_p]
        L.orc_mt64_next.argtypes = [C.c_void_p]
        L.orc_mt64_next.restype = C.c_uint64
        L.orc_random_csr.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.POINTER(_OrcCsr)]
        L.orc_random_x.argtypes = [C.c_void_p, C.c_int64, _f64p]
        L.orc_coo_to_csr.argtypes = [_i64p, _i64p, _f64p, C.c_int64, C.c_int64, C.c_int64,
                                     C.POINTER(_OrcCsr)]
        L.orc_generate_synthetic.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                             C.c_double, C.POINTER(_OrcCsr)]
        L.orc_csr_free.argtypes = [C.POINTER(_OrcCsr)]

    # -- scalar helpers -------------------------------------------------
    def select_sigma(self, npr: float, r=4, s=32, t=256, u=4) -> int:
        out = C.c_int64()
        err = C.create_string_buffer(256)
        rc = self.L.orc_select_sigma(npr, r, s, t, u, C.byref(out), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return out.value

    def layout(self, omega: int, sigma: int):
        yb, sb, wb = C.c_int(), C.c_int(), C.c_int()
        err = C.create_string_buffer(256)
        rc = self.L.orc_layout(omega, sigma, C.byref(yb), C.byref(sb), C.byref(wb), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        return yb.value, sb.value, wb.value

    def validate(self, omega, sigma, r=4, s=32, t=256, u=4):
        err = C.create_string_buffer(256)
        rc = self.L.orc_validate_params(omega, sigma, r, s, t, u, err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())

    def ceil_log2(self, v: int) -> int:
        return self.L.orc_ceil_log2(v)

    def row_of_nonzero(self, row_ptr, g: int) -> int:
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        return self.L.orc_row_of_nonzero(_p(rp, _i64p), len(rp) - 1, g)

    def bit_flag(self, a: Csr, tid: int, omega: int, sigma: int) -> np.ndarray:
        bf = np.zeros(omega * sigma, dtype=np.uint8)
        self.L.orc_bit_flag(_p(a.row_ptr, _i64p), a.m, tid, omega, sigma, _p(bf, _u8p))
        return bf

    def y_seg_offset(self, bf, omega, sigma):
        bf = np.ascontiguousarray(bf, dtype=np.uint8)
        y = np.zeros(omega, dtype=np.int64)
        s = np.zeros(omega, dtype=np.int64)
        self.L.orc_y_seg_offset(_p(bf, _u8p), omega, sigma, _p(y, _i64p), _p(s, _i64p))
        return y, s

    def pack(self, y, seg, bf, omega, sigma):
        yb, sb, _ = self.layout(omega, sigma)
        y = np.ascontiguousarray(y, dtype=np.int64)
        seg = np.ascontiguousarray(seg, dtype=np.int64)
        bf = np.ascontiguousarray(bf, dtype=np.uint8)
        w = np.zeros(omega, dtype=np.uint64)
        rc = self.L.orc_pack_desc(_p(y, _i64p), _p(seg, _i64p), _p(bf, _u8p), omega, sigma, yb, sb,
                                  _p(w, _u64p))
        if rc:
            raise OracleError(rc, "pack_tile_descriptor: field overflow")
        return w

    def unpack(self, words, omega, sigma):
        yb, sb, _ = self.layout(omega, sigma)
        w = np.ascontiguousarray(words, dtype=np.uint64)
        y = np.zeros(omega, dtype=np.int64)
        s = np.zeros(omega, dtype=np.int64)
        bf = np.zeros(omega * sigma, dtype=np.uint8)
        self.L.orc_unpack_desc(_p(w, _u64p), omega, sigma, yb, sb, _p(y, _i64p), _p(s, _i64p),
                               _p(bf, _u8p))
        return y, s, bf

    def serial_segsum(self, data, flags):
        d = np.array(data, dtype=np.float64)
        f = np.ascontiguousarray(flags, dtype=np.uint8)
        self.L.orc_serial_segsum(_p(d, _f64p), _p(f, _u8p), len(d))
        return d

    def fast_segsum(self, data, seg):
        d = np.array(data, dtype=np.float64)
        s = np.ascontiguousarray(seg, dtype=np.int64)
        rc = self.L.orc_fast_segsum(_p(d, _f64p), _p(s, _i64p), len(d))
        if rc:
            raise OracleError(rc, "fast_segmented_sum: seg_offset reaches past the end")
        return d

    # -- format + spmv --------------------------------------------------
    def _build_struct(self, a: Csr, omega, sigma, r=4, s=32, t=256, u=4):
        st = _OrcCsr5()
        err = C.create_string_buffer(512)
        rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(a.col_idx, dtype=np.int64)
        va = np.ascontiguousarray(a.val, dtype=np.float64)
        rc = self.L.orc_build(a.m, a.n, _p(rp, _i64p), _p(ci, _i64p), _p(va, _f64p), omega, sigma,
                              r, s, t, u, C.byref(st), err, 512)
        if rc:
            raise OracleError(rc, err.value.decode())
        return st

    def build(self, a: Csr, omega: int, sigma: int, r=4, s=32, t=256, u=4) -> Csr5Arrays:
        st = self._build_struct(a, omega, sigma, r, s, t, u)
        try:
            return Csr5Arrays(
                m=st.m, n=st.n, nnz=st.nnz, omega=st.omega, sigma=st.sigma, p=st.p, pc=st.pc,
                tail_len=st.tail_len, tile_ptr_bits=st.tile_ptr_bits, word_bits=st.word_bits,
                y_bits=st.y_bits, seg_bits=st.seg_bits,
                tile_ptr=_copy(st.tile_ptr, st.p + 1, np.uint64),
                tile_desc=_copy(st.tile_desc, st.pc * st.omega, np.uint64),
                eo_ptr=_copy(st.eo_ptr, st.pc + 1, np.int64),
                eo=_copy(st.eo, int(st.eo_ptr[st.pc]) if st.pc >= 0 else 0, np.int64),
                col_idx=_copy(st.col_idx, st.nnz, np.int64),
                val=_copy(st.val, st.nnz, np.float64),
            )
        finally:
            self.L.orc_free(C.byref(st))

    def spmv(self, a: Csr, x: np.ndarray, omega=32, sigma=None) -> np.ndarray:
        """Deterministic spmv_csr5 (spmv.cpp:224-272) after csr_to_csr5."""
        if sigma is None:
            sigma = self.select_sigma(a.nnz / a.m if a.m else 0.0)
        st = self._build_struct(a, omega, sigma)
        try:
            y = np.zeros(a.m, dtype=np.float64)
            xx = np.ascontiguousarray(x, dtype=np.float64)
            self.L.orc_spmv(C.byref(st), _p(xx, _f64p), _p(y, _f64p))
            return y
        finally:
            self.L.orc_free(C.byref(st))

    def tile_contrib(self, a: Csr, omega, sigma, tid, x):
        st = self._build_struct(a, omega, sigma)
        try:
            cap = omega * sigma + 1
            rows = np.zeros(cap, dtype=np.int64)
            vals = np.zeros(cap, dtype=np.float64)
            acc = np.zeros(cap, dtype=np.uint8)
            xx = np.ascontiguousarray(x, dtype=np.float64)
            k = self.L.orc_tile_contrib(C.byref(st), tid, _p(xx, _f64p), _p(rows, _i64p),
                                        _p(vals, _f64p), _p(acc, _u8p), cap)
            if k < 0:
                raise OracleError(1, f"spmv_csr5_tile: tile {tid} is not a complete tile")
            return rows[:k], vals[:k], acc[:k].astype(bool)
        finally:
            self.L.orc_free(C.byref(st))

    def to_csr(self, a: Csr, omega, sigma):
        st = self._build_struct(a, omega, sigma)
        try:
            ci = np.zeros(a.nnz, dtype=np.int64)
            va = np.zeros(a.nnz, dtype=np.float64)
            self.L.orc_csr5_to_csr(C.byref(st), _p(ci, _i64p), _p(va, _f64p))
            return ci, va
        finally:
            self.L.orc_free(C.byref(st))

    def dense_spmv(self, a: Csr, x) -> np.ndarray:
        y = np.zeros(a.m, dtype=np.float64)
        xx = np.ascontiguousarray(x, dtype=np.float64)
        rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(a.col_idx, dtype=np.int64)
        va = np.ascontiguousarray(a.val, dtype=np.float64)
        self.L.orc_dense_spmv(a.m, _p(rp, _i64p), _p(ci, _i64p), _p(va, _f64p), _p(xx, _f64p),
                              _p(y, _f64p))
        return y

    # -- generators (tests/test_helpers.hpp, synthetic.cpp) ---------------
    def _take_csr(self, st: _OrcCsr) -> Csr:
        try:
            return Csr(st.m, st.n, _copy(st.row_ptr, st.m + 1, np.int64),
                       _copy(st.col_idx, st.nnz, np.int64), _copy(st.val, st.nnz, np.float64))
        finally:
            self.L.orc_csr_free(C.byref(st))

    def rng(self, seed: int) -> "Rng":
        return Rng(self, seed)

    def coo_to_csr(self, rows, cols, vals, m, n) -> Csr:
        r = np.ascontiguousarray(rows, dtype=np.int64)
        c = np.ascontiguousarray(cols, dtype=np.int64)
        v = np.ascontiguousarray(vals, dtype=np.float64)
        st = _OrcCsr()
        self.L.orc_coo_to_csr(_p(r, _i64p), _p(c, _i64p), _p(v, _f64p), len(r), m, n, C.byref(st))
        return self._take_csr(st)

    def generate_synthetic(self, kind: int, m, n, nnz, seed, frac=0.15) -> Csr:
        st = _OrcCsr()
        rc = self.L.orc_generate_synthetic(kind, m, n, nnz, seed, frac, C.byref(st))
        if rc:
            raise OracleError(1, "generate_synthetic: infeasible target")
        return self._take_csr(st)


class Rng:
    """std::mt19937_64 restated (testgen.c); state shared across helpers."""

    def __init__(self, orc: Oracle, seed: int):
        self.o = orc
        self.h = C.c_void_p(orc.L.orc_mt64_new(seed))

    def __del__(self):
        try:
            self.o.L.orc_mt64_delete(self.h)
        except Exception:
            pass

    def __call__(self) -> int:
        return int(self.o.L.orc_mt64_next(self.h))

    def random_csr(self, m, n, nnz_target) -> Csr:
        st = _OrcCsr()
        self.o.L.orc_random_csr(self.h, m, n, nnz_target, C.byref(st))
        return self.o._take_csr(st)

    def random_x(self, n) -> np.ndarray:
        x = np.zeros(n, dtype=np.float64)
        self.o.L.orc_random_x(self.h, n, _p(x, _f64p))
        return x


class Ref:
    """The unmodified reference library (oracle/_ref/libcsr5ref.so)."""

    def __init__(self, path: str = LIB_REF):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (built only where /root/reference exists)")
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_build.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _f64p] + [C.c_int64] * 6 + [
            C.c_int, C.POINTER(C.c_void_p), _f64p]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_info.argtypes = [C.c_void_p, _i64p]
        L.ref_metadata_bytes.argtypes = [C.c_void_p]
        L.ref_metadata_bytes.restype = C.c_int64
        L.ref_export.argtypes = [C.c_void_p, _u64p, _u64p, _i64p, _i64p, _i64p, _f64p]
        L.ref_spmv.argtypes = [C.c_void_p, _f64p, _f64p, C.c_int]
        L.ref_vec_new.argtypes = [_f64p, C.c_int64]
        L.ref_vec_new.restype = C.c_void_p
        L.ref_vec_free.argtypes = [C.c_void_p]
        L.ref_time_spmv.argtypes = [C.c_void_p, C.c_void_p, _f64p, C.c_int, C.c_int]
        L.ref_time_spmv.restype = C.c_double
        L.ref_time_csr_scalar.argtypes = [C.c_void_p, C.c_void_p, _f64p, C.c_int]
        L.ref_time_csr_scalar.restype = C.c_double
        L.ref_tile_contrib.argtypes = [C.c_void_p, C.c_int64, _f64p, _i64p, _f64p, _u8p, C.c_int64]
        L.ref_tile_contrib.restype = C.c_int64
        L.ref_to_csr.argtypes = [C.c_void_p, _i64p, _f64p]
        L.ref_dense_spmv.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.ref_select_sigma.argtypes = [C.c_double] + [C.c_int64] * 4 + [_i64p]
        L.ref_generate.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_double,
                                   C.POINTER(C.c_int)]
        L.ref_generate.restype = C.c_void_p
        L.ref_csr_nnz.argtypes = [C.c_void_p]
        L.ref_csr_nnz.restype = C.c_int64
        L.ref_csr_get.argtypes = [C.c_void_p, _i64p, _i64p, _f64p]
        L.ref_csr_free.argtypes = [C.c_void_p]
        L.ref_max_threads.restype = C.c_int
        L.ref_dump_format.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.ref_dump_format.restype = C.c_int64
        L.ref_set_threads.argtypes = [C.c_int]

    def _err(self, rc):
        raise OracleError(rc, self.L.ref_last_error().decode())

    def max_threads(self) -> int:
        return self.L.ref_max_threads()

    def set_threads(self, n: int):
        self.L.ref_set_threads(n)

    def build_handle(self, a: Csr, omega, sigma, r=4, s=32, t=256, u=4, parallel=True):
        h = C.c_void_p()
        ms = C.c_double()
        rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(a.col_idx, dtype=np.int64)
        va = np.ascontiguousarray(a.val, dtype=np.float64)
        rc = self.L.ref_build(a.m, a.n, _p(rp, _i64p), _p(ci, _i64p), _p(va, _f64p), omega, sigma,
                              r, s, t, u, int(parallel), C.byref(h), C.byref(ms))
        if rc:
            self._err(rc)
        return h, ms.value

    def build(self, a: Csr, omega: int, sigma: int, r=4, s=32, t=256, u=4) -> Csr5Arrays:
        h, _ = self.build_handle(a, omega, sigma, r, s, t, u)
        try:
            info = np.zeros(8, dtype=np.int64)
            self.L.ref_info(h, _p(info, _i64p))
            p, pc, tail, tpb, wb, neo, yb, sb = (int(v) for v in info)
            tile_ptr = np.zeros(p + 1, dtype=np.uint64)
            tile_desc = np.zeros(pc * omega, dtype=np.uint64)
            eo_ptr = np.zeros(pc + 1, dtype=np.int64)
            eo = np.zeros(neo, dtype=np.int64)
            ci = np.zeros(a.nnz, dtype=np.int64)
            va = np.zeros(a.nnz, dtype=np.float64)
            self.L.ref_export(h, _p(tile_ptr, _u64p), _p(tile_desc, _u64p), _p(eo_ptr, _i64p),
                              _p(eo, _i64p), _p(ci, _i64p), _p(va, _f64p))
            return Csr5Arrays(a.m, a.n, a.nnz, omega, sigma, p, pc, tail, tpb, wb, yb, sb, tile_ptr,
                              tile_desc, eo_ptr, eo, ci, va)
        finally:
            self.L.ref_free(h)

    def dump_format(self, a: Csr, omega: int, sigma: int) -> str:
        """format.cpp:267-305: the reference's own text dump of its build."""
        h, _ = self.build_handle(a, omega, sigma)
        try:
            n = self.L.ref_dump_format(h, None, 0)
            buf = C.create_string_buffer(n + 1)
            self.L.ref_dump_format(h, buf, n)
            return buf.raw[:n].decode()
        finally:
            self.L.ref_free(h)

    def spmv(self, a: Csr, x, omega=32, sigma=None, mode=0) -> np.ndarray:
        if sigma is None:
            sigma = self.select_sigma(a.nnz / a.m if a.m else 0.0)
        h, _ = self.build_handle(a, omega, sigma)
        try:
            y = np.zeros(a.m, dtype=np.float64)
            xx = np.ascontiguousarray(x, dtype=np.float64)
            rc = self.L.ref_spmv(h, _p(xx, _f64p), _p(y, _f64p), mode)
            if rc:
                self._err(rc)
            return y
        finally:
            self.L.ref_free(h)

    def tile_contrib(self, a: Csr, omega, sigma, tid, x):
        h, _ = self.build_handle(a, omega, sigma)
        try:
            cap = omega * sigma + 1
            rows = np.zeros(cap, dtype=np.int64)
            vals = np.zeros(cap, dtype=np.float64)
            acc = np.zeros(cap, dtype=np.uint8)
            xx = np.ascontiguousarray(x, dtype=np.float64)
            k = self.L.ref_tile_contrib(h, tid, _p(xx, _f64p), _p(rows, _i64p), _p(vals, _f64p),
                                        _p(acc, _u8p), cap)
            if k < 0:
                self._err(1)
            return rows[:k], vals[:k], acc[:k].astype(bool)
        finally:
            self.L.ref_free(h)

    def to_csr(self, a: Csr, omega, sigma):
        h, _ = self.build_handle(a, omega, sigma)
        try:
            ci = np.zeros(a.nnz, dtype=np.int64)
            va = np.zeros(a.nnz, dtype=np.float64)
            rc = self.L.ref_to_csr(h, _p(ci, _i64p), _p(va, _f64p))
            if rc:
                self._err(rc)
            return ci, va
        finally:
            self.L.ref_free(h)

    def select_sigma(self, npr, r=4, s=32, t=256, u=4) -> int:
        out = C.c_int64()
        rc = self.L.ref_select_sigma(npr, r, s, t, u, C.byref(out))
        if rc:
            self._err(rc)
        return out.value

    def dense_spmv(self, a: Csr, x) -> np.ndarray:
        y = np.zeros(a.m, dtype=np.float64)
        xx = np.ascontiguousarray(x, dtype=np.float64)
        self.L.ref_dense_spmv(a.m, a.n, _p(np.ascontiguousarray(a.row_ptr), _i64p),
                              _p(np.ascontiguousarray(a.col_idx), _i64p),
                              _p(np.ascontiguousarray(a.val), _f64p), _p(xx, _f64p), _p(y, _f64p))
        return y

    def generate_synthetic(self, kind, m, n, nnz, seed, frac=0.15) -> Csr:
        rc = C.c_int()
        h = self.L.ref_generate(kind, m, n, nnz, seed, frac, C.byref(rc))
        if rc.value:
            self._err(rc.value)
        try:
            nz = self.L.ref_csr_nnz(h)
            rp = np.zeros(m + 1, dtype=np.int64)
            ci = np.zeros(nz, dtype=np.int64)
            va = np.zeros(nz, dtype=np.float64)
            self.L.ref_csr_get(h, _p(rp, _i64p), _p(ci, _i64p), _p(va, _f64p))
            return Csr(m, n, rp, ci, va)
        finally:
            self.L.ref_csr_free(h)


def have_ref() -> bool:
    return os.path.exists(LIB_REF)


def stencil_box_size(kind: int, a: int, layers: int) -> tuple[int, int]:
    """(m, nnz) of the a x .. x layers stencil (mirrors csr5g_stencil_box_size)."""
    def ax(e):
        return 1 if e == 1 else 3 * e - 2
    if kind == 0:
        return a * layers, a * layers + 2 * (a - 1) * layers + 2 * (layers - 1) * a
    return a * a * layers, ax(a) * ax(a) * ax(layers)


def stencil(orc: "Oracle", kind: int, a: int, layers: int | None = None) -> Csr:
    """Host twin of csr5g_stencil_box_fill (testgen.c orc_stencil_box)."""
    import ctypes as C
    layers = a if layers is None else layers
    m, nnz = stencil_box_size(kind, a, layers)
    rp = np.empty(m + 1, np.int64)
    ci = np.empty(nnz, np.int64)
    va = np.empty(nnz, np.float64)
    fn = orc.L.orc_stencil_box
    fn.argtypes = [C.c_int, C.c_int64, C.c_int64, _i64p, _i64p, _f64p]
    fn(kind, a, layers, _p(rp, _i64p), _p(ci, _i64p), _p(va, _f64p))
    return Csr(m, m, rp, ci, va)
