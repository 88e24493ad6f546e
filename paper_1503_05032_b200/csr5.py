"""Host-side mirror of the reference API (namespace csr5, proj/core) over the
CUDA C ABI.  Same names, argument meaning and error behaviour:

=========================  =====================================================
reference (proj/core)      here
=========================  =====================================================
TuningParams               TuningParams (omega must be 32; sigma=0 -> auto rule)
CsrMatrix                  CsrMatrix (device tensors: int64 row_ptr, int32 col_idx,
                           float64 val)
csr_to_csr5(a, params)     csr_to_csr5(a, params) -> Csr5Matrix (device handle)
spmv_csr5(a5, x, y, mode)  spmv_csr5(a5, x, y=None, mode="deterministic")
csr5_to_csr(a5)            csr5_to_csr(a5) -> CsrMatrix
dump_format(a5, out)       dump_format(a5) -> str
Csr5Matrix dtor            Csr5Matrix.release() (also on garbage collection)
std::invalid_argument      ValueError (same message text)
=========================  =====================================================

torch is used only as device-memory and stream plumbing; all compute is in
libcsr5g.so.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import (MODE_ATOMIC, MODE_DETERMINISTIC, Info, Params, Partial, check, lib)

_MODES = {"deterministic": MODE_DETERMINISTIC, "atomic": MODE_ATOMIC,
          MODE_DETERMINISTIC: MODE_DETERMINISTIC, MODE_ATOMIC: MODE_ATOMIC}


@dataclass
class TuningParams:
    """tuning.hpp:13-24.  GPU tiles are one warp wide, so omega = 32."""

    omega: int = 32
    sigma: int = 0  # 0: select_sigma(nnz/m, <r,s,t,u>) like `spmv-bench --sigma auto`
    r: int = 4
    s: int = 32
    t: int = 256
    u: int = 4

    def _c(self) -> Params:
        return Params(self.omega, self.sigma, self.r, self.s, self.t, self.u)


@dataclass
class CsrMatrix:
    """Canonical CSR on the device (csr.hpp:25-35)."""

    m: int
    n: int
    row_ptr: torch.Tensor  # int64 [m+1]
    col_idx: torch.Tensor  # int32 [nnz]
    val: torch.Tensor  # float64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    @staticmethod
    def from_host(m, n, row_ptr, col_idx, val, device="cuda") -> "CsrMatrix":
        return CsrMatrix(
            int(m), int(n),
            torch.as_tensor(np.ascontiguousarray(row_ptr, dtype=np.int64)).to(device),
            torch.as_tensor(np.ascontiguousarray(col_idx, dtype=np.int32)).to(device),
            torch.as_tensor(np.ascontiguousarray(val, dtype=np.float64)).to(device),
        )


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def select_sigma(nnz_per_row: float, r=4, s=32, t=256, u=4) -> int:
    """tuning.cpp:25-34."""
    out = C.c_int64()
    check(lib().csr5g_select_sigma(float(nnz_per_row), r, s, t, u, C.byref(out)))
    return out.value


def layout(omega: int, sigma: int):
    """descriptor.cpp:22-36 -> (y_offset_bits, seg_offset_bits, word_bits)."""
    yb, sb, wb = C.c_int32(), C.c_int32(), C.c_int32()
    check(lib().csr5g_layout(omega, sigma, C.byref(yb), C.byref(sb), C.byref(wb)))
    return yb.value, sb.value, wb.value


class Csr5Matrix:
    """Owning handle to the device CSR5 arrays (format.hpp:130-176)."""

    def __init__(self, handle: C.c_void_p, device: int):
        self._h = handle
        self.device = device
        info = Info()
        check(lib().csr5g_info_get(self._h, C.byref(info)))
        self.info = info

    # reference field names
    def __getattr__(self, name):
        info = self.__dict__.get("info")
        if info is not None and name in dict(Info._fields_):
            return getattr(info, name)
        raise AttributeError(name)

    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise ValueError("csr5g: matrix was released")
        return self._h

    def release(self) -> None:
        if getattr(self, "_h", None) is not None:
            lib().csr5g_release(self._h)
            self._h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass

    def export(self) -> dict:
        """All held arrays on the host, widened like the reference (uint64 words,
        int64 indices)."""
        i = self.info
        pcs = i.tile_end - i.tile_begin
        out = dict(
            tile_ptr=np.zeros(i.tile_ptr_len, np.uint64),
            tile_desc=np.zeros(pcs * i.omega, np.uint64),
            eo_ptr=np.zeros(pcs + 1, np.int64),
            eo=np.zeros(i.empty_offset_len, np.int64),
            col_idx=np.zeros(i.nnz_held, np.int64),
            val=np.zeros(i.nnz_held, np.float64),
        )
        check(lib().csr5g_export(self.handle, *(C.c_void_p(a.ctypes.data) for a in out.values())))
        return out

    def send_record_ptr(self) -> int:
        p = C.c_void_p()
        check(lib().csr5g_shard_send_record(self.handle, C.byref(p)))
        return p.value


def _check_csr(a: CsrMatrix):
    for name, t, dt in (("row_ptr", a.row_ptr, torch.int64), ("col_idx", a.col_idx, torch.int32),
                        ("val", a.val, torch.float64)):
        if not t.is_cuda or t.dtype != dt or not t.is_contiguous():
            raise ValueError(f"csr5g: {name} must be a contiguous CUDA {dt} tensor")
    if a.row_ptr.numel() != a.m + 1:
        raise ValueError(f"csr: row_ptr has size {a.row_ptr.numel()}, expected {a.m + 1}")


def csr_to_csr5(a: CsrMatrix, params: TuningParams | None = None, stream=None) -> Csr5Matrix:
    """format.cpp:165-252: build the tiled format on the device (input untouched)."""
    params = params or TuningParams()
    _check_csr(a)
    dev = a.row_ptr.device.index or 0
    h = C.c_void_p()
    with torch.cuda.device(dev):
        check(lib().csr5g_build(dev, a.m, a.n, a.nnz, a.row_ptr.data_ptr(), a.col_idx.data_ptr(),
                                a.val.data_ptr(), C.byref(params._c()), _stream_ptr(stream),
                                C.byref(h)))
    return Csr5Matrix(h, dev)


def csr_to_csr5_shard(a_row_ptr: torch.Tensor, col_slice: torch.Tensor, val_slice: torch.Tensor,
                      m: int, n: int, nnz: int, params: TuningParams, tile_begin: int,
                      tile_end: int, with_tail: bool, stream=None) -> Csr5Matrix:
    """Shard of the global tile range [tile_begin, tile_end) (multi-GPU driver)."""
    dev = a_row_ptr.device.index or 0
    h = C.c_void_p()
    with torch.cuda.device(dev):
        check(lib().csr5g_build_shard(dev, m, n, nnz, a_row_ptr.data_ptr(), col_slice.data_ptr(),
                                      val_slice.data_ptr(), C.byref(params._c()), tile_begin,
                                      tile_end, int(with_tail), _stream_ptr(stream), C.byref(h)))
    return Csr5Matrix(h, dev)


def spmv_csr5(a5: Csr5Matrix, x: torch.Tensor, y: torch.Tensor | None = None,
              mode="deterministic", stream=None) -> torch.Tensor:
    """spmv.cpp:224-298: y = A x on the device; y is fully overwritten."""
    if x.dim() != 1 or x.numel() != a5.n:
        raise ValueError(f"spmv: x has length {x.numel()}, expected {a5.n}")
    if y is None:
        y = torch.empty(a5.m, dtype=torch.float64, device=x.device)
    elif y.numel() != a5.m:
        raise ValueError(f"spmv: y has length {y.numel()}, expected {a5.m}")
    if x.dtype != torch.float64 or y.dtype != torch.float64 or not x.is_cuda or not y.is_cuda:
        raise ValueError("spmv: x and y must be CUDA float64 tensors")
    if mode not in _MODES:
        raise ValueError(f"spmv: unknown mode {mode!r}")
    with torch.cuda.device(a5.device):
        check(lib().csr5g_spmv(a5.handle, x.data_ptr(), y.data_ptr(), _MODES[mode],
                               _stream_ptr(stream)))
    return y


def spmv_host(a5: Csr5Matrix, x: np.ndarray, mode="deterministic") -> np.ndarray:
    """Host-vector overload (spmv.hpp:60) through csr5g_spmv_host: x H2D, SpMV,
    y D2H on the handle's pipeline; returns a new host y."""
    if mode not in _MODES:
        raise ValueError(f"spmv: unknown mode {mode!r}")
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim != 1 or x.size != a5.n:
        raise ValueError(f"spmv: x has length {x.size}, expected {a5.n}")
    y = np.empty(a5.m, dtype=np.float64)
    with torch.cuda.device(a5.device):
        check(lib().csr5g_spmv_host(a5.handle, x.ctypes.data, y.ctypes.data, _MODES[mode]))
    return y


def _host_ptr(v, length: int, what: str) -> int:
    if isinstance(v, torch.Tensor):
        if v.is_cuda or v.dtype != torch.float64 or not v.is_contiguous() or v.numel() != length:
            raise ValueError(f"spmv: {what} must be a contiguous host float64 tensor of length "
                             f"{length}")
        return v.data_ptr()
    if (not isinstance(v, np.ndarray) or v.dtype != np.float64 or not v.flags.c_contiguous
            or v.size != length):
        raise ValueError(f"spmv: {what} must be a contiguous float64 array of length {length}")
    return v.ctypes.data


def spmv_host_batch(a5: Csr5Matrix, xs, ys, mode="deterministic", stream=None) -> None:
    """y_k = A x_k for host vectors xs[k] -> ys[k] (numpy arrays or CPU tensors,
    pinned for overlap): one H2D + SpMV + D2H per vector, pipelined so that
    x_{k+1}'s copy in and y_k's copy out overlap SpMV k (csr5g_spmv_host_batch).
    Stream-ordered on `stream`: synchronise it before reading ys."""
    if len(xs) != len(ys):
        raise ValueError(f"spmv: {len(xs)} x vectors but {len(ys)} y vectors")
    if mode not in _MODES:
        raise ValueError(f"spmv: unknown mode {mode!r}")
    k = len(xs)
    px = (C.c_void_p * max(k, 1))(*[_host_ptr(v, a5.n, "x") for v in xs])
    py = (C.c_void_p * max(k, 1))(*[_host_ptr(v, a5.m, "y") for v in ys])
    with torch.cuda.device(a5.device):
        check(lib().csr5g_spmv_host_batch(a5.handle, px, py, k, _MODES[mode],
                                          _stream_ptr(stream)))


_CSR_KERNELS = {"csr-scalar": 0, "csr-segsum": 1}


def spmv_csr(a: CsrMatrix, x: torch.Tensor, y: torch.Tensor | None = None,
             kernel: str = "csr-scalar", stream=None) -> torch.Tensor:
    """spmv.cpp:139-209 spmv_csr_scalar / spmv_csr_segsum on the device
    (csr5g_csr_spmv): the plain-CSR baselines of run_benchmark."""
    if kernel not in _CSR_KERNELS:
        raise ValueError(f"unknown kernel '{kernel}' (expected csr-scalar or csr-segsum)")
    if x.dim() != 1 or x.numel() != a.n:
        raise ValueError(f"spmv: x has length {x.numel()}, expected {a.n}")
    if y is None:
        y = torch.empty(a.m, dtype=torch.float64, device=x.device)
    elif y.numel() != a.m:
        raise ValueError(f"spmv: y has length {y.numel()}, expected {a.m}")
    dev = a.row_ptr.device.index or 0
    with torch.cuda.device(dev):
        check(lib().csr5g_csr_spmv(dev, _CSR_KERNELS[kernel], a.m, a.n, a.nnz,
                                   a.row_ptr.data_ptr(), a.col_idx.data_ptr(), a.val.data_ptr(),
                                   x.data_ptr(), y.data_ptr(), _stream_ptr(stream)))
    return y


def read_matrix_market(path: str):
    """matrix_market.cpp:38-96 (csr5g_mm_read): (m, n, rows, cols, vals) as
    host numpy arrays, 0-based, symmetric files expanded.  Parse errors raise
    RuntimeError with the reference's text."""
    h, m, n, cnt = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int64()
    check(lib().csr5g_mm_read(os.fsencode(path), C.byref(h), C.byref(m), C.byref(n),
                              C.byref(cnt)))
    try:
        rows = np.empty(cnt.value, np.int64)
        cols = np.empty(cnt.value, np.int64)
        vals = np.empty(cnt.value, np.float64)
        check(lib().csr5g_coo_get(h, rows.ctypes.data, cols.ctypes.data, vals.ctypes.data))
    finally:
        lib().csr5g_coo_release(h)
    return m.value, n.value, rows, cols, vals


def coo_to_csr(rows, cols, vals, m: int, n: int, device="cuda", stream=None) -> CsrMatrix:
    """csr.cpp:35-72 on the device (csr5g_coo_to_csr): sort by (row, col), sum
    duplicates in input order.  Out-of-range entries raise ValueError with the
    reference's std::invalid_argument text."""
    r = torch.as_tensor(rows, dtype=torch.int64).to(device).contiguous()
    c = torch.as_tensor(cols, dtype=torch.int64).to(device).contiguous()
    v = torch.as_tensor(vals, dtype=torch.float64).to(device).contiguous()
    k = r.numel()
    if c.numel() != k or v.numel() != k:
        raise ValueError("coo_to_csr: rows, cols and vals differ in length")
    rp = torch.empty(m + 1, dtype=torch.int64, device=device)
    ci = torch.empty(max(k, 1), dtype=torch.int32, device=device)
    va = torch.empty(max(k, 1), dtype=torch.float64, device=device)
    nnz = C.c_int64()
    dev = rp.device.index or 0
    with torch.cuda.device(dev):
        check(lib().csr5g_coo_to_csr(dev, m, n, k, r.data_ptr(), c.data_ptr(), v.data_ptr(),
                                     rp.data_ptr(), ci.data_ptr(), va.data_ptr(), C.byref(nnz),
                                     _stream_ptr(stream)))
    return CsrMatrix(m, n, rp, ci[:nnz.value].clone(), va[:nnz.value].clone())


def load_matrix_market(path: str, device="cuda") -> CsrMatrix:
    """matrix_market.cpp:98-101 load_matrix_market: read, then coo_to_csr on
    the device."""
    m, n, rows, cols, vals = read_matrix_market(path)
    return coo_to_csr(rows, cols, vals, m, n, device=device)


def csr5_to_csr(a5: Csr5Matrix, row_ptr: torch.Tensor, stream=None) -> CsrMatrix:
    """format.cpp:254-265: undo the tile transposition (row_ptr is unchanged by
    the format, so the caller's copy is reused)."""
    i = a5.info
    dev = f"cuda:{a5.device}"
    col = torch.empty(i.nnz_held, dtype=torch.int32, device=dev)
    val = torch.empty(i.nnz_held, dtype=torch.float64, device=dev)
    with torch.cuda.device(a5.device):
        check(lib().csr5g_to_csr(a5.handle, col.data_ptr(), val.data_ptr(), _stream_ptr(stream)))
    return CsrMatrix(i.m, i.n, row_ptr, col, val)


def spmv_csr5_tile(a5: Csr5Matrix, tid: int, x):
    """spmv.cpp:211-222 (TileContribution hook): the contributions of complete
    tile `tid`, computed by the GPU tile kernel itself (csr5g_spmv_tile), in
    the reference's emission order.  Returns (rows, values, accumulate)."""
    xh = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if xh.shape != (a5.n,):
        raise ValueError(f"spmv: x has length {xh.size}, expected {a5.n}")
    cap = 32 * a5.sigma + 1
    rows = np.zeros(cap, dtype=np.int64)
    vals = np.zeros(cap, dtype=np.float64)
    acc = np.zeros(cap, dtype=np.uint8)
    cnt = C.c_int64()
    check(lib().csr5g_spmv_tile(a5.handle, tid, xh.ctypes.data, rows.ctypes.data,
                                vals.ctypes.data, acc.ctypes.data, cap, C.byref(cnt)))
    k = cnt.value
    return rows[:k], vals[:k], acc[:k].astype(bool)


def dump_format(a5: Csr5Matrix) -> str:
    """format.cpp:267-305 text dump, produced from the device arrays."""
    i = a5.info
    ex = a5.export()
    om, sg = i.omega, i.sigma
    yb, sb = i.y_offset_bits, i.seg_offset_bits
    lines = [f"csr5 m={i.m} n={i.n} nnz={i.nnz} omega={om} sigma={sg} tiles={i.p} "
             f"complete={i.p_complete} tail={i.tail_len} tile_ptr_bits={i.tile_ptr_bits} "
             f"desc_word_bits={i.word_bits} metadata_bytes={i.metadata_bytes} "
             f"empty_offset_entries={i.empty_offset_len}"]
    ntiles = i.tile_ptr_len - 1
    for k in range(ntiles):
        tid = i.tile_begin + k
        raw = int(ex["tile_ptr"][k])
        row, emp = raw & 0x7FFFFFFF, raw >> 31
        s = f"tile {tid}: row={row} empty={emp}"
        if tid >= i.p_complete:
            lines.append(s + f" tail nnz={i.tail_len}")
            continue
        words = [int(w) for w in ex["tile_desc"][k * om:(k + 1) * om]]
        ys = [(w >> (sb + sg)) & ((1 << yb) - 1) for w in words]
        ss = [(w >> sg) & ((1 << sb) - 1) for w in words]
        bfs = ["".join("1" if (w >> (sg - 1 - j)) & 1 else "0" for j in range(sg)) for w in words]
        s += " y_offset=[" + ",".join(map(str, ys)) + "] seg_offset=[" + ",".join(map(str, ss))
        s += "] bit_flag=[" + ",".join(bfs) + "]"
        if emp:
            lo, hi = int(ex["eo_ptr"][k]), int(ex["eo_ptr"][k + 1])
            s += " empty_offset=[" + ",".join(str(int(v)) for v in ex["eo"][lo:hi]) + "]"
        lines.append(s)
    return "\n".join(lines) + "\n"


def stencil(kind: int, a: int, device="cuda", stream=None) -> CsrMatrix:
    """Synthetic 2D 5-point (kind 0) / 3D 27-point (kind 1) matrix on the device."""
    m, nnz = C.c_int64(), C.c_int64()
    check(lib().csr5g_stencil_size(kind, a, C.byref(m), C.byref(nnz)))
    rp = torch.empty(m.value + 1, dtype=torch.int64, device=device)
    ci = torch.empty(nnz.value, dtype=torch.int32, device=device)
    va = torch.empty(nnz.value, dtype=torch.float64, device=device)
    check(lib().csr5g_stencil_fill(kind, a, rp.data_ptr(), ci.data_ptr(), va.data_ptr(),
                                   _stream_ptr(stream)))
    return CsrMatrix(m.value, m.value, rp, ci, va)


def stencil_box_size(kind: int, a: int, layers: int) -> tuple[int, int]:
    """(m, nnz) of the stencil on an a x .. x layers box (csr5g_stencil_box_size)."""
    m, nnz = C.c_int64(), C.c_int64()
    check(lib().csr5g_stencil_box_size(kind, a, layers, C.byref(m), C.byref(nnz)))
    return m.value, nnz.value


def stencil_box(kind: int, a: int, layers: int, pos_begin: int = 0, pos_end: int | None = None,
                device="cuda", stream=None):
    """Stencil on a box whose outermost axis has `layers` points: the full
    row_ptr and the entries at global positions [pos_begin, pos_end) (a shard's
    slice).  Returns (m, nnz, row_ptr, col_slice, val_slice)."""
    m, nnz = stencil_box_size(kind, a, layers)
    hi = nnz if pos_end is None else pos_end
    rp = torch.empty(m + 1, dtype=torch.int64, device=device)
    ci = torch.empty(max(hi - pos_begin, 0), dtype=torch.int32, device=device)
    va = torch.empty(max(hi - pos_begin, 0), dtype=torch.float64, device=device)
    check(lib().csr5g_stencil_box_fill(kind, a, layers, pos_begin, hi, rp.data_ptr(),
                                       ci.data_ptr(), va.data_ptr(), _stream_ptr(stream)))
    return m, nnz, rp, ci, va


class Generator:
    """A sized synthetic matrix on the device (csr5g_rmat_create /
    csr5g_mixed_create): the full row_ptr and any slice of the entries."""

    def __init__(self, gen: C.c_void_p, m: int, nnz: int, device):
        self._g, self.m, self.n, self.nnz, self.device = gen, m, m, nnz, torch.device(device)

    def fill(self, pos_begin: int = 0, pos_end: int | None = None, with_row_ptr: bool = True,
             stream=None):
        """(row_ptr or None, col_idx[pos_begin:pos_end], val[pos_begin:pos_end])."""
        hi = self.nnz if pos_end is None else pos_end
        with torch.cuda.device(self.device):
            rp = (torch.empty(self.m + 1, dtype=torch.int64, device=self.device)
                  if with_row_ptr else None)
            ci = torch.empty(max(hi - pos_begin, 0), dtype=torch.int32, device=self.device)
            va = torch.empty(max(hi - pos_begin, 0), dtype=torch.float64, device=self.device)
            check(lib().csr5g_gen_fill_range(self._g, pos_begin, hi,
                                             rp.data_ptr() if rp is not None else None,
                                             ci.data_ptr(), va.data_ptr(), _stream_ptr(stream)))
            torch.cuda.synchronize(self.device)
        return rp, ci, va

    def matrix(self, stream=None) -> CsrMatrix:
        rp, ci, va = self.fill(stream=stream)
        return CsrMatrix(self.m, self.n, rp, ci, va)

    def release(self) -> None:
        if self._g:
            lib().csr5g_gen_release(self._g)
            self._g = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


def rmat_generator(scale: int, edge_factor: int = 16, seed: int = 1, permute: bool = True,
                   device="cuda", stream=None) -> Generator:
    """Graph500 R-MAT (a,b,c,d = .57,.19,.19,.05), duplicates removed."""
    g, m, nnz = C.c_void_p(), C.c_int64(), C.c_int64()
    with torch.cuda.device(torch.device(device)):
        check(lib().csr5g_rmat_create(scale, edge_factor, seed, int(permute), _stream_ptr(stream),
                                      C.byref(g), C.byref(m), C.byref(nnz)))
    return Generator(g, m.value, nnz.value, device)


def mixed_generator(log2_m: int = 23, p_empty: float = 0.4, n_long: int = 4,
                    long_len: int = 1 << 20, min_len: int = 1, max_len: int = 32, seed: int = 1,
                    device="cuda", stream=None) -> Generator:
    """40% empty rows plus a few 1M-nnz rows."""
    g, m, nnz = C.c_void_p(), C.c_int64(), C.c_int64()
    with torch.cuda.device(torch.device(device)):
        check(lib().csr5g_mixed_create(log2_m, p_empty, n_long, long_len, min_len, max_len, seed,
                                       _stream_ptr(stream), C.byref(g), C.byref(m),
                                       C.byref(nnz)))
    return Generator(g, m.value, nnz.value, device)


def rmat(scale: int, edge_factor: int = 16, seed: int = 1, permute: bool = True,
         device="cuda", stream=None) -> CsrMatrix:
    """Graph500 R-MAT (a,b,c,d = .57,.19,.19,.05), duplicates removed."""
    g = rmat_generator(scale, edge_factor, seed, permute, device, stream)
    try:
        return g.matrix(stream)
    finally:
        g.release()


def mixed(log2_m: int = 23, p_empty: float = 0.4, n_long: int = 4, long_len: int = 1 << 20,
          min_len: int = 1, max_len: int = 32, seed: int = 1, device="cuda",
          stream=None) -> CsrMatrix:
    """40% empty rows plus a few 1M-nnz rows."""
    g = mixed_generator(log2_m, p_empty, n_long, long_len, min_len, max_len, seed, device, stream)
    try:
        return g.matrix(stream)
    finally:
        g.release()


class Event:
    """cudaEvent from libcsr5g (timing on the launching stream)."""

    def __init__(self):
        self.p = C.c_void_p()
        check(lib().csr5g_event_create(C.byref(self.p)))

    def record(self, stream=None):
        check(lib().csr5g_event_record(self.p, _stream_ptr(stream)))

    def elapsed_ms(self, end: "Event") -> float:
        ms = C.c_float()
        check(lib().csr5g_event_elapsed_ms(self.p, end.p, C.byref(ms)))
        return ms.value

    def __del__(self):
        try:
            lib().csr5g_event_destroy(self.p)
        except Exception:
            pass


def spmv_csr5_evt(a5: Csr5Matrix, x: torch.Tensor, y: torch.Tensor, ev0: Event, ev1: Event,
                  mode="deterministic", stream=None) -> torch.Tensor:
    """spmv_csr5 recording ev0/ev1 around the tile kernel (roofline timing)."""
    check(lib().csr5g_spmv_evt(a5.handle, x.data_ptr(), y.data_ptr(), _MODES[mode],
                               _stream_ptr(stream), ev0.p, ev1.p))
    return y


__all__ = ["TuningParams", "CsrMatrix", "Csr5Matrix", "csr_to_csr5", "csr_to_csr5_shard",
           "spmv_csr5", "spmv_csr5_tile", "spmv_csr", "read_matrix_market", "coo_to_csr", "load_matrix_market", "spmv_host", "spmv_host_batch", "csr5_to_csr", "dump_format", "select_sigma", "layout",
           "stencil", "stencil_box", "stencil_box_size", "Event", "spmv_csr5_evt", "Partial"]
