"""Loads libcsr5g.so (the CUDA product) and declares its C ABI (include/csr5g.h).

There is no fallback: if the shared library is missing or has no usable
sm_100 device, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CSR5G_LIB_OVERRIDE") or os.path.join(HERE, "libcsr5g.so")  # A/B experiments

OK, EINVAL, ERUNTIME, ERANGE, ECUDA, ENOMEM = 0, 1, 2, 3, 4, 5
MODE_DETERMINISTIC, MODE_ATOMIC = 0, 1
IPC_HANDLE_BYTES, MAX_WORLD = 64, 64


class Csr5CudaError(RuntimeError):
    """A CUDA-side failure (no device, launch error)."""


class Params(C.Structure):
    _fields_ = [("omega", C.c_int64), ("sigma", C.c_int64), ("r", C.c_int64), ("s", C.c_int64),
                ("t", C.c_int64), ("u", C.c_int64)]


class Info(C.Structure):
    _fields_ = [
        ("m", C.c_int64), ("n", C.c_int64), ("nnz", C.c_int64),
        ("omega", C.c_int64), ("sigma", C.c_int64),
        ("p", C.c_int64), ("p_complete", C.c_int64), ("tail_len", C.c_int64),
        ("tile_begin", C.c_int64), ("tile_end", C.c_int64),
        ("has_tail", C.c_int32),
        ("tile_ptr_bits", C.c_int32), ("word_bits", C.c_int32), ("y_offset_bits", C.c_int32),
        ("seg_offset_bits", C.c_int32),
        ("num_sms", C.c_int32), ("spmv_warps", C.c_int32),
        ("tile_ptr_len", C.c_int64), ("empty_offset_len", C.c_int64), ("nnz_held", C.c_int64),
        ("metadata_bytes", C.c_int64), ("device_bytes", C.c_int64), ("spmv_bytes", C.c_int64),
        ("first_row", C.c_int64), ("last_row", C.c_int64),
        ("own_row_begin", C.c_int64), ("own_row_end", C.c_int64),
        ("build_ms", C.c_double), ("alloc_ms", C.c_double),
        ("lines_per_gather", C.c_double),
        ("warps_per_cta", C.c_int32), ("stages", C.c_int32), ("smem_bytes", C.c_int32),
        ("x_mode", C.c_int32), ("x_window", C.c_int32), ("kernel_variant", C.c_int32),
        ("long_rows", C.c_int64),
        ("hot_cols", C.c_int64),
        ("hot_coverage", C.c_double),
    ]


class Partial(C.Structure):
    _fields_ = [("row", C.c_int64), ("value", C.c_double)]


_vp = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32

# name -> (restype, argtypes); the single source the symbol test checks against
SIGNATURES = {
    "csr5g_last_error": (C.c_char_p, []),
    "csr5g_version": (C.c_char_p, []),
    "csr5g_select_sigma": (C.c_int, [C.c_double, _i64, _i64, _i64, _i64, C.POINTER(_i64)]),
    "csr5g_layout": (C.c_int, [_i64, _i64, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32)]),
    "csr5g_build": (C.c_int, [C.c_int, _i64, _i64, _i64, _vp, _vp, _vp, C.POINTER(Params), _vp,
                              C.POINTER(_vp)]),
    "csr5g_build_shard": (C.c_int, [C.c_int, _i64, _i64, _i64, _vp, _vp, _vp, C.POINTER(Params),
                                    _i64, _i64, _i32, _vp, C.POINTER(_vp)]),
    "csr5g_info_get": (C.c_int, [_vp, C.POINTER(Info)]),
    "csr5g_export": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "csr5g_spmv": (C.c_int, [_vp, _vp, _vp, _i32, _vp]),
    "csr5g_spmv_evt": (C.c_int, [_vp, _vp, _vp, _i32, _vp, _vp, _vp]),
    "csr5g_shard_send_record": (C.c_int, [_vp, C.POINTER(_vp)]),
    "csr5g_set_send_buffer": (C.c_int, [_vp, _vp]),
    "csr5g_fixup": (C.c_int, [_vp, _vp, _i32, _i32, _vp, _vp]),
    "csr5g_mailbox_create": (C.c_int, [C.c_int, _i32, _i32, _i64, C.POINTER(_vp)]),
    "csr5g_mailbox_vector": (C.c_int, [_vp, _i32, C.POINTER(_vp)]),
    "csr5g_mailbox_ipc_handle": (C.c_int, [_vp, _vp]),
    "csr5g_mailbox_open_peer": (C.c_int, [_vp, _i32, _vp]),
    "csr5g_mailbox_link_local": (C.c_int, [_vp, _i32, _vp]),
    "csr5g_mailbox_errors": (C.c_int, [_vp, C.POINTER(C.c_uint32)]),
    "csr5g_mailbox_release": (C.c_int, [_vp]),
    "csr5g_mcast_supported": (C.c_int, [C.c_int, C.POINTER(C.c_int32)]),
    "csr5g_mailbox_mcast_create": (C.c_int, [_vp, _i32, _vp]),
    "csr5g_mailbox_mcast_import": (C.c_int, [_vp, _i32, _vp]),
    "csr5g_mailbox_mcast_add": (C.c_int, [_vp]),
    "csr5g_mailbox_mcast_bind": (C.c_int, [_vp]),
    "csr5g_mailbox_mcast_release": (C.c_int, [_vp]),
    "csr5g_mailbox_mcast_selftest": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "csr5g_mg_bind": (C.c_int, [_vp, _vp, _i32, _i32, _i32, _i32]),
    "csr5g_mg_spmv_post": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "csr5g_mg_spmv_fixup": (C.c_int, [_vp, _vp, _vp]),
    "csr5g_mg_spmv": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "csr5g_mg_iter_post": (C.c_int, [_vp, _i64, _vp, _vp, _vp]),
    "csr5g_mg_iter_finish": (C.c_int, [_vp, _i64, _vp]),
    "csr5g_mg_iter": (C.c_int, [_vp, _i64, _vp, _vp, _vp]),
    "csr5g_to_csr": (C.c_int, [_vp, _vp, _vp, _vp]),
    "csr5g_release": (C.c_int, [_vp]),
    "csr5g_build_host": (C.c_int, [C.c_int, _i64, _i64, _i64, _vp, _vp, _vp, C.POINTER(Params),
                                   C.POINTER(_vp)]),
    "csr5g_spmv_host": (C.c_int, [_vp, _vp, _vp, _i32]),
    "csr5g_spmv_host_batch": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "csr5g_to_csr_host": (C.c_int, [_vp, _vp, _vp]),
    "csr5g_mm_read": (C.c_int, [C.c_char_p, C.POINTER(_vp), C.POINTER(_i64), C.POINTER(_i64),
                                C.POINTER(_i64)]),
    "csr5g_mm_parse": (C.c_int, [C.c_char_p, _i64, C.POINTER(_vp), C.POINTER(_i64),
                                 C.POINTER(_i64), C.POINTER(_i64)]),
    "csr5g_coo_get": (C.c_int, [_vp, _vp, _vp, _vp]),
    "csr5g_csr_spmv_host": (C.c_int, [C.c_int, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "csr5g_export_row_ptr": (C.c_int, [_vp, _vp]),
    "csr5g_spmv_tile": (C.c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _i64, C.POINTER(_i64)]),
    "csr5g_coo_release": (C.c_int, [_vp]),
    "csr5g_coo_to_csr": (C.c_int, [C.c_int, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                   C.POINTER(_i64), _vp]),
    "csr5g_coo_to_csr_host": (C.c_int, [C.c_int, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                        C.POINTER(_i64)]),
    "csr5g_csr_spmv": (C.c_int, [C.c_int, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "csr5g_event_create": (C.c_int, [C.POINTER(_vp)]),
    "csr5g_event_record": (C.c_int, [_vp, _vp]),
    "csr5g_event_elapsed_ms": (C.c_int, [_vp, _vp, C.POINTER(C.c_float)]),
    "csr5g_event_destroy": (C.c_int, [_vp]),
    "csr5g_stream_synchronize": (C.c_int, [_vp]),
    "csr5g_stencil_size": (C.c_int, [_i32, _i64, C.POINTER(_i64), C.POINTER(_i64)]),
    "csr5g_stencil_fill": (C.c_int, [_i32, _i64, _vp, _vp, _vp, _vp]),
    "csr5g_stencil_box_size": (C.c_int, [_i32, _i64, _i64, C.POINTER(_i64), C.POINTER(_i64)]),
    "csr5g_stencil_box_fill": (C.c_int, [_i32, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp]),
    "csr5g_rmat_create": (C.c_int, [_i32, _i32, C.c_uint64, _i32, _vp, C.POINTER(_vp),
                                    C.POINTER(_i64), C.POINTER(_i64)]),
    "csr5g_mixed_create": (C.c_int, [_i32, C.c_double, _i32, _i64, _i32, _i32, C.c_uint64, _vp,
                                     C.POINTER(_vp), C.POINTER(_i64), C.POINTER(_i64)]),
    "csr5g_gen_fill": (C.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "csr5g_bench_x": (C.c_int, [_i64, C.c_uint64, _vp]),
    "csr5g_gen_fill_range": (C.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "csr5g_gen_release": (C.c_int, [_vp]),
}

_LIB = None


def lib() -> C.CDLL:
    """The loaded product library (raises if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make lib` (or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(rc: int) -> None:
    """Raise the Python analogue of the reference's exception for a status."""
    if rc == OK:
        return
    msg = lib().csr5g_last_error().decode()
    if rc == EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == ERANGE:
        raise IndexError(msg)  # std::out_of_range
    if rc == ENOMEM:
        raise MemoryError(msg)
    if rc == ECUDA:
        raise Csr5CudaError(msg)
    raise RuntimeError(msg)  # std::runtime_error
