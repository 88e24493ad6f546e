"""Helpers shared by the test modules (host-side checks only)."""
import numpy as np

from oracle.oracle import Csr


def row_tolerance(a: Csr, x: np.ndarray, rel: float = 1e-12) -> np.ndarray:
    """Per-row bound rel * max(1, nnz_i) * max_k |a_ik x_k| (SURVEY 8a / north star)."""
    prod = np.abs(a.val * x[a.col_idx]) if a.nnz else np.zeros(0)
    rmax = np.zeros(a.m)
    lens = np.diff(a.row_ptr)
    nz = lens > 0
    if a.nnz:
        starts = a.row_ptr[:-1][nz]
        rmax[nz] = np.maximum.reduceat(prod, starts)
    return rel * np.maximum(1, lens) * rmax


def assert_y_close(y: np.ndarray, y_ref: np.ndarray, a: Csr, x: np.ndarray, what=""):
    """y within the stated fp64 tolerance of the reference, empty rows exactly 0,
    and the reference's own max_relative_error <= 1e-12 (bench.cpp:75-84)."""
    tol = row_tolerance(a, x)
    diff = np.abs(y - y_ref)
    bad = np.nonzero(diff > tol)[0]
    assert bad.size == 0, f"{what}: {bad.size} rows out of tolerance, first {bad[:5]} " \
                          f"y={y[bad[:5]]} ref={y_ref[bad[:5]]}"
    empty = np.diff(a.row_ptr) == 0
    assert np.all(y[empty] == 0.0), f"{what}: empty rows not zero"
    rel = diff / np.maximum(1.0, np.abs(y_ref))
    assert rel.max(initial=0.0) <= 1e-12, f"{what}: max relative error {rel.max()}"
