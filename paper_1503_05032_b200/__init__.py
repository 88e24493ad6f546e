"""B200-native CSR5 SpMV (Liu & Vinter, arXiv 1503.05032).

The compute path is libcsr5g.so (hand-written sm_100a CUDA behind the C ABI in
include/csr5g.h).  This package is the host-side mirror of the reference's
csr5:: API plus the multi-GPU driver; it has no CPU compute path.
"""
from ._lib import LIB_PATH, lib  # noqa: F401

__all__ = ["LIB_PATH", "lib"]
