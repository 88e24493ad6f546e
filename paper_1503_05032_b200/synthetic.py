"""Synthetic inputs for the benchmark (BASELINE.json configs).

x follows the reference harness convention (bench.cpp:103-105):
std::mt19937_64 seeded with x_seed = 1, x_i = 0.5 + (rng() >> 11) * 2^-53.
The engine is restated here in vectorised numpy (MT19937-64, Matsumoto &
Nishimura); tests check it against the oracle's scalar engine.

Matrices are generated on the device by libcsr5g (csr5g_stencil_fill).
"""
from __future__ import annotations

import numpy as np

_N, _M = 312, 156
_UPPER = np.uint64(0xFFFFFFFF80000000)
_LOWER = np.uint64(0x7FFFFFFF)
_A = np.uint64(0xB5026F5AA96619E9)


def _seed(seed: int) -> np.ndarray:
    mt = np.zeros(_N, dtype=np.uint64)
    mt[0] = seed
    f = 6364136223846793005
    for i in range(1, _N):
        prev = int(mt[i - 1])
        mt[i] = (f * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
    return mt


def _twist(mt: np.ndarray) -> None:
    def step(i0, i1, nxt, far):
        y = (mt[i0:i1] & _UPPER) | (nxt & _LOWER)
        v = far ^ (y >> np.uint64(1))
        v ^= np.where((y & np.uint64(1)) != 0, _A, np.uint64(0))
        mt[i0:i1] = v
    step(0, _M, mt[1:_M + 1].copy(), mt[_M:_N].copy())           # far = old values
    step(_M, _N - 1, mt[_M + 1:_N].copy(), mt[0:_N - 1 - _M].copy())  # far = new values
    step(_N - 1, _N, mt[0:1].copy(), mt[_M - 1:_M].copy())


def _temper(x: np.ndarray) -> np.ndarray:
    x = x ^ ((x >> np.uint64(29)) & np.uint64(0x5555555555555555))
    x = x ^ ((x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000))
    x = x ^ ((x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000))
    return x ^ (x >> np.uint64(43))


def mt19937_64(seed: int, count: int) -> np.ndarray:
    """First `count` outputs of std::mt19937_64(seed)."""
    mt = _seed(seed)
    out = np.empty(((count + _N - 1) // _N) * _N, dtype=np.uint64)
    for b in range(0, len(out), _N):
        _twist(mt)
        out[b:b + _N] = _temper(mt)
    return out[:count]


def bench_x_numpy(n: int, seed: int = 1) -> np.ndarray:
    """x as run_benchmark generates it (bench.cpp:103-105), restated in numpy
    (the cross-check of the native generator)."""
    r = mt19937_64(seed, n)
    return 0.5 + (r >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def bench_x(n: int, seed: int = 1) -> np.ndarray:
    """x as run_benchmark generates it (bench.cpp:103-105): std::mt19937_64 in
    libcsr5g (csr5g_bench_x, host code; no GPU needed)."""
    import ctypes

    from ._lib import check, lib
    x = np.empty(n, dtype=np.float64)
    check(lib().csr5g_bench_x(n, seed, x.ctypes.data_as(ctypes.c_void_p)))
    return x


WORKLOADS = {
    "st27_200": dict(gen="stencil", kind=1, a=200,
                     desc="3D 27-point stencil 200^3 (8M rows, 213.8M nnz), values 26/-1"),
    "lap5_1000": dict(gen="stencil", kind=0, a=1000,
                      desc="2D 5-point Laplacian 1000^2 (1M rows, 4.996M nnz), values 4/-1"),
    "rmat24": dict(gen="rmat", scale=24, edge_factor=16, permute=True, seed=1,
                   desc="R-MAT scale 24, edge factor 16, Graph500 .57/.19/.19/.05, dedup, "
                        "vertices permuted, values U[0.5,1.5)"),
    "rmat24_raw": dict(gen="rmat", scale=24, edge_factor=16, permute=False, seed=1,
                       desc="R-MAT scale 24, edge factor 16, Graph500, dedup, unpermuted"),
    "mixed23": dict(gen="mixed", log2_m=23, p_empty=0.4, n_long=4, long_len=1 << 20,
                    min_len=1, max_len=32, seed=1,
                    desc="mixed 2^23 x 2^23: 40% empty rows, 4 rows of 1,048,576 nnz, others "
                         "U[1,32] nnz, values U[0.5,1.5)"),
    "rmat25": dict(gen="rmat", scale=25, edge_factor=16, permute=True, seed=1,
                   desc="R-MAT scale 25, edge factor 16, Graph500, dedup, vertices permuted"),
    "rmat26": dict(gen="rmat", scale=26, edge_factor=16, permute=True, seed=1,
                   desc="R-MAT scale 26, edge factor 16, Graph500, dedup, vertices permuted"),
    "rmat27": dict(gen="rmat", scale=27, edge_factor=16, permute=True, seed=1,
                   desc="R-MAT scale 27, edge factor 16, Graph500, dedup, vertices permuted"),
}


def make_matrix(wl: dict, device="cuda"):
    """The workload's CSR, generated on the device by libcsr5g."""
    from . import csr5
    if wl["gen"] == "stencil" and wl.get("layers", wl["a"]) != wl["a"]:
        m, nnz, rp, ci, va = csr5.stencil_box(wl["kind"], wl["a"], wl["layers"], device=device)
        return csr5.CsrMatrix(m, m, rp, ci, va)
    return _make_matrix(wl, device)


def scaled_workload(wl: dict, world: int) -> dict:
    """Weak scaling: the global problem on `world` GPUs is `world` times the
    1-GPU problem -- stencils grow along the outermost axis (layers = a*world),
    graphs by log2(world) in scale (R-MAT s24 at 8 GPUs is s27, BASELINE
    config 5)."""
    w = dict(wl)
    if world == 1:
        return w
    if wl["gen"] == "stencil":
        w["layers"] = wl["a"] * world
    else:
        if world & (world - 1):
            raise ValueError("weak scaling of a graph workload needs a power-of-two GPU count")
        k = world.bit_length() - 1
        w["scale" if wl["gen"] == "rmat" else "log2_m"] += k
    w["desc"] = f"{wl['desc']}; x{world} for weak scaling"
    return w


class WorkloadMatrix:
    """A workload's global CSR for a multi-GPU rank: the full row_ptr on the
    device and `entries(lo, hi)` giving (col_idx, val) at global positions
    [lo, hi).  Every generator produces just the asked-for slice (graphs
    regenerate the row blocks that hold it, synth_graph.cu), so no rank ever
    holds the whole matrix."""

    def __init__(self, wl: dict, device="cuda"):
        from . import csr5
        self.wl, self.device = wl, device
        self.gen = None
        if wl["gen"] == "stencil":
            self.layers = wl.get("layers", wl["a"])
            self.m, self.nnz = csr5.stencil_box_size(wl["kind"], wl["a"], self.layers)
            _, _, self.row_ptr, _, _ = csr5.stencil_box(wl["kind"], wl["a"], self.layers, 0, 0,
                                                        device=device)
        else:
            self.gen = _generator(wl, device)
            self.m, self.nnz = self.gen.m, self.gen.nnz
            self.row_ptr = self.gen.fill(0, 0)[0]
        self.n = self.m

    def entries(self, lo: int, hi: int):
        from . import csr5
        if self.gen is not None:
            _, ci, va = self.gen.fill(lo, hi, with_row_ptr=False)
            return ci, va
        _, _, _, ci, va = csr5.stencil_box(self.wl["kind"], self.wl["a"], self.layers, lo, hi,
                                           device=self.device)
        return ci, va

    def drop(self):
        """Release the generator state (its device row_ptr copy)."""
        if self.gen is not None:
            self.gen.release()
            self.gen = None


def _generator(wl: dict, device="cuda"):
    from . import csr5
    if wl["gen"] == "rmat":
        return csr5.rmat_generator(wl["scale"], wl["edge_factor"], wl["seed"], wl["permute"],
                                   device=device)
    if wl["gen"] == "mixed":
        return csr5.mixed_generator(wl["log2_m"], wl["p_empty"], wl["n_long"], wl["long_len"],
                                    wl["min_len"], wl["max_len"], wl["seed"], device=device)
    raise ValueError(f"unknown generator {wl['gen']!r}")


def _make_matrix(wl: dict, device="cuda"):
    """The workload's CSR, generated on the device by libcsr5g."""
    from . import csr5
    if wl["gen"] == "stencil":
        return csr5.stencil(wl["kind"], wl["a"], device=device)
    if wl["gen"] == "rmat":
        return csr5.rmat(wl["scale"], wl["edge_factor"], wl["seed"], wl["permute"], device=device)
    if wl["gen"] == "mixed":
        return csr5.mixed(wl["log2_m"], wl["p_empty"], wl["n_long"], wl["long_len"],
                          wl["min_len"], wl["max_len"], wl["seed"], device=device)
    raise ValueError(f"unknown generator {wl['gen']!r}")
