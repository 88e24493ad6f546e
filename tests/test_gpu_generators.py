"""The synthetic BASELINE matrices (synth_graph.cu) against a numpy
restatement of their definition, and the row-blocked R-MAT generator against
itself: any block split, any entry slice, the same CSR.

The restatement below is test code only: Graph500 R-MAT quadrant draws from
splitmix64 counters, the keyed relabelling, duplicate removal, values from the
key hash (synth_graph.cu header)."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
M64 = (1 << 64) - 1


def _splitmix(x):
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(M64)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def _permute(x, bits, key):
    mask = np.uint64((1 << bits) - 1)
    s1 = np.uint64(max((bits + 1) // 2, 1))
    for r in range(3):
        k = int(_splitmix(np.uint64(key + r)))
        x = (x * np.uint64(k | 1) + np.uint64(k >> 17)) & mask
        x = x ^ (x >> s1)
    return x & mask


def rmat_numpy(scale, edge_factor, seed, permute):
    """(row_ptr, col, val) of the R-MAT generator, restated."""
    with np.errstate(over="ignore"):
        E = edge_factor << scale
        e = np.arange(E, dtype=np.uint64)
        u = np.zeros(E, dtype=np.uint64)
        v = np.zeros(E, dtype=np.uint64)
        h = np.zeros(E, dtype=np.uint64)
        for lvl in range(scale):
            if lvl % 4 == 0:
                h = _splitmix(np.uint64(seed) ^ _splitmix(e * np.uint64(7) + np.uint64(lvl >> 2)))
            r = h & np.uint64(0xFFFF)
            h = h >> np.uint64(16)
            bu = (r >= 49807).astype(np.uint64)
            bv = (((r >= 37355) & (r < 49807)) | (r >= 62259)).astype(np.uint64)
            u = (u << np.uint64(1)) | bu
            v = (v << np.uint64(1)) | bv
        if permute:
            u = _permute(u, scale, seed * 31 + 1)
            v = _permute(v, scale, seed * 31 + 1)
        keys = np.unique((u << np.uint64(32)) | v)
        rows = (keys >> np.uint64(32)).astype(np.int64)
        col = (keys & np.uint64(0xFFFFFFFF)).astype(np.int32)
        hv = _splitmix(np.uint64(seed * 0x51ED27) + keys)
        val = 0.5 + (hv >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    m = 1 << scale
    row_ptr = np.zeros(m + 1, dtype=np.int64)
    np.add.at(row_ptr, rows + 1, 1)
    return np.cumsum(row_ptr), col, val


@pytest.mark.gpu
@pytest.mark.parametrize("permute", [True, False])
def test_rmat_matches_its_definition(permute):
    from paper_1503_05032_b200 import csr5
    a = csr5.rmat(12, 16, 3, permute, device="cuda")
    rp, col, val = rmat_numpy(12, 16, 3, permute)
    assert np.array_equal(a.row_ptr.cpu().numpy(), rp)
    assert np.array_equal(a.col_idx.cpu().numpy(), col)
    assert np.array_equal(a.val.cpu().numpy().view(np.uint64), val.view(np.uint64))


_DUMP = """
import sys, hashlib
sys.path.insert(0, {root!r})
from paper_1503_05032_b200 import csr5
g = csr5.rmat_generator(15, 16, 1, True, device="cuda")
rp, ci, va = g.fill()
h = hashlib.sha256()
for t in (rp, ci, va):
    h.update(t.cpu().numpy().tobytes())
print(g.nnz, h.hexdigest())
"""


@pytest.mark.gpu
def test_rmat_blocks_do_not_change_the_matrix():
    """2^19 raw edges cut into ~100 row blocks (CSR5G_GEN_BLOCK_EDGES) give the
    same CSR as one block."""
    out = []
    for env in ({}, {"CSR5G_GEN_BLOCK_EDGES": "5000"}):
        r = subprocess.run([sys.executable, "-c", _DUMP.format(root=ROOT)], capture_output=True,
                           text=True, env={**os.environ, **env}, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out.append(r.stdout.split()[-2:])
    assert out[0] == out[1]


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["rmat", "mixed"])
def test_generator_slices_equal_the_whole(kind):
    from paper_1503_05032_b200 import csr5
    g = (csr5.rmat_generator(14, 16, 5, True, device="cuda") if kind == "rmat" else
         csr5.mixed_generator(14, 0.4, 2, 3000, 1, 32, 5, device="cuda"))
    rp, ci, va = g.fill()
    nnz = g.nnz
    cuts = [0, 1, nnz // 3, nnz // 3 + 7, nnz - 1, nnz]
    for lo, hi in zip(cuts, cuts[1:]):
        r2, c2, v2 = g.fill(lo, hi, with_row_ptr=False)
        assert r2 is None
        assert bool((c2 == ci[lo:hi]).all()) and bool((v2 == va[lo:hi]).all()), (lo, hi)
    g.release()
    # canonical CSR: columns strictly increasing within each row
    rpn, cn = rp.cpu().numpy(), ci.cpu().numpy().astype(np.int64)
    starts = np.zeros(len(cn), dtype=bool)
    starts[rpn[:-1][rpn[:-1] < len(cn)]] = True
    assert np.all((np.diff(cn) > 0) | starts[1:])
