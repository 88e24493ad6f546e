"""Maximum supported sizes: m = 2^31 - 1 rows (the largest row index a u32
tile pointer with its MSB flag can hold) and n = 2^31 - 1 columns (the largest
int32 col_idx).  CSR5 arrays bit-exact against the oracle; y checked on the
rows that hold entries, every other row exactly 0.  Needs ~70 GB of device
and ~70 GB of host memory; skipped where either is missing."""
import os

import numpy as np
import pytest

from oracle.oracle import Csr

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

M = N = 2**31 - 1


def _mem_ok(dev_gb, host_gb):
    if not torch.cuda.is_available():
        return False
    free, _ = torch.cuda.mem_get_info()
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 0
    return free > dev_gb * 1e9 and avail > host_gb * 1e9


def _rows_spec(rng):
    """(row, length) pairs in increasing row order: leading empty rows, short
    rows, a long row crossing tiles, a sparse run inside a 10^9-row empty
    range, and the last rows of the matrix."""
    spec = [(r, 3) for r in range(7, 207)]
    spec += [(1_000_000_000, 5000)]
    spec += [(r, 1) for r in range(1_500_000_000, 1_500_002_000, 3)]
    spec += [(r, 2) for r in range(M - 300, M)]
    return spec


def _entries(rng, spec, ncols, col_hi):
    cols, vals = [], []
    for _, k in spec:
        c = np.sort(rng.choice(ncols, size=k, replace=False))
        c = np.where(c % 2 == 0, c, col_hi - c)  # both ends of the column range
        cols.append(np.unique(c))
        vals.append(rng.uniform(0.5, 1.5, len(cols[-1])))
    return cols, vals


@pytest.mark.skipif(not _mem_ok(75, 75), reason="needs ~75 GB device + host memory")
def test_max_rows(orc):
    from paper_1503_05032_b200 import csr5
    rng = np.random.default_rng(1)
    spec = _rows_spec(rng)
    cols, vals = _entries(rng, spec, 6000, 5999)
    lens = [len(c) for c in cols]
    rp = np.empty(M + 1, np.int64)
    rp[:spec[0][0] + 1] = 0
    acc = 0
    for i, (r, _) in enumerate(spec):
        acc += lens[i]
        nxt = spec[i + 1][0] if i + 1 < len(spec) else M
        rp[r + 1:nxt + 1] = acc
    a = Csr(M, 6000, rp, np.concatenate(cols).astype(np.int64), np.concatenate(vals))
    x = orc.rng(3).random_x(a.n)
    for sigma in (16, 20):
        ref = orc.build(a, 32, sigma)
        d = csr5.CsrMatrix(M, a.n, torch.from_numpy(rp).cuda(),
                           torch.from_numpy(a.col_idx.astype(np.int32)).cuda(),
                           torch.from_numpy(a.val).cuda())
        a5 = csr5.csr_to_csr5(d, csr5.TuningParams(sigma=sigma))
        ex = a5.export()
        for f in ("tile_ptr", "tile_desc", "eo_ptr", "eo", "col_idx", "val"):
            assert np.array_equal(ex[f], getattr(ref, f)), (sigma, f)
        assert int(ex["tile_ptr"][-1]) & 0x7FFFFFFF == M - 1
        y = csr5.spmv_csr5(a5, torch.as_tensor(x).cuda())
        del d
        a5.release()
        nz_rows = np.array([r for r, _ in spec], np.int64)
        got = y[torch.from_numpy(nz_rows).cuda()].cpu().numpy()
        assert int(torch.count_nonzero(y)) == len(nz_rows)
        del y
        torch.cuda.empty_cache()
        exp = np.array([np.dot(v, x[c]) for c, v in zip(cols, vals)])
        assert np.max(np.abs(got - exp) / np.maximum(1.0, np.abs(exp))) <= 1e-12, sigma


@pytest.mark.skipif(not _mem_ok(40, 20), reason="needs ~40 GB device memory")
def test_max_columns(orc):
    from paper_1503_05032_b200 import csr5
    rng = np.random.default_rng(2)
    m = 4000
    rows = [(r, int(rng.integers(0, 60))) for r in range(m)]
    cols, vals = _entries(rng, rows, 1 << 20, N - 1)
    cols[0], vals[0] = np.array([0, 12345, N - 1]), np.array([0.75, 1.25, 1.5])  # both ends
    lens = np.array([len(c) for c in cols])
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    a = Csr(m, N, rp, np.concatenate(cols).astype(np.int64), np.concatenate(vals))
    assert a.col_idx.max() == N - 1 and a.col_idx.min() == 0
    sigma = orc.select_sigma(a.nnz / m)
    ref = orc.build(a, 32, sigma)
    d = csr5.CsrMatrix.from_host(m, N, rp, a.col_idx.astype(np.int32), a.val)
    a5 = csr5.csr_to_csr5(d, csr5.TuningParams(sigma=sigma))
    ex = a5.export()
    for f in ("tile_ptr", "tile_desc", "eo_ptr", "eo", "col_idx", "val"):
        assert np.array_equal(ex[f], getattr(ref, f)), f
    # x_j = 1 + (j mod 1000) / 1000 over all 2^31 - 1 columns, built in chunks
    x = torch.empty(N, dtype=torch.float64, device="cuda")
    step = 1 << 28
    for lo in range(0, N, step):
        hi = min(N, lo + step)
        x[lo:hi] = 1.0 + (torch.arange(lo, hi, device="cuda") % 1000).double() / 1000.0
    y = csr5.spmv_csr5(a5, x).cpu().numpy()
    xc = 1.0 + (a.col_idx % 1000) / 1000.0
    exp = np.array([np.dot(a.val[rp[i]:rp[i + 1]], xc[rp[i]:rp[i + 1]]) for i in range(m)])
    assert np.max(np.abs(y - exp) / np.maximum(1.0, np.abs(exp))) <= 1e-12
    assert np.all(y[lens == 0] == 0.0)
    a5.release()
    with pytest.raises(IndexError, match="2\\^31"):
        csr5.csr_to_csr5(csr5.CsrMatrix.from_host(1, N + 1, [0, 0], np.zeros(0, np.int32),
                                                  np.zeros(0)))
