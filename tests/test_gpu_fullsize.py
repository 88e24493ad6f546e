"""Full-size parity: the BASELINE 1-GPU configurations (Laplacian 1000^2,
27-point stencil 200^3, R-MAT s24 permuted, mixed 2^23) converted and
multiplied at their real sizes, checked through properties that do not need
the CPU oracle to finish on hundreds of millions of entries:

* every CSR5 array bit-exact against an independent torch restatement of the
  reference's construction run on the device (tile_ptr: format.cpp:52-82,
  bit_flag / y_offset / seg_offset / packing: format.cpp:84-121 and
  descriptor.cpp:38-62, empty_offset: format.cpp:123-136 + 213-224, the tile
  transposition: format.hpp:76-88);
* the round trip csr5_to_csr(csr_to_csr5(A)) == A bit for bit;
* y: exact power-of-two scaling (A(2x) == 2 Ax, deterministic mode),
  bit-stable reruns, the checksum identity 1^T (A x) = (1^T A) x, and every row
  against cuSPARSE within the tolerance of tests/_util.py.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
WORKLOADS = ["lap5_1000", "st27_200", "mixed23", "rmat24"]


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_1503_05032_b200 import csr5
    return csr5


def row_of_nonzero(rp, m, g):
    """format.cpp:42-50 on the device: upper_bound(row_ptr, g) - 1, clamped."""
    return (torch.searchsorted(rp, g, right=True) - 1).clamp(0, max(m - 1, 0))


def expected_arrays(a, sigma):
    """The reference's CSR5 arrays (omega = 32) from the CSR, in torch."""
    dev = a.row_ptr.device
    rp, m, nnz = a.row_ptr, a.m, a.nnz
    B = 32 * sigma
    p, pc = -(-nnz // B), nnz // B
    # tile_ptr: rows of tile starts, closing entry m - 1, empty-row flags over
    # the inclusive row span [rows[t], rows[t+1]]
    rows = row_of_nonzero(rp, m, torch.arange(p + 1, device=dev, dtype=torch.int64) * B)
    rows[p] = m - 1
    empty = (rp[1:] == rp[:-1]).to(torch.int64)
    E = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), empty.cumsum(0)])
    n_empty = E[rows[1:] + 1] - E[rows[:-1]]
    flag = torch.cat([n_empty > 0, torch.zeros(1, dtype=torch.bool, device=dev)])
    tile_ptr = rows | (flag.to(torch.int64) << 31)
    # bit flags: a row start inside a complete tile (empty runs collapse) plus
    # the forced bit 0 of every tile
    heads = torch.zeros(pc * B, dtype=torch.bool, device=dev)
    starts = rp[:-1]
    heads[starts[starts < pc * B]] = True
    heads[::B] = True
    hb = heads.view(pc, 32, sigma)
    weights = (1 << (sigma - 1 - torch.arange(sigma, device=dev, dtype=torch.int64)))
    flags = (hb.to(torch.int64) * weights).sum(-1)                       # depth j at bit sigma-1-j
    cnt = hb.sum(-1)
    yoff = cnt.cumsum(1) - cnt
    lane = torch.arange(32, device=dev).expand(pc, 32)
    idx = torch.where(cnt > 0, lane, torch.full_like(lane, 32))
    # next head-bearing lane strictly right of each lane
    nxt = torch.cat([idx[:, 1:], torch.full((pc, 1), 32, device=dev, dtype=idx.dtype)], 1)
    nxt = nxt.flip(1).cummin(1).values.flip(1)
    seg = torch.where(cnt > 0, torch.where(nxt < 32, nxt - lane - 1, 31 - lane), torch.zeros_like(lane))
    desc = (yoff << (5 + sigma)) | (seg.to(torch.int64) << sigma) | flags
    # empty_offset: heads of flagged complete tiles, in position order
    fl = flag[:pc]
    eo_cnt = torch.where(fl, cnt.sum(1), torch.zeros_like(fl, dtype=torch.int64))
    eo_ptr = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), eo_cnt.cumsum(0)])
    pos = heads.nonzero().squeeze(1)
    tid = pos // B
    sel = fl[tid]
    pos, tid = pos[sel], tid[sel]
    eo = row_of_nonzero(rp, m, pos) - rows[tid]
    # transposition of the complete tiles; the tail stays in CSR order
    col = a.col_idx.to(torch.int64)
    val = a.val
    col_t = torch.cat([col[:pc * B].view(pc, 32, sigma).transpose(1, 2).reshape(-1), col[pc * B:]])
    val_t = torch.cat([val[:pc * B].view(pc, 32, sigma).transpose(1, 2).reshape(-1), val[pc * B:]])
    return dict(tile_ptr=tile_ptr, tile_desc=desc.reshape(-1), eo_ptr=eo_ptr, eo=eo,
                col_idx=col_t, val=val_t)


@pytest.mark.gpu
@pytest.mark.parametrize("name", WORKLOADS)
def test_fullsize(g, name):
    from paper_1503_05032_b200.synthetic import WORKLOADS as W, bench_x, make_matrix
    a = make_matrix(W[name], "cuda")
    sigma = g.select_sigma(a.nnz / a.m)
    a5 = g.csr_to_csr5(a, g.TuningParams(sigma=sigma))
    try:
        # ---- arrays, bit for bit ----
        got = a5.export()
        exp = expected_arrays(a, sigma)
        for f in ("tile_ptr", "tile_desc", "eo_ptr", "eo", "col_idx", "val"):
            e = exp[f]
            t = torch.from_numpy(got[f].view(np.int64) if got[f].dtype == np.uint64 else got[f])
            t = t.to(e.device)
            assert t.shape == e.shape, f"{name}: {f} shape {tuple(t.shape)} != {tuple(e.shape)}"
            if f == "val":
                assert torch.equal(t.view(torch.int64), e.view(torch.int64)), f"{name}: {f}"
            else:
                bad = (t != e).nonzero()
                assert bad.numel() == 0, f"{name}: {f} differs at {bad[:8].flatten().tolist()}"
        del got, exp
        # ---- round trip ----
        back = g.csr5_to_csr(a5, a.row_ptr)
        assert torch.equal(back.col_idx, a.col_idx), f"{name}: round-trip col_idx"
        assert torch.equal(back.val.view(torch.int64), a.val.view(torch.int64)), f"{name}: round-trip val"
        del back
        # ---- y ----
        x = torch.as_tensor(bench_x(a.n)).cuda()
        y = g.spmv_csr5(a5, x)
        y2 = g.spmv_csr5(a5, 2.0 * x)
        assert torch.equal(y2, 2.0 * y), f"{name}: A(2x) != 2 Ax"
        assert torch.equal(g.spmv_csr5(a5, x), y), f"{name}: rerun not bit-stable"
        # checksum of checksums: 1^T (A x) = (1^T A) x
        colsum = torch.zeros(a.n, dtype=torch.float64, device="cuda")
        colsum.index_add_(0, a.col_idx.long(), a.val)
        absum = torch.zeros(a.n, dtype=torch.float64, device="cuda")
        absum.index_add_(0, a.col_idx.long(), a.val.abs())
        lhs, rhs = y.sum().item(), (colsum * x).sum().item()
        scale = (absum * x.abs()).sum().item()
        assert abs(lhs - rhs) <= 1e-12 * scale, f"{name}: checksum {lhs} vs {rhs}"
        # every row against cuSPARSE, tolerance 1e-12 * max(1, nnz_i) * max_k |a_ik x_k|
        A = torch.sparse_csr_tensor(a.row_ptr, a.col_idx.long(), a.val, (a.m, a.n))
        y_ref = (A @ x.unsqueeze(1)).squeeze(1)
        prod = (a.val * x[a.col_idx.long()]).abs()
        rows = torch.repeat_interleave(torch.arange(a.m, device="cuda"), a.row_ptr.diff())
        amax = torch.zeros(a.m, dtype=torch.float64, device="cuda").scatter_reduce_(
            0, rows, prod, reduce="amax")
        nnz_i = a.row_ptr.diff().clamp(min=1).to(torch.float64)
        tol = 1e-12 * nnz_i * amax
        assert bool(((y - y_ref).abs() <= tol).all()), f"{name}: y outside tolerance"
        assert bool((y[a.row_ptr.diff() == 0] == 0).all()), f"{name}: empty rows not exactly 0"
    finally:
        a5.release()
        torch.cuda.empty_cache()


@pytest.mark.parametrize("sigma", [1, 5, 16, 27, 48])
def test_torch_restatement_matches_oracle(orc, sigma):
    """CPU, no GPU: the torch restatement above equals the pinned oracle on the
    hard small shapes (tails, empty-row runs, flagged tiles, long rows), so its
    full-size agreement with the GPU is agreement with the reference."""
    from types import SimpleNamespace
    from tests.test_gpu_parity import hard_shapes
    for label, a in hard_shapes(orc):
        if a.m == 0 or a.nnz < 32 * sigma:
            continue
        t = SimpleNamespace(m=a.m, n=a.n, nnz=a.nnz,
                            row_ptr=torch.as_tensor(np.asarray(a.row_ptr, np.int64)),
                            col_idx=torch.as_tensor(np.asarray(a.col_idx, np.int32)),
                            val=torch.as_tensor(np.asarray(a.val, np.float64)))
        exp = expected_arrays(t, sigma)
        ref = orc.build(a, 32, sigma)
        for f in ("tile_ptr", "tile_desc", "eo_ptr", "eo", "col_idx", "val"):
            r = np.asarray(getattr(ref, f))
            e = exp[f].numpy()
            if r.dtype == np.uint64:
                r = r.view(np.int64)
            assert np.array_equal(e, r), f"{label} sigma={sigma}: {f}"
