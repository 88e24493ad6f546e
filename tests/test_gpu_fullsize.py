"""Full-size parity: the BASELINE 1-GPU configurations (Laplacian 1000^2,
27-point stencil 200^3, R-MAT s24 permuted, mixed 2^23, R-MAT s27 permuted:
2.1G entries) converted and
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
WORKLOADS = ["lap5_1000", "st27_200", "mixed23", "rmat24", "rmat27"]


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_1503_05032_b200 import csr5
    return csr5


def row_of_nonzero(rp, m, g):
    """format.cpp:42-50 on the device: upper_bound(row_ptr, g) - 1, clamped."""
    return (torch.searchsorted(rp, g, right=True) - 1).clamp(0, max(m - 1, 0))


def expected_arrays(a, sigma, entries=True):
    """The reference's CSR5 arrays (omega = 32) from the CSR, in torch
    (col_idx / val only when `entries`; check_entries compares those in
    chunks for the 2G-entry matrix)."""
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
    del empty
    n_empty = E[rows[1:] + 1] - E[rows[:-1]]
    del E
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
    flags = torch.zeros(pc, 32, dtype=torch.int64, device=dev)
    for j in range(sigma):                                           # depth j at bit sigma-1-j
        flags |= hb[:, :, j].to(torch.int64) * int(weights[j])
    cnt = hb.sum(-1)
    yoff = cnt.cumsum(1) - cnt
    lane = torch.arange(32, device=dev).expand(pc, 32)
    idx = torch.where(cnt > 0, lane, torch.full_like(lane, 32))
    # next head-bearing lane strictly right of each lane
    nxt = torch.cat([idx[:, 1:], torch.full((pc, 1), 32, device=dev, dtype=idx.dtype)], 1)
    nxt = nxt.flip(1).cummin(1).values.flip(1)
    seg = torch.where(cnt > 0, torch.where(nxt < 32, nxt - lane - 1, 31 - lane), torch.zeros_like(lane))
    desc = (yoff << (5 + sigma)) | (seg.to(torch.int64) << sigma) | flags
    del flags, yoff, seg, nxt, idx, lane
    # empty_offset: heads of flagged complete tiles, in position order
    fl = flag[:pc]
    eo_cnt = torch.where(fl, cnt.sum(1), torch.zeros_like(fl, dtype=torch.int64))
    eo_ptr = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), eo_cnt.cumsum(0)])
    fl_idx = fl.nonzero().squeeze(1)
    if fl_idx.numel():
        sel = heads.view(pc, B)[fl].reshape(-1).nonzero().squeeze(1)
        tid = fl_idx[sel // B]
        pos = tid * B + sel % B
        eo = row_of_nonzero(rp, m, pos) - rows[tid]
        del sel, tid, pos
    else:
        eo = torch.zeros(0, dtype=torch.int64, device=dev)
    del heads, hb
    out = dict(tile_ptr=tile_ptr, tile_desc=desc.reshape(-1), eo_ptr=eo_ptr, eo=eo)
    if entries:
        # transposition of the complete tiles; the tail stays in CSR order
        col = a.col_idx.to(torch.int64)
        val = a.val
        out["col_idx"] = torch.cat([col[:pc * B].view(pc, 32, sigma).transpose(1, 2).reshape(-1),
                                    col[pc * B:]])
        out["val"] = torch.cat([val[:pc * B].view(pc, 32, sigma).transpose(1, 2).reshape(-1),
                                val[pc * B:]])
    return out


def check_entries(a, sigma, got_col, got_val, name, chunk_tiles=1 << 19):
    """The transposed col_idx / val (host exports) against the CSR, one chunk
    of tiles at a time on the device (format.hpp:76-88; the tail unchanged)."""
    B = 32 * sigma
    pc = a.nnz // B
    for t0 in range(0, pc, chunk_tiles):
        t1 = min(pc, t0 + chunk_tiles)
        lo, hi = t0 * B, t1 * B
        ec = a.col_idx[lo:hi].view(t1 - t0, 32, sigma).transpose(1, 2).reshape(-1).to(torch.int64)
        ev = a.val[lo:hi].view(t1 - t0, 32, sigma).transpose(1, 2).reshape(-1)
        gc = torch.from_numpy(got_col[lo:hi]).to(ec.device)
        gv = torch.from_numpy(got_val[lo:hi]).to(ev.device)
        assert torch.equal(gc, ec), f"{name}: col_idx differs in tiles [{t0}, {t1})"
        assert torch.equal(gv.view(torch.int64), ev.view(torch.int64)), \
            f"{name}: val differs in tiles [{t0}, {t1})"
    lo = pc * B
    assert np.array_equal(got_col[lo:], a.col_idx[lo:].to(torch.int64).cpu().numpy()), f"{name}: tail col"
    assert np.array_equal(got_val[lo:].view(np.int64), a.val[lo:].cpu().numpy().view(np.int64)), \
        f"{name}: tail val"


@pytest.mark.gpu
@pytest.mark.parametrize("name", WORKLOADS)
def test_fullsize(g, name):
    from paper_1503_05032_b200.synthetic import WORKLOADS as W, bench_x, make_matrix
    a = make_matrix(W[name], "cuda")
    sigma = g.select_sigma(a.nnz / a.m)
    free0 = torch.cuda.mem_get_info()[0]
    a5 = g.csr_to_csr5(a, g.TuningParams(sigma=sigma))
    print(f"{name}: nnz={a.nnz} sigma={sigma} handle device bytes {a5.info.device_bytes / 1e9:.2f} GB, "
          f"device memory in use after the build {(torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 1e9:.1f} GB "
          f"(build took {(free0 - torch.cuda.mem_get_info()[0]) / 1e9:.2f} GB)")
    try:
        # ---- arrays, bit for bit ----
        got = a5.export()
        exp = expected_arrays(a, sigma, entries=False)
        for f in ("tile_ptr", "tile_desc", "eo_ptr", "eo"):
            e = exp.pop(f)
            t = torch.from_numpy(got.pop(f).view(np.int64) if got[f].dtype == np.uint64 else got.pop(f))
            t = t.to(e.device)
            assert t.shape == e.shape, f"{name}: {f} shape {tuple(t.shape)} != {tuple(e.shape)}"
            bad = (t != e).nonzero()
            assert bad.numel() == 0, f"{name}: {f} differs at {bad[:8].flatten().tolist()}"
            del t, e
        del exp
        torch.cuda.empty_cache()
        check_entries(a, sigma, got["col_idx"], got["val"], name)
        del got
        # ---- round trip ----
        back = g.csr5_to_csr(a5, a.row_ptr)
        assert torch.equal(back.col_idx, a.col_idx), f"{name}: round-trip col_idx"
        assert torch.equal(back.val.view(torch.int64), a.val.view(torch.int64)), f"{name}: round-trip val"
        del back
        torch.cuda.empty_cache()
        # ---- y ----
        x = torch.as_tensor(bench_x(a.n)).cuda()
        y = g.spmv_csr5(a5, x)
        y2 = g.spmv_csr5(a5, 2.0 * x)
        assert torch.equal(y2, 2.0 * y), f"{name}: A(2x) != 2 Ax"
        del y2
        assert torch.equal(g.spmv_csr5(a5, x), y), f"{name}: rerun not bit-stable"
        # checksum of checksums: 1^T (A x) = (1^T A) x
        colsum = torch.zeros(a.n, dtype=torch.float64, device="cuda")
        absum = torch.zeros(a.n, dtype=torch.float64, device="cuda")
        step = 1 << 28
        for lo in range(0, a.nnz, step):
            ci = a.col_idx[lo:lo + step].long()
            colsum.index_add_(0, ci, a.val[lo:lo + step])
            absum.index_add_(0, ci, a.val[lo:lo + step].abs())
            del ci
        lhs, rhs = y.sum().item(), (colsum * x).sum().item()
        scale = (absum * x.abs()).sum().item()
        assert abs(lhs - rhs) <= 1e-12 * scale, f"{name}: checksum {lhs} vs {rhs}"
        del colsum, absum
        # every row against cuSPARSE, tolerance 1e-12 * max(1, nnz_i) * max_k |a_ik x_k|
        A = torch.sparse_csr_tensor(a.row_ptr, a.col_idx.long(), a.val, (a.m, a.n))
        y_ref = (A @ x.unsqueeze(1)).squeeze(1)
        del A
        torch.cuda.empty_cache()
        amax = torch.zeros(a.m, dtype=torch.float64, device="cuda")
        for lo in range(0, a.nnz, step):
            hi = min(a.nnz, lo + step)
            prod = (a.val[lo:hi] * x[a.col_idx[lo:hi].long()]).abs()
            rows = torch.searchsorted(a.row_ptr, torch.arange(lo, hi, device="cuda"), right=True) - 1
            amax.scatter_reduce_(0, rows, prod, reduce="amax")
            del prod, rows
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
