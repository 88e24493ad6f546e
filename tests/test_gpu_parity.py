"""GPU parity: the CUDA converter and SpMV (through the C ABI) against the
reference's golden arrays and the pinned CPU oracle on identical inputs.

CSR5 arrays must be bit-exact; y within 1e-12 * max(1, nnz_i) * max_k|a_ik x_k|
of the reference with empty rows exactly 0 (tests/_util.py).
"""
import numpy as np
import pytest

from oracle.oracle import Csr
from tests import _shard_emulation as emu
from tests._util import assert_y_close

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FIELDS = ("tile_ptr", "tile_desc", "eo_ptr", "eo", "col_idx", "val")


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_1503_05032_b200 import csr5
    return csr5


def to_dev(g, a: Csr):
    return g.CsrMatrix.from_host(a.m, a.n, a.row_ptr, a.col_idx.astype(np.int32), a.val)


def gpu_build(g, a: Csr, sigma: int):
    return g.csr_to_csr5(to_dev(g, a), g.TuningParams(sigma=sigma))


def gpu_y(g, a5, x, mode="deterministic"):
    xd = torch.as_tensor(x).cuda()
    y = torch.full((a5.m,), float("nan"), dtype=torch.float64, device="cuda")
    g.spmv_csr5(a5, xd, y, mode=mode)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def compare_arrays(ex: dict, ref, what):
    for f in FIELDS:
        got, exp = ex[f], getattr(ref, f) if not isinstance(ref, dict) else ref[f]
        assert got.shape == exp.shape, f"{what}: {f} shape {got.shape} != {exp.shape}"
        assert np.array_equal(got, exp), f"{what}: {f} differs at {np.nonzero(got != exp)[0][:8]}"


def test_golden_w32(g, golden, orc):
    """Every golden case of the reference: arrays bit-exact, y in tolerance."""
    z, meta = golden
    for c in meta:
        k, mk = c["key"], c["mat"]
        a = Csr(c["m"], c["n"], z[f"{mk}_row_ptr"], z[f"{mk}_col_idx"].astype(np.int64), z[f"{mk}_val"])
        a5 = gpu_build(g, a, c["sigma"])
        i = a5.info
        assert (i.p, i.p_complete, i.tail_len, i.word_bits) == (c["p"], c["pc"], c["tail"], c["word_bits"])
        ex = a5.export()
        assert np.array_equal(ex["tile_ptr"], z[f"{k}_tile_ptr"]), (c, ex["tile_ptr"][:8], z[f"{k}_tile_ptr"][:8])
        assert np.array_equal(ex["tile_desc"], z[f"{k}_tile_desc"]), c
        assert np.array_equal(ex["eo_ptr"], z[f"{k}_eo_ptr"]), c
        assert np.array_equal(ex["eo"], z[f"{k}_eo"]), c
        assert np.array_equal(ex["col_idx"], z[f"{k}_tcol"].astype(np.int64)), c
        x = z[f"{mk}_x"]
        for mode in ("deterministic", "atomic"):
            y = gpu_y(g, a5, x, mode)
            assert_y_close(y, z[f"{k}_y"], a, x, f"{c['name']} sigma={c['sigma']} {mode}")
        a5.release()


def test_random_corpus_vs_oracle(g, orc):
    """acceptance.cpp:53-104 shape classes at omega=32 over sigma in [1, 48]."""
    rng = orc.rng(2024)
    for case in range(160):
        m, n = 1 + rng() % 400, 1 + rng() % 300
        kind = case % 4
        try:
            if kind == 3:
                a = rng.random_csr(m, n, rng() % 8000)
            else:
                a = orc.generate_synthetic(kind, m, n, min(m * n, rng() % 8000), rng(), 0.3)
        except Exception:
            a = rng.random_csr(m, n, rng() % 3000)
        sigma = 1 + rng() % 48
        x = rng.random_x(a.n)
        ref = orc.build(a, 32, sigma)
        a5 = gpu_build(g, a, sigma)
        compare_arrays(a5.export(), ref, f"case {case} m={m} n={n} nnz={a.nnz} sigma={sigma}")
        assert_y_close(gpu_y(g, a5, x), orc.spmv(a, x, 32, sigma), a, x, f"case {case}")
        a5.release()


def test_auto_sigma_matches_reference_rule(g, orc):
    rng = orc.rng(11)
    for npr in (1, 3, 5, 10, 17, 27, 40, 300):
        m = 200
        a = orc.generate_synthetic(0, m, 400, m * npr, rng())
        a5 = g.csr_to_csr5(to_dev(g, a))  # sigma = 0 -> auto
        assert a5.sigma == orc.select_sigma(npr)
        a5.release()


def hard_shapes(orc):
    rng = orc.rng(67)
    yield "m=1 wide row", orc.generate_synthetic(0, 1, 5000, 5000, 1)
    yield "n=1 tall column", orc.generate_synthetic(0, 3000, 1, 3000, 1)
    yield "all rows empty", orc.coo_to_csr([], [], [], 77, 7)
    yield "empty 0x0", Csr(0, 0, np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0))
    yield "one long row 30%", orc.generate_synthetic(1, 500, 6000, 18000, 7, 0.3)
    yield "exact multiple", orc.generate_synthetic(0, 64, 64, 64 * 48, 3)
    yield "singletons", orc.generate_synthetic(0, 4000, 4000, 4000, 4)
    # long runs of empty rows (> 32, exercising the cooperative zeroing path)
    rows = [3] * 50 + [4000] * 20 + [4001] * 700 + [9000] * 5
    cols = list(range(50)) + list(range(20)) + list(range(700)) + list(range(5))
    yield "long empty gaps", orc.coo_to_csr(rows, cols, np.linspace(0.5, 1.5, len(rows)), 12000, 800)
    # every other row empty, plus leading and trailing empties
    r2 = [5 + 2 * k for k in range(3000) for _ in range(3)]
    c2 = [j for k in range(3000) for j in range(3)]
    yield "alternating empties", orc.coo_to_csr(r2, c2, np.linspace(0.5, 1.5, len(r2)), 7000, 5)
    yield "random skew", orc.generate_synthetic(2, 5000, 3000, 40000, rng())
    # many heads per flagged tile over a wide row span (> 2048 rows: k_eo's
    # binary-search path) and a narrow one (its row_ptr scan path)
    for gap, name in ((97, "wide gappy heads"), (3, "narrow gappy heads")):
        r4 = [gap * k + 1 for k in range(2500) for _ in range(2)]
        c4 = [(7 * k + j) % 600 for k in range(2500) for j in range(2)]
        yield name, orc.coo_to_csr(r4, c4, np.linspace(0.5, 1.5, len(r4)), gap * 2500 + 5, 600)
    # regions of singleton rows (tiles with more heads than the shared-memory
    # slots: spill path) between regions of long rows (shared-memory path), so
    # both kinds of tile alternate inside one warp's tile range
    r3, c3, row = [], [], 0
    for blk in range(40):
        for _ in range(700):
            r3.append(row); c3.append((row * 7) % 900); row += 1
        for _ in range(30):
            r3.extend([row] * 45); c3.extend(range(blk, blk + 45)); row += 1
    yield "spill/shared alternation", orc.coo_to_csr(r3, c3, np.linspace(0.5, 1.5, len(r3)), row, 900)


@pytest.mark.parametrize("sigma", [1, 4, 5, 16, 17, 18, 27, 48])
def test_hard_shapes(g, orc, sigma):
    for name, a in hard_shapes(orc):
        x = orc.rng(9).random_x(a.n)
        ref = orc.build(a, 32, sigma)
        a5 = gpu_build(g, a, sigma)
        compare_arrays(a5.export(), ref, f"{name} sigma={sigma}")
        if a.m:
            assert_y_close(gpu_y(g, a5, x), orc.spmv(a, x, 32, sigma), a, x, f"{name} sigma={sigma}")
            assert_y_close(gpu_y(g, a5, x, "atomic"), orc.dense_spmv(a, x), a, x, f"{name} atomic")
        a5.release()


def test_deterministic_is_bitwise_stable(g, orc):
    a = orc.generate_synthetic(2, 20000, 5000, 400000, 77)
    a5 = gpu_build(g, a, 16)
    x = orc.rng(78).random_x(a.n)
    y0 = gpu_y(g, a5, x)
    for _ in range(5):
        assert np.array_equal(gpu_y(g, a5, x), y0)


def test_power_of_two_scaling_exact(g, orc):  # test_spmv.cpp:232-242
    rng = orc.rng(61)
    a = rng.random_csr(400, 400, 9000)
    x = rng.random_x(400)
    a5 = gpu_build(g, a, 8)
    assert np.array_equal(gpu_y(g, a5, 8.0 * x), 8.0 * gpu_y(g, a5, x))


def test_roundtrip(g, orc):  # format.cpp:254-265, acceptance criterion 2
    rng = orc.rng(23)
    for sigma in (1, 2, 4, 12, 16, 33):
        a = rng.random_csr(300, 200, 9000)
        d = to_dev(g, a)
        a5 = g.csr_to_csr5(d, g.TuningParams(sigma=sigma))
        back = g.csr5_to_csr(a5, d.row_ptr)
        assert np.array_equal(back.col_idx.cpu().numpy(), a.col_idx.astype(np.int32))
        assert np.array_equal(back.val.cpu().numpy(), a.val)


def test_errors_mirror_reference(g, orc):
    a = orc.coo_to_csr([0], [0], [1.0], 2, 3)
    d = to_dev(g, a)
    with pytest.raises(ValueError, match="omega must be 32"):
        g.csr_to_csr5(d, g.TuningParams(omega=4, sigma=16))
    with pytest.raises(ValueError, match="omega \\* sigma must be >= 2"):
        g.csr_to_csr5(d, g.TuningParams(omega=1, sigma=1))
    with pytest.raises(ValueError, match="smaller sigma"):
        g.csr_to_csr5(d, g.TuningParams(sigma=49))
    with pytest.raises(ValueError, match="r <= s <= t"):
        g.csr_to_csr5(d, g.TuningParams(sigma=4, r=10, s=5))
    a5 = g.csr_to_csr5(d, g.TuningParams(sigma=4))
    with pytest.raises(ValueError, match="spmv: x has length 2, expected 3"):
        g.spmv_csr5(a5, torch.ones(2, dtype=torch.float64, device="cuda"))


def test_stencil_generator(g, orc):
    for kind, a_, nnz_fn in ((0, 13, lambda s: 5 * s * s - 4 * s), (1, 7, lambda s: (3 * s - 2) ** 3)):
        d = g.stencil(kind, a_)
        rp = d.row_ptr.cpu().numpy()
        ci = d.col_idx.cpu().numpy().astype(np.int64)
        va = d.val.cpu().numpy()
        assert rp[-1] == nnz_fn(a_)
        # canonical and symmetric, diagonal dominant values
        for r in range(d.m):
            cols = ci[rp[r]:rp[r + 1]]
            assert np.all(np.diff(cols) > 0)
            assert r in cols
        A = np.zeros((d.m, d.m))
        for r in range(d.m):
            A[r, ci[rp[r]:rp[r + 1]]] = va[rp[r]:rp[r + 1]]
        assert np.array_equal(A, A.T)


def test_shards_concatenate_and_fix_up(g, orc):
    """Multi-GPU partition on one device, run shard by shard: the shard arrays
    are slices of the single-device arrays and boundary fix-ups reproduce y."""
    from paper_1503_05032_b200 import mg
    rng = orc.rng(5)
    cases = [orc.generate_synthetic(1, 300, 30000, 60000, 3, 0.5),  # one long row
             orc.generate_synthetic(2, 5000, 4000, 120000, 4),
             orc.generate_synthetic(0, 2000, 2000, 54000, 5)]
    for a in cases:
        x = rng.random_x(a.n)
        sigma = orc.select_sigma(a.nnz / a.m)
        full = orc.build(a, 32, sigma)
        y_ref = orc.spmv(a, x, 32, sigma)
        for world in (2, 3, 5, 8):
            y = emu.emulate_shards_on_one_device(a, x, sigma, world)
            assert_y_close(y, y_ref, a, x, f"world={world}")
            ex = emu.emulate_shard_exports(a, sigma, world)
            for f in ("tile_desc", "eo", "col_idx", "val"):
                assert np.array_equal(np.concatenate([e[f] for e in ex]), getattr(full, f)), f
            tp = np.concatenate([e["tile_ptr"][:-1] for e in ex[:-1]] + [ex[-1]["tile_ptr"]])
            assert np.array_equal(tp, full.tile_ptr)


def test_p2p_exchange_on_one_device(g, orc):
    """The NVLink P2P boundary exchange (p2p.cu) with all shards in one process:
    partials stored into the owners' mailboxes by the SpMV kernel,
    flags/acks over several calls (epochs), y equal to the collective form and
    within tolerance of the oracle, no protocol errors."""
    from paper_1503_05032_b200 import mg
    rng = orc.rng(9)
    cases = [orc.generate_synthetic(1, 300, 30000, 60000, 3, 0.5),  # one long row
             orc.generate_synthetic(2, 5000, 4000, 120000, 4),
             orc.generate_synthetic(0, 2000, 2000, 54000, 5)]
    for a in cases:
        sigma = orc.select_sigma(a.nnz / a.m)
        xs = [rng.random_x(a.n) for _ in range(3)]
        for world in (2, 3, 8, 16):
            ys, errs, dest, senders = emu.emulate_p2p_on_one_device(a, xs, sigma, world)
            assert errs == [0] * len(errs), (world, errs)
            for x, y in zip(xs, ys):
                assert_y_close(y, orc.spmv(a, x, 32, sigma), a, x, f"p2p world={world}")
                y_coll = emu.emulate_shards_on_one_device(a, x, sigma, world)
                assert np.array_equal(y, y_coll), f"p2p != collective, world={world}"
        if a.m == 300:  # the long row lies in one shard (mg.plan_tiles moved the edges off
            # it), so every row split by an edge has one partial per side
            assert max(se - sb for sb, se in senders) <= 1, senders


def test_p2p_fused_iterative_on_one_device(g, orc):
    """Fused iterative mode (csr5g_mg_iter): every final y value also stored
    into each peer's next-x buffer by the kernels producing it.  After every
    iteration all shards hold the same x_{k+1} bit for bit, equal to the
    sharded SpMV of x_k (collective form) and within tolerance of the oracle."""
    from paper_1503_05032_b200 import mg
    rng = orc.rng(11)
    cases = [orc.generate_synthetic(1, 30000, 30000, 60000, 3, 0.3),  # a long row spans shards
             orc.generate_synthetic(2, 5000, 5000, 120000, 4),
             orc.generate_synthetic(0, 2000, 2000, 54000, 5)]
    for a in cases:
        sigma = orc.select_sigma(a.nnz / a.m)
        x0 = rng.random_x(a.n) / 32.0
        for world in (2, 3, 8):
            outs, errs = emu.emulate_p2p_iterative_on_one_device(a, x0, sigma, world, 3)
            assert errs == [0] * len(errs), (world, errs)
            x = x0
            for it, bufs in enumerate(outs):
                for b in bufs[1:]:
                    assert np.array_equal(b, bufs[0]), f"world={world} it={it}: shards disagree"
                y_coll = emu.emulate_shards_on_one_device(a, x, sigma, world)
                assert np.array_equal(bufs[0], y_coll), f"world={world} it={it}: != sharded SpMV"
                assert_y_close(bufs[0], orc.spmv(a, x, 32, sigma), a, x, f"iter {it} world={world}")
                x = bufs[0]


def test_two_plans_of_one_kernel(g, orc):
    """Two live handles whose plans differ for the same sigma-specialised
    kernel (banded: local gathers, large shared-memory ring; random columns:
    random plan, smaller ring): each SpMV launches with its own plan, in any
    order (kernel attributes follow the launch, not the last build)."""
    rng = np.random.default_rng(3)
    m = n = 20000
    rows = np.repeat(np.arange(m), 27)
    band = (rows + np.tile(np.arange(27), m)) % n
    rnd = rng.integers(0, n, rows.size)
    mats = []
    for cols in (band, rnd):
        a = orc.coo_to_csr(rows.tolist(), cols.tolist(), np.linspace(0.5, 1.5, rows.size), m, n)
        mats.append(a)
    hs = [gpu_build(g, a, 27) for a in mats]
    assert hs[0].info.smem_bytes != hs[1].info.smem_bytes, "plans should differ"
    x = orc.rng(4).random_x(n)
    for order in ((0, 1), (1, 0), (0, 0, 1, 1, 0)):
        for i in order:
            assert_y_close(gpu_y(g, hs[i], x), orc.spmv(mats[i], x, 32, 27), mats[i], x, f"plan {i}")
    for h in hs:
        h.release()


def test_concurrent_streams_one_handle(g, orc):
    """One handle, SpMVs in flight on several streams at once with different x
    (the reference allows concurrent spmv_csr5 calls on one matrix): every y
    equals the single-stream result bit for bit (deterministic mode)."""
    a = orc.generate_synthetic(2, 20000, 15000, 600000, 8)
    sigma = orc.select_sigma(a.nnz / a.m)
    rng = orc.rng(12)
    xs = [rng.random_x(a.n) for _ in range(4)]
    # the build is synchronous: a stream that never saw it can use the handle at once
    fresh = torch.cuda.Stream()
    x0 = torch.as_tensor(xs[0]).cuda()
    d = to_dev(g, a)
    torch.cuda.synchronize()
    a5 = g.csr_to_csr5(d, g.TuningParams(sigma=sigma))
    with torch.cuda.stream(fresh):
        y0 = g.spmv_csr5(a5, x0, stream=fresh)
    fresh.synchronize()
    assert_y_close(y0.cpu().numpy(), orc.spmv(a, xs[0], 32, sigma), a, xs[0], "fresh stream")
    ref = [gpu_y(g, a5, x) for x in xs]
    streams = [torch.cuda.Stream() for _ in xs]
    xd = [torch.as_tensor(x).cuda() for x in xs]
    torch.cuda.synchronize()
    for rep in range(3):
        ys = [torch.full((a.m,), float("nan"), dtype=torch.float64, device="cuda") for _ in xs]
        torch.cuda.synchronize()
        for s, x, y in zip(streams, xd, ys):
            with torch.cuda.stream(s):
                for _ in range(3):  # several launches per stream, interleaved across streams
                    g.spmv_csr5(a5, x, y, stream=s)
        torch.cuda.synchronize()
        for i, y in enumerate(ys):
            assert np.array_equal(y.cpu().numpy(), ref[i]), f"stream {i} rep {rep}"
    a5.release()


def test_cuda_graph_capture(g, orc):
    """One SpMV is one kernel (calibration inside it), so a solver loop can be
    captured into a CUDA graph and replayed: y_{k+1} = A y_k for 4 steps per
    replay, new x each replay, results bit-equal to eager calls."""
    a = orc.generate_synthetic(0, 6000, 6000, 150000, 21)
    sigma = orc.select_sigma(a.nnz / a.m)
    a5 = gpu_build(g, a, sigma)
    s = torch.cuda.Stream()
    bufs = [torch.zeros(a.n, dtype=torch.float64, device="cuda") for _ in range(2)]
    with torch.cuda.stream(s):  # warm-up: the stream's scratch exists before capture
        g.spmv_csr5(a5, bufs[0], bufs[1], stream=s)
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for k in range(4):
            g.spmv_csr5(a5, bufs[k & 1], bufs[(k + 1) & 1])
    rng = orc.rng(22)
    for rep in range(3):
        x0 = rng.random_x(a.n) / 8.0
        bufs[0].copy_(torch.as_tensor(x0))
        graph.replay()
        torch.cuda.synchronize()
        got = bufs[0].cpu().numpy()  # after 4 steps the result is back in bufs[0]
        x = torch.as_tensor(x0).cuda()
        for _ in range(4):
            x = g.spmv_csr5(a5, x)
        assert np.array_equal(got, x.cpu().numpy()), f"replay {rep}"
    del graph
    a5.release()


def test_kernel_variants(g, orc):
    """The plan's kernel variants on matrices made for them, each against the
    oracle: NF (no flagged tile, heads fit the slots, sigma <= 8) on a 2D
    5-point Laplacian and a banded matrix, the general kernel on the same
    Laplacian with empty rows spliced in (flagged tiles), VR on random columns."""
    from oracle.oracle import stencil
    lap = stencil(orc, 0, 40, 40)  # 1600 rows, sigma 5
    rows = np.repeat(np.arange(3000), 7)
    band = orc.coo_to_csr(rows.tolist(), ((rows + np.tile(np.arange(7), 3000)) % 3000).tolist(),
                          np.linspace(0.5, 1.5, rows.size), 3000, 3000)
    r2 = [r + r // 50 for r in lap_rows(lap)]  # every 50th row becomes empty
    gap = orc.coo_to_csr(r2, lap.col_idx.tolist(), lap.val.tolist(), max(r2) + 1, lap.n)
    rr = np.repeat(np.arange(40000), 8)
    rc = np.random.default_rng(31).integers(0, 400000, rr.size)
    rnd = orc.coo_to_csr(rr.tolist(), rc.tolist(), np.linspace(0.5, 1.5, rr.size), 40000, 400000)
    for name, a, want in (("laplacian", lap, 2), ("band", band, 2), ("gaps", gap, 0),
                          ("random", rnd, 1)):
        sigma = orc.select_sigma(a.nnz / a.m)
        a5 = gpu_build(g, a, sigma)
        assert a5.info.kernel_variant == want, (name, sigma, a5.info.kernel_variant)
        x = orc.rng(5).random_x(a.n)
        assert_y_close(gpu_y(g, a5, x), orc.spmv(a, x, 32, sigma), a, x, name)
        compare_arrays(a5.export(), orc.build(a, 32, sigma), name)
        a5.release()


def lap_rows(a):
    return np.repeat(np.arange(a.m), np.diff(np.asarray(a.row_ptr))).tolist()


def test_host_vector_paths(g, orc):
    """csr5g_spmv_host and the pipelined csr5g_spmv_host_batch (pinned and
    pageable host vectors, batches longer than the two buffer pairs, a second
    batch reusing the handle's pipeline) give the device path's y."""
    rng = orc.rng(11)
    a = orc.generate_synthetic(2, 4000, 3000, 90000, 9)
    sigma = orc.select_sigma(a.nnz / a.m)
    a5 = gpu_build(g, a, sigma)
    xs = [rng.random_x(a.n) for _ in range(5)]
    ys_dev = [gpu_y(g, a5, x) for x in xs]
    for x, yd in zip(xs, ys_dev):
        assert_y_close(yd, orc.spmv(a, x, 32, sigma), a, x, "device path")
        assert np.array_equal(g.spmv_host(a5, x), yd)  # deterministic mode: bit-stable
    for pinned in (True, False):
        for count in (1, 2, 5):
            hx = [torch.as_tensor(x) for x in xs[:count]]
            hy = [torch.full((a.m,), float("nan"), dtype=torch.float64) for _ in range(count)]
            if pinned:
                hx = [t.pin_memory() for t in hx]
                hy = [t.pin_memory() for t in hy]
            g.spmv_host_batch(a5, hx, hy)
            torch.cuda.current_stream().synchronize()
            for k in range(count):
                assert np.array_equal(hy[k].numpy(), ys_dev[k]), (pinned, count, k)
    with pytest.raises(ValueError, match="2 x vectors but 1 y"):
        g.spmv_host_batch(a5, xs[:2], [np.empty(a.m)])
    with pytest.raises(ValueError, match="length"):
        g.spmv_host_batch(a5, [np.empty(a.n + 1)], [np.empty(a.m)])
    a5.release()


def test_skewed_tile_work(g, orc):
    """Tiles of long rows followed by tiles spanning thousands of short and
    empty rows: the warps' tile ranges are split by work (k_warp_bounds), not
    by count.  Arrays and y against the oracle, random-gather and local plans."""
    rng = np.random.default_rng(8)
    for n_long, n_short, n in ((2000, 300000, 50000), (300, 120000, 2000000)):
        lens = np.concatenate([rng.integers(200, 400, n_long),
                               rng.integers(0, 2, n_short) * rng.integers(1, 3, n_short)])
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        cols = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) for k in lens])
        a = Csr(len(lens), n, rp, cols.astype(np.int64), rng.uniform(0.5, 1.5, len(cols)))
        x = orc.rng(4).random_x(n)
        for sigma in (16, 32):
            a5 = gpu_build(g, a, sigma)
            compare_arrays(a5.export(), orc.build(a, 32, sigma), f"skew sigma={sigma}")
            for mode in ("deterministic", "atomic"):
                assert_y_close(gpu_y(g, a5, x, mode), orc.spmv(a, x, 32, sigma), a, x,
                               f"skew sigma={sigma} {mode}")
            a5.release()


@pytest.mark.parametrize("sigma", [1, 5, 16, 24])
def test_gather_orders_give_identical_y(g, orc, sigma, monkeypatch):
    """The VR kernel's x-gather paths (x_mode 1: lane-per-column order, the
    default below 3x L2; 8: CSR order through the shared-memory exchange with a
    64-byte L2 prefetch, the plan for x several times the L2; 5, 7: the other
    two combinations) fetch the same x values into the same depth-loop slots,
    so y is bit-identical across them and within tolerance of the oracle; the
    arrays stay bit-exact."""
    rng = np.random.default_rng(sigma)
    m = 6000
    lens = rng.integers(0, 2 * sigma + 1, m)
    lens[rng.integers(0, m, 3)] = 900  # rows spanning tiles
    rows = np.repeat(np.arange(m), lens)
    cols = rng.integers(0, 500000, rows.size)
    a = orc.coo_to_csr(rows.tolist(), cols.tolist(), rng.uniform(0.5, 1.5, rows.size).tolist(),
                       m, 500000)
    x = orc.rng(3).random_x(a.n)
    ref = orc.build(a, 32, sigma)
    ys = {}
    for mode in ("1", "5", "7", "8"):
        monkeypatch.setenv("CSR5G_XMODE", mode)
        a5 = gpu_build(g, a, sigma)
        assert a5.info.kernel_variant == 1 and a5.info.x_mode == int(mode), (mode, a5.info.x_mode)
        ys[mode] = gpu_y(g, a5, x)
        compare_arrays(a5.export(), ref, f"x_mode {mode}")
        a5.release()
    for mode, y in ys.items():
        assert np.array_equal(y.view(np.int64), ys["1"].view(np.int64)), mode
    assert_y_close(ys["8"], orc.spmv(a, x, 32, sigma), a, x, "csr-order gathers")


def test_nf_kernel_multi_tile_warps(g, orc, monkeypatch):
    """The NF kernel's lean write-back and run merge (every NF tile has >= 2
    heads; only the last head carries over) with many tiles per warp: a
    200^2 Laplacian (1,245 tiles) on 1, 2 and 5 warps per CTA -- y against
    the oracle, and bit-identical across the warp splits (partition-invariant
    deterministic mode)."""
    from oracle.oracle import stencil
    a = stencil(orc, 0, 200, 200)
    sigma = orc.select_sigma(a.nnz / a.m)
    x = orc.rng(8).random_x(a.n)
    y_ref = orc.spmv(a, x, 32, sigma)
    ys = []
    for nw in (1, 2, 5):
        monkeypatch.setenv("CSR5G_NW", str(nw))
        a5 = gpu_build(g, a, sigma)
        assert a5.info.kernel_variant == 2 and a5.info.warps_per_cta == nw
        y = gpu_y(g, a5, x)
        assert_y_close(y, y_ref, a, x, f"nf nw={nw}")
        ys.append(y)
        a5.release()
    for y in ys[1:]:
        assert np.array_equal(y.view(np.int64), ys[0].view(np.int64))
    # the two-tiles-per-iteration NF kernel (spmv_nf2.cuh, opt-in) gives the
    # same bits
    monkeypatch.delenv("CSR5G_NW")
    monkeypatch.setenv("CSR5G_NF2", "1")
    a5 = gpu_build(g, a, sigma)
    y2 = gpu_y(g, a5, x)
    a5.release()
    assert np.array_equal(y2.view(np.int64), ys[0].view(np.int64))
