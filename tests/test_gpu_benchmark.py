"""The device run_benchmark harness (paper_1503_05032_b200.benchmark): the
plain-CSR baselines' y against the oracle, the validation guard, the
iteration-scenario fields and the CSV, mirroring the reference's own
test_bench.cpp checks."""
import numpy as np
import pytest

from tests._util import assert_y_close

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_1503_05032_b200 import benchmark, csr5
    return csr5, benchmark


def test_csr_baselines_match_oracle(g, orc):
    csr5, _ = g
    rng = orc.rng(21)
    from oracle.oracle import Csr
    cases = [orc.generate_synthetic(2, 3000, 2500, 40000, 3),
             orc.generate_synthetic(1, 200, 20000, 30000, 4, 0.5),
             orc.generate_synthetic(0, 1000, 1000, 3000, 5),
             Csr(5, 4, np.zeros(6, np.int64), np.zeros(0, np.int64), np.zeros(0))]
    for a in cases:
        x = rng.random_x(a.n)
        y_ref = orc.dense_spmv(a, x)
        d = csr5.CsrMatrix.from_host(a.m, a.n, a.row_ptr, a.col_idx.astype(np.int32), a.val)
        xd = torch.as_tensor(x).cuda()
        for k in ("csr-scalar", "csr-segsum"):
            y = csr5.spmv_csr(d, xd, kernel=k).cpu().numpy()
            assert_y_close(y, y_ref, a, x, k)
    with pytest.raises(ValueError, match="unknown kernel 'csr-vector'"):
        csr5.spmv_csr(d, xd, kernel="csr-vector")


def test_run_benchmark(g):
    csr5, B = g
    a = csr5.stencil(1, 24)
    cfg = B.BenchConfig(runs=3, inner_iters=5, warmup=2)
    rep = B.run_benchmark(a, "st27_24", cfg)
    assert (rep.matrix, rep.m, rep.n, rep.nnz) == ("st27_24", a.m, a.n, a.nnz)
    assert [k.kernel for k in rep.kernels] == ["csr-scalar", "csr-segsum", "csr5"]
    base = rep.kernels[0]
    for k in rep.kernels:
        assert len(k.sample_ms) == 3 and k.best_ms == min(k.sample_ms) > 0
        assert k.gflops == pytest.approx(2 * a.nnz / (k.best_ms * 1e6))
        assert k.conv_ms == 0.0 if k.kernel != "csr5" else k.conv_ms > 0.0
        assert k.speedup_n50 == B.iteration_speedup(base.best_ms, k.conv_ms, k.best_ms, 50)
        assert k.speedup_n500 == B.iteration_speedup(base.best_ms, k.conv_ms, k.best_ms, 500)
    assert base.speedup_n50 == pytest.approx(1.0)
    csv = B.emit_csv(rep).splitlines()
    assert csv[0] == B.CSV_HEADER and len(csv) == 4 and csv[3].startswith("st27_24,")
    # without csr-scalar the first kernel is the baseline (bench.cpp:166-169)
    rep2 = B.run_benchmark(a, "s", B.BenchConfig(kernels=B.parse_kernel_list("csr5,csr-segsum"),
                                                 runs=2, inner_iters=3, warmup=1))
    assert rep2.kernels[0].kernel == "csr5" and rep2.kernels[0].speedup_n500 < 1.0


@pytest.mark.parametrize("kind", ["csr-scalar", "csr-segsum", "csr5"])
def test_correctness_guard_trips(g, kind):
    csr5, B = g
    a = csr5.stencil(0, 30)
    cfg = B.BenchConfig(runs=1, inner_iters=1, warmup=0, corrupt_for_test=B.KernelKind(kind))
    with pytest.raises(B.CorrectnessError, match=f"kernel {kind} disagrees with the dense "
                                                 f"reference on 'lap': max relative error"):
        B.run_benchmark(a, "lap", cfg)
    with pytest.raises(ValueError, match="runs and inner_iters must be >= 1"):
        B.run_benchmark(a, "lap", B.BenchConfig(runs=0))
