"""Hot-column x staging (hotx.cu) leaves every result bit for bit unchanged.

A random-gather plan whose x exceeds the L2 renumbers its hot columns in an
execution copy of col_idx and gathers their x values from a per-call staged
array.  The products and their order are the same, so y must equal the
unstaged kernel's bit for bit in both modes, across streams (each stream
stages its own copy), and the exported CSR5 arrays (the reference's
col_idx, format.cpp:226-249) must not see the renumbering.  Small R-MAT
matrices force the staging with CSR5G_HOT=1 and a column budget
(CSR5G_HOT_COLS) so that hot and cold columns both occur."""
import numpy as np
import pytest

from tests._util import assert_y_close

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _build(d, monkeypatch, **env):
    from paper_1503_05032_b200 import csr5
    for k in ("CSR5G_HOT", "CSR5G_HOT_COLS", "CSR5G_HOT_STRIDE", "CSR5G_HOT_L1", "CSR5G_HOT_ORDER",
              "CSR5G_XMODE", "CSR5G_GM"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))
    return csr5.csr_to_csr5(d, csr5.TuningParams())


# the staged gather paths, forced on small matrices: the plans' default
# (hottest first, hot values L1-allocated, cold ones 64-byte prefetched:
# GM 3), the ascending-order path without L1 allocation (GM 5), and the
# runtime switch (GM 0)
PATHS = {"gm3": {}, "gm5": {"CSR5G_HOT_L1": 0, "CSR5G_HOT_ORDER": 0, "CSR5G_XMODE": 1},
         "gm0": {"CSR5G_GM": 0}}


@pytest.mark.parametrize("path", sorted(PATHS))
@pytest.mark.parametrize("scale,stride", [(14, 1), (17, 8)])
def test_hot_staging_is_bit_identical(scale, stride, path, orc, monkeypatch):
    from oracle.oracle import Csr
    from paper_1503_05032_b200 import csr5
    d = csr5.rmat(scale, 16, 3, True)
    m, n = d.m, d.n
    x = orc.rng(5).random_x(n)
    xd = torch.as_tensor(x).cuda()
    plain = _build(d, monkeypatch, CSR5G_HOT=0)
    hot = _build(d, monkeypatch, CSR5G_HOT=1, CSR5G_HOT_COLS=n // 16, CSR5G_HOT_STRIDE=stride,
                 **PATHS[path])
    assert plain.info.kernel_variant == 1, "R-MAT should take the random-gather (VR) plan"
    assert plain.info.hot_cols == 0
    assert hot.info.x_mode == (1 if path == "gm5" else 5)
    assert 0 < hot.info.hot_cols <= 2 * (n // 16), hot.info.hot_cols
    assert hot.info.hot_coverage > 0.3, hot.info.hot_coverage  # power law: few columns, most gathers
    # the exported CSR5 arrays are the reference's, not the execution copy
    e0, e1 = plain.export(), hot.export()
    for k in e0:
        assert np.array_equal(e0[k], e1[k]), k
    for mode in ("deterministic", "atomic"):
        y0 = csr5.spmv_csr5(plain, xd, mode=mode).cpu().numpy()
        y1 = csr5.spmv_csr5(hot, xd, mode=mode).cpu().numpy()
        if mode == "deterministic":
            assert np.array_equal(y0.view(np.int64), y1.view(np.int64))
        else:  # atomic adds land in any order; values stay within tolerance
            np.testing.assert_allclose(y1, y0, rtol=1e-12, atol=0)
    # a second stream stages its own copy; results again identical
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y2 = csr5.spmv_csr5(hot, xd * 2.0, stream=s)
    s.synchronize()
    y2 = y2.cpu().numpy()
    y0x2 = csr5.spmv_csr5(plain, xd * 2.0).cpu().numpy()
    assert np.array_equal(y2.view(np.int64), y0x2.view(np.int64))
    # and y is the reference's within the north-star tolerance
    rp = d.row_ptr.cpu().numpy()
    a = Csr(m, n, rp, d.col_idx.cpu().numpy().astype(np.int64), d.val.cpu().numpy())
    assert_y_close(y0, orc.spmv(a, x, 32, int(plain.info.sigma)), a, x, f"rmat{scale}")
    # tile-range shards build their own hot sets; deterministic y is partition
    # invariant, so every shard count gives the single-device bits
    yd = csr5.spmv_csr5(plain, xd).cpu().numpy()
    sigma = int(plain.info.sigma)
    plain.release()
    hot.release()
    from tests import _shard_emulation as emu
    for world in (2, 3):
        ys = emu.emulate_shards_on_one_device(a, x, sigma, world)
        assert np.array_equal(ys.view(np.int64), yd.view(np.int64)), world
