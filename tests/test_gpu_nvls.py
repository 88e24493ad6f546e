"""NVSwitch multicast (NVLS) x buffers of the fused iterative mode (p2p.cu,
csr5g_mailbox_mcast_*), on the one GPU the test box has: a one-device
multicast object.  The multi-rank protocol (fabric-handle export / import,
every rank adding its device) needs several GPUs; what one GPU proves is the
mechanism -- the VMM allocation bound to a multicast object, the unicast and
multicast mappings, multimem.st from a kernel landing in the bound copy --
and that the fused iterative SpMV with its mirror stores going through the
multicast mapping gives the peer-store path's x_k bit for bit."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _mcast_ok(L):
    """Multicast reported and an object can be created here (the test box's
    driver reports support but rejects cuMulticastCreate with one GPU
    visible: then the test skips and says so)."""
    v = C.c_int32()
    if L.csr5g_mcast_supported(0, C.byref(v)) != 0 or v.value != 1:
        return False, "device reports no NVSwitch multicast support"
    mb = C.c_void_p()
    if L.csr5g_mailbox_create(0, 1, 0, 1 << 16, C.byref(mb)) != 0:
        return False, "mailbox"
    try:
        if L.csr5g_mailbox_mcast_create(mb, 1, None) != 0:
            L.csr5g_last_error.restype = C.c_char_p
            return False, "multicast object creation refused: " + L.csr5g_last_error().decode()
        return True, ""
    finally:
        L.csr5g_mailbox_release(mb)


def _iterate(a, x0, sigma, iters, mcast):
    from paper_1503_05032_b200 import csr5
    from paper_1503_05032_b200._lib import check, lib
    from paper_1503_05032_b200.mg import _device_view
    L = lib()
    d = csr5.CsrMatrix.from_host(a.m, a.n, a.row_ptr, a.col_idx.astype(np.int32), a.val)
    pc = a.nnz // (32 * sigma)
    h = csr5.csr_to_csr5_shard(d.row_ptr, d.col_idx, d.val, a.m, a.n, a.nnz,
                               csr5.TuningParams(sigma=sigma), 0, pc, int(a.nnz % (32 * sigma) > 0))
    mb = C.c_void_p()
    check(L.csr5g_mailbox_create(0, 1, 0, a.m, C.byref(mb)))
    try:
        if mcast:
            check(L.csr5g_mailbox_mcast_create(mb, 1, None))
            check(L.csr5g_mailbox_mcast_add(mb))
            check(L.csr5g_mailbox_mcast_bind(mb))
            bad = C.c_int64(-1)
            check(L.csr5g_mailbox_mcast_selftest(mb, C.byref(bad)))
            assert bad.value == 0, f"{bad.value} multimem stores did not land"
        check(L.csr5g_mg_bind(h.handle, mb, -1, 0, 0, 1))

        def buf(which):
            p = C.c_void_p()
            check(L.csr5g_mailbox_vector(mb, which, C.byref(p)))
            return _device_view(p.value, a.m, 0)

        buf(0).copy_(torch.as_tensor(x0).cuda())
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        outs = []
        for it in range(iters):
            check(L.csr5g_mg_iter(h.handle, it, stream, None, None))
            outs.append(buf(it + 1).cpu().numpy().copy())
        torch.cuda.synchronize()
        return outs
    finally:
        torch.cuda.synchronize()
        h.release()
        L.csr5g_mailbox_release(mb)


def test_nvls_fused_iteration_matches_peer_stores(orc):
    from paper_1503_05032_b200._lib import lib
    from oracle.oracle import stencil
    ok, why = _mcast_ok(lib())
    if not ok:
        pytest.skip(why)
    a = stencil(orc, 0, 120, 120)  # square, 14,400 rows
    sigma = orc.select_sigma(a.nnz / a.m)
    x0 = orc.rng(3).random_x(a.n)
    ref = _iterate(a, x0, sigma, 3, mcast=False)
    got = _iterate(a, x0, sigma, 3, mcast=True)
    for k, (r, g) in enumerate(zip(ref, got)):
        assert np.array_equal(r.view(np.int64), g.view(np.int64)), k
    # and x_1 is A x_0 (oracle, within tolerance)
    y = orc.spmv(a, x0, 32, sigma)
    assert np.max(np.abs(got[0] - y) / np.maximum(1.0, np.abs(y))) <= 1e-12
