"""Single-device emulation of the multi-GPU partition (test infrastructure).

The same C-ABI calls as the distributed driver (paper_1503_05032_b200/mg.py),
run shard after shard in one process on one device, with the all-gather done
by hand and the P2P mailboxes linked directly (csr5g_mailbox_link_local)."""
import ctypes as C

import numpy as np

from paper_1503_05032_b200._lib import check, lib
from paper_1503_05032_b200.mg import _device_view, effective_world, plan_exchange, shard_view


def _shards_on_device(a, sigma: int, world: int):
    import torch

    from paper_1503_05032_b200.csr5 import TuningParams, csr_to_csr5_shard
    rp = torch.as_tensor(np.ascontiguousarray(a.row_ptr, np.int64)).cuda()
    col = torch.as_tensor(np.ascontiguousarray(a.col_idx, np.int32)).cuda()
    val = torch.as_tensor(np.ascontiguousarray(a.val, np.float64)).cuda()
    out = []
    w = effective_world(a.nnz // (32 * sigma), world, a.row_ptr, 32 * sigma)
    for g in range(w):
        v = shard_view(a.nnz, sigma, g, w, a.row_ptr)
        out.append(csr_to_csr5_shard(rp, col[v.pos_begin:], val[v.pos_begin:], a.m, a.n, a.nnz,
                                     TuningParams(sigma=sigma), v.tile_begin, v.tile_end,
                                     v.with_tail))
    return out


def emulate_shard_exports(a, sigma: int, world: int) -> list[dict]:
    return [s.export() for s in _shards_on_device(a, sigma, world)]


def emulate_shards_on_one_device(a, x: np.ndarray, sigma: int, world: int) -> np.ndarray:
    import torch

    from paper_1503_05032_b200.csr5 import spmv_csr5
    shards = _shards_on_device(a, sigma, world)
    w = len(shards)
    xd = torch.as_tensor(np.ascontiguousarray(x, np.float64)).cuda()
    table = torch.zeros(2 * w, dtype=torch.int64, device="cuda")
    ys = []
    for g, s in enumerate(shards):
        check(lib().csr5g_set_send_buffer(s.handle, C.c_void_p(table.data_ptr() + 16 * g)))
        y = torch.full((a.m,), float("nan"), dtype=torch.float64, device="cuda")
        spmv_csr5(s, xd, y)
        ys.append(y)
    stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for g, s in enumerate(shards):
        check(lib().csr5g_fixup(s.handle, C.c_void_p(table.data_ptr()), w, g,
                                C.c_void_p(ys[g].data_ptr()), stream))
    y = torch.full((a.m,), float("nan"), dtype=torch.float64, device="cuda")
    for g, s in enumerate(shards):
        lo, hi = s.info.own_row_begin, s.info.own_row_end
        y[lo:hi] = ys[g][lo:hi]
    torch.cuda.synchronize()
    ranges = [(s.info.own_row_begin, s.info.own_row_end) for s in shards]
    assert ranges[0][0] == 0 and ranges[-1][1] == a.m, ranges
    for (l0, h0), (l1, h1) in zip(ranges, ranges[1:]):
        assert h0 == l1, ranges
    return y.cpu().numpy()


def emulate_p2p_on_one_device(a, xs, sigma: int, world: int):
    """The P2P exchange (p2p.cu) with every shard in this process on one
    device: mailboxes linked directly, one stream, all posts of a call before
    its fix-ups (so every stream wait is already satisfied -- no shard ever
    waits on another).  xs: list of x vectors, one SpMV call each (epochs
    advance, acks recycle the slots).  Returns [y per call], mailbox errors."""
    import torch

    L = lib()
    shards = _shards_on_device(a, sigma, world)
    w = len(shards)
    infos = [s.info for s in shards]
    owns = [(i.own_row_begin, i.own_row_end) for i in infos]
    firsts = [(i.first_row, int(g == 0 or i.own_row_begin == i.first_row))
              for g, i in enumerate(infos)]
    dest, senders = plan_exchange(firsts, owns)
    boxes = []
    for g in range(w):
        mb = C.c_void_p()
        check(L.csr5g_mailbox_create(torch.cuda.current_device(), w, g, 0, C.byref(mb)))
        boxes.append(mb)
    try:
        for g in range(w):
            peers = set(([dest[g]] if dest[g] >= 0 else []) + list(range(*senders[g])))
            for p in sorted(peers):
                check(L.csr5g_mailbox_link_local(boxes[g], p, boxes[p]))
            check(L.csr5g_mg_bind(shards[g].handle, boxes[g], dest[g], *senders[g], w))
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        outs = []
        for x in xs:
            xd = torch.as_tensor(np.ascontiguousarray(x, np.float64)).cuda()
            ys = [torch.full((a.m,), float("nan"), dtype=torch.float64, device="cuda")
                  for _ in range(w)]
            for g in reversed(range(w)):  # senders post before their owners
                check(L.csr5g_mg_spmv_post(shards[g].handle, C.c_void_p(xd.data_ptr()),
                                           C.c_void_p(ys[g].data_ptr()), stream, None, None))
            for g in range(w):
                check(L.csr5g_mg_spmv_fixup(shards[g].handle, C.c_void_p(ys[g].data_ptr()), stream))
            y = torch.full((a.m,), float("nan"), dtype=torch.float64, device="cuda")
            for g, (lo, hi) in enumerate(owns):
                y[lo:hi] = ys[g][lo:hi]
            outs.append(y.cpu().numpy())
        errs = []
        for mb in boxes:
            e = C.c_uint32()
            check(L.csr5g_mailbox_errors(mb, C.byref(e)))
            errs.append(e.value)
        return outs, errs, dest, senders
    finally:
        for s in shards:
            s.release()
        for mb in boxes:
            L.csr5g_mailbox_release(mb)


def emulate_p2p_iterative_on_one_device(a, x0, sigma: int, world: int, iters: int):
    """The fused iterative mode (csr5g_mg_iter) with every shard in this
    process on one device: per iteration all posts, then all finishes, on one
    stream (each stream wait already satisfied).  Returns, per iteration, the
    x_{k+1} buffer of every shard (they must agree bit for bit), and the
    mailbox errors."""
    import torch

    L = lib()
    assert a.m == a.n
    shards = _shards_on_device(a, sigma, world)
    w = len(shards)
    infos = [s.info for s in shards]
    owns = [(i.own_row_begin, i.own_row_end) for i in infos]
    firsts = [(i.first_row, int(g == 0 or i.own_row_begin == i.first_row))
              for g, i in enumerate(infos)]
    dest, senders = plan_exchange(firsts, owns)
    dev = torch.cuda.current_device()
    boxes = []
    for g in range(w):
        mb = C.c_void_p()
        check(L.csr5g_mailbox_create(dev, w, g, a.m, C.byref(mb)))
        boxes.append(mb)
    try:
        for g in range(w):
            for p in range(w):
                if p != g:
                    check(L.csr5g_mailbox_link_local(boxes[g], p, boxes[p]))
            check(L.csr5g_mg_bind(shards[g].handle, boxes[g], dest[g], *senders[g], w))

        def buf(g, which):
            p = C.c_void_p()
            check(L.csr5g_mailbox_vector(boxes[g], which, C.byref(p)))
            return _device_view(p.value, a.m, dev)

        xd = torch.as_tensor(np.ascontiguousarray(x0, np.float64)).cuda()
        for g in range(w):
            buf(g, 0).copy_(xd)
            buf(g, 1).fill_(float("nan"))
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        outs = []
        for it in range(iters):
            for g in reversed(range(w)):
                check(L.csr5g_mg_iter_post(shards[g].handle, it, stream, None, None))
            for g in range(w):
                check(L.csr5g_mg_iter_finish(shards[g].handle, it, stream))
            outs.append([buf(g, it + 1).cpu().numpy() for g in range(w)])
        errs = []
        for mb in boxes:
            e = C.c_uint32()
            check(L.csr5g_mailbox_errors(mb, C.byref(e)))
            errs.append(e.value)
        return outs, errs
    finally:
        torch.cuda.synchronize()
        for s in shards:
            s.release()
        for mb in boxes:
            L.csr5g_mailbox_release(mb)
