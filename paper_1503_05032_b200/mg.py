"""Multi-GPU driver for one NVSwitch box: one process per GPU (torchrun),
torch.distributed for the plumbing.

Partition: rank g holds the global complete tiles
[floor(g*pc/G), floor((g+1)*pc/G)); the last rank also holds the CSR tail.
Shard edges are global tile boundaries, so each shard's CSR5 arrays are slices
of the single-device arrays (bit for bit).  x is replicated.

Per SpMV there is one real exchange step: a row whose nonzeros straddle a
shard edge gets a partial sum from each shard.  The row's owner is the shard
holding its first nonzero.  Each shard has at most one partial to send (its
first row, when it does not own it); the driver all-gathers the 16-byte
records and every owner adds the partials of later shards in shard order
(csr5g_fixup) -- deterministic.  In the iterative mode (y -> x, square A) the
owned row ranges of y are all-gathered (one NCCL all-gather, ranges padded to
the longest) into every rank's x.

The reference has no distributed backend; this is new ("Multi-GPU
driver").  Host logic is covered by world_size-2 gloo tests on CPU
(tests/test_mg_gloo.py); the CUDA calls are exercised shard by shard on one
device (emulate_shards_on_one_device).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib


def plan_tiles(pc: int, world: int) -> list[tuple[int, int]]:
    """Contiguous equal-tile ranges (CSR5 tiles are equal-nnz work units)."""
    return [(g * pc // world, (g + 1) * pc // world) for g in range(world)]


def effective_world(pc: int, world: int) -> int:
    """Ranks that hold at least one tile (a matrix smaller than the box uses
    fewer shards; the extra ranks hold nothing)."""
    return max(1, min(world, pc))


@dataclass
class ShardView:
    """What a rank needs to build its shard from the global CSR."""

    tile_begin: int
    tile_end: int
    with_tail: bool
    pos_begin: int  # global nonzero position of the shard's first entry
    pos_end: int    # one past the last


def shard_view(nnz: int, sigma: int, rank: int, world: int) -> ShardView | None:
    B = 32 * sigma
    pc = nnz // B
    w = effective_world(pc, world)
    if rank >= w:
        return None
    tb, te = plan_tiles(pc, w)[rank]
    last = te == pc
    return ShardView(tb, te, last and nnz % B > 0, tb * B, nnz if last else te * B)


def owned_ranges(infos) -> list[tuple[int, int]]:
    """Rows each shard writes in y (contiguous, covering [0, m))."""
    return [(int(i.own_row_begin), int(i.own_row_end)) for i in infos]


def _staged(dist, group=None) -> bool:
    """gloo process groups (CPU tests, or several ranks sharing one GPU for a
    functional check) stage CUDA tensors through host memory."""
    return dist.get_backend(group) == "gloo"


def all_gather_flat(dist, out, inp, group=None):
    """out[world * k] <- every rank's inp[k]: NCCL all_gather_into_tensor, or a
    host-staged list all_gather on gloo."""
    if not _staged(dist, group) or not inp.is_cuda:
        if _staged(dist, group):
            parts = list(out.view(-1, inp.numel()).unbind(0))
            dist.all_gather(parts, inp, group=group)
        else:
            dist.all_gather_into_tensor(out, inp, group=group)
        return out
    import torch
    h = inp.cpu()
    parts = [torch.empty_like(h) for _ in range(out.numel() // inp.numel())]
    dist.all_gather(parts, h, group=group)
    out.copy_(torch.cat(parts).to(out.device))
    return out


def exchange_records(dist, send, world: int, group=None):
    """All-gather every rank's 16-byte boundary record (int64 row, f64 value
    bits) -> [world, 2] int64 on send's device.  Backend-agnostic (NCCL on the
    GPU box, gloo in the CPU tests)."""
    import torch
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send, group=group)
    return torch.stack(parts)


class Csr5Sharded:
    """Rank-local shard of a CSR5 matrix plus the exchange (torch.distributed)."""

    def __init__(self, row_ptr, col_slice, val_slice, m: int, n: int, nnz: int, sigma: int,
                 rank: int, world: int, group=None):
        import torch
        import torch.distributed as dist

        from .csr5 import TuningParams, csr_to_csr5_shard
        self.torch, self.dist, self.group = torch, dist, group
        self.rank, self.world = rank, world
        self.m, self.n, self.nnz, self.sigma = m, n, nnz, sigma
        view = shard_view(nnz, sigma, rank, world)
        self.active = view is not None
        self.world_eff = effective_world(nnz // (32 * sigma), world)
        dev = row_ptr.device
        if self.active:
            self.a5 = csr_to_csr5_shard(row_ptr, col_slice, val_slice, m, n, nnz,
                                        TuningParams(sigma=sigma), view.tile_begin, view.tile_end,
                                        view.with_tail)
            self.own = (self.a5.info.own_row_begin, self.a5.info.own_row_end)
        else:
            self.a5 = None
            self.own = (m, m)
        # 16-byte boundary records: this rank's slot and the gathered table
        self.send = torch.zeros(2, dtype=torch.int64, device=dev)
        self.table = torch.zeros(2 * world, dtype=torch.int64, device=dev)
        if self.active:
            check(lib().csr5g_set_send_buffer(self.a5.handle, C.c_void_p(self.send.data_ptr())))
        own = torch.tensor([self.own[0], self.own[1]], dtype=torch.int64, device=dev)
        allown = torch.zeros(2 * world, dtype=torch.int64, device=dev)
        all_gather_flat(dist, allown, own, group)
        t = allown.cpu().tolist()
        self.ranges = [(t[2 * g], t[2 * g + 1]) for g in range(world)]

    @staticmethod
    def slices_for(nnz: int, sigma: int, rank: int, world: int):
        v = shard_view(nnz, sigma, rank, world)
        return (0, 0) if v is None else (v.pos_begin, v.pos_end)

    def spmv(self, x, y, events=None):
        """y[own rows] = (A x)[own rows]; other rows of y are scratch.  `events`
        (csr5.Event pair) brackets this rank's tile kernel."""
        from .csr5 import spmv_csr5, spmv_csr5_evt
        torch = self.torch
        if self.active and events is not None:
            spmv_csr5_evt(self.a5, x, y, events[0], events[1])
        elif self.active:
            spmv_csr5(self.a5, x, y)
        else:
            self.send.copy_(torch.tensor([-1, 0], dtype=torch.int64, device=self.send.device))
        all_gather_flat(self.dist, self.table, self.send, self.group)
        if self.active:
            check(lib().csr5g_fixup(self.a5.handle, C.c_void_p(self.table.data_ptr()),
                                    self.world_eff, self.rank, C.c_void_p(y.data_ptr()),
                                    C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return y

    def gather_y_into_x(self, y, x):
        """Iterative mode (square A): every rank's x <- the owned ranges of y,
        one all-gather (gather_owned)."""
        gather_owned(self.dist, y, x, self.ranges, self.rank, self.group)
        return x


def gather_owned(dist, y, x, ranges, rank, group=None):
    """x[lo:hi] <- rank g's y[lo:hi] for every g: one all-gather of the owned
    ranges (NCCL over NVLink; host-staged on gloo).  Ranges are uneven, so each
    rank sends its range padded to the longest and the received blocks are
    copied into place.  Host logic shared with the gloo tests."""
    import torch
    lens = [max(0, hi - lo) for lo, hi in ranges]
    width = max(lens) if lens else 0
    if width == 0:
        return x
    send = torch.zeros(width, dtype=y.dtype, device=y.device)
    lo, hi = ranges[rank]
    if hi > lo:
        send[:hi - lo].copy_(y[lo:hi])
    recv = torch.empty(width * len(ranges), dtype=y.dtype, device=y.device)
    all_gather_flat(dist, recv, send, group)
    for g, (lo, hi) in enumerate(ranges):
        if hi > lo:
            x[lo:hi].copy_(recv[g * width:g * width + hi - lo])
    return x


# ---------------------------------------------------------------------------
# Single-device emulation of the partition (tests): the same C-ABI calls as the
# distributed path, run shard after shard, with the all-gather done by hand.
# ---------------------------------------------------------------------------
def _shards_on_device(a, sigma: int, world: int):
    import torch

    from .csr5 import TuningParams, csr_to_csr5_shard
    rp = torch.as_tensor(np.ascontiguousarray(a.row_ptr, np.int64)).cuda()
    col = torch.as_tensor(np.ascontiguousarray(a.col_idx, np.int32)).cuda()
    val = torch.as_tensor(np.ascontiguousarray(a.val, np.float64)).cuda()
    out = []
    w = effective_world(a.nnz // (32 * sigma), world)
    for g in range(w):
        v = shard_view(a.nnz, sigma, g, w)
        out.append(csr_to_csr5_shard(rp, col[v.pos_begin:], val[v.pos_begin:], a.m, a.n, a.nnz,
                                     TuningParams(sigma=sigma), v.tile_begin, v.tile_end,
                                     v.with_tail))
    return out


def emulate_shard_exports(a, sigma: int, world: int) -> list[dict]:
    return [s.export() for s in _shards_on_device(a, sigma, world)]


def emulate_shards_on_one_device(a, x: np.ndarray, sigma: int, world: int) -> np.ndarray:
    import torch

    from .csr5 import spmv_csr5
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
