"""Multi-GPU driver for one NVSwitch box: one process per GPU (torchrun),
torch.distributed for the plumbing.

Partition: rank g holds the global complete tiles
[floor(g*pc/G), floor((g+1)*pc/G)); the last rank also holds the CSR tail.
Shard edges are global tile boundaries, so each shard's CSR5 arrays are slices
of the single-device arrays (bit for bit).  x is replicated.

Per SpMV there is one real exchange step: a row whose nonzeros straddle a
shard edge gets a partial sum from each shard.  The row's owner is the shard
holding its first nonzero.  Each shard has at most one partial to send (its
first row, when it does not own it), to a destination fixed by the matrix
structure (plan_exchange).  The default exchange is NVLink P2P (p2p.cu):
the shard's SpMV kernel stores the 16-byte partial straight into the
owner's mailbox and raises a flag; the owner's stream waits on the flags of
its senders, adds their partials in shard order (deterministic) and
acknowledges -- no collective, no host sync.  CSR5G_EXCHANGE=collective
selects the earlier form (all-gather of every shard's record, csr5g_fixup).
In the iterative mode (y -> x, square A) the owned row ranges of y are
all-gathered (one NCCL all-gather, ranges padded to the longest) into every
rank's x.

The reference has no distributed backend; this is new ("Multi-GPU
driver").  Host logic is covered by world_size-2/3 gloo tests on CPU
(tests/test_mg_gloo.py); the CUDA calls are exercised shard by shard on one
device (tests/_shard_emulation.py, mailboxes linked in one process) and by
several ranks sharing one GPU (tests/test_gpu_multirank.py; the two phases
then separated by host barriers, since ranks on one GPU must never wait on
each other inside the stream).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from ._lib import IPC_HANDLE_BYTES, check, lib


def plan_tiles(pc: int, world: int, row_ptr=None, B: int | None = None) -> list[tuple[int, int]]:
    """Contiguous tile ranges of the non-empty shards, at most `world` of them
    (CSR5 tiles are equal-nnz work units: the equal split).

    With the matrix's row_ptr (numpy or torch) and the tile size B, an edge
    inside a long row (nonzeros in three or more parts: tiles, the tail)
    moves to the tile where that row starts -- or, if that would empty the
    shard on its left, past the row's last tile -- so every long row lies in
    one shard: its parts meet in that shard's fixed-order sum, and a row split
    by an edge has one partial on each side, which the fix-up adds (a + b).  y
    is then bit-identical for every shard count (deterministic mode).  A row
    larger than the shards leaves fewer of them (the last ranks hold nothing)."""
    if world <= 1 or pc <= 1:
        return [(0, pc)]
    edges = [0]
    for g in range(1, world):
        e = max(g * pc // world, edges[-1] + 1)
        if row_ptr is not None and B:
            for _ in range(64):
                if e >= pc:
                    break
                r = _row_of(row_ptr, e * B)
                lo, hi = _at(row_ptr, r), _at(row_ptr, r + 1)
                first, last = min(lo // B, pc), min((hi - 1) // B, pc)
                if lo == e * B or last - first < 2:
                    break  # the row starts at the edge, or is not long
                e = first if first > edges[-1] else last + 1
        if e >= pc:
            break
        edges.append(e)
    edges.append(pc)
    return [(edges[g], edges[g + 1]) for g in range(len(edges) - 1)]


def _at(row_ptr, i: int) -> int:
    return int(row_ptr[i])


def _row_of(row_ptr, g: int) -> int:
    """format.cpp:42-50 row_of_nonzero on a host or device row_ptr."""
    m = len(row_ptr) - 1
    if type(row_ptr).__module__.startswith("torch"):
        import torch
        r = int(torch.searchsorted(row_ptr, torch.tensor([g], dtype=row_ptr.dtype,
                                                          device=row_ptr.device), right=True)) - 1
    else:
        r = int(np.searchsorted(row_ptr, g, side="right")) - 1
    return min(max(r, 0), max(m - 1, 0))


def effective_world(pc: int, world: int, row_ptr=None, B: int | None = None) -> int:
    """Ranks that hold at least one tile (a matrix smaller than the box, or
    one whose long rows swallow shards, uses fewer; the extra ranks hold
    nothing)."""
    return len(plan_tiles(pc, max(1, min(world, pc)), row_ptr, B))


@dataclass
class ShardView:
    """What a rank needs to build its shard from the global CSR."""

    tile_begin: int
    tile_end: int
    with_tail: bool
    pos_begin: int  # global nonzero position of the shard's first entry
    pos_end: int    # one past the last


def shard_view(nnz: int, sigma: int, rank: int, world: int, row_ptr=None) -> ShardView | None:
    B = 32 * sigma
    pc = nnz // B
    plan = plan_tiles(pc, max(1, min(world, pc)), row_ptr, B)
    if rank >= len(plan):
        return None
    tb, te = plan[rank]
    last = te == pc
    return ShardView(tb, te, last and nnz % B > 0, tb * B, nnz if last else te * B)


def owned_ranges(infos) -> list[tuple[int, int]]:
    """Rows each shard writes in y (contiguous, covering [0, m))."""
    return [(int(i.own_row_begin), int(i.own_row_end)) for i in infos]


class _CudaArray:
    """__cuda_array_interface__ over library-owned device memory."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def _device_view(ptr: int, n: int, device: int):
    import torch
    return torch.as_tensor(_CudaArray(ptr, n), device=f"cuda:{device}")


def plan_exchange(firsts, owns):
    """Static routing of the boundary partials (host logic, shared with the
    gloo tests).

    firsts[g] = (first_row, first_owned) of shard g, owns[g] = its owned row
    range [lo, hi) (empty for a shard lying inside one row).  Returns
    dest[g] (the rank owning shard g's first row, -1 when g owns it) and
    senders[g] = (sb, se): the later ranks whose partial g receives, always the
    contiguous block right after g."""
    w = len(firsts)
    dest = [-1] * w
    for g, (row, owned) in enumerate(firsts):
        if owned:
            continue
        hits = [o for o in range(g) if owns[o][0] <= row < owns[o][1]]
        if len(hits) != 1:
            raise RuntimeError(f"shard {g}: row {row} has {len(hits)} owners among {owns[:g]}")
        dest[g] = hits[0]
    senders = []
    for g in range(w):
        src = [s for s in range(w) if dest[s] == g]
        if src and src != list(range(g + 1, g + 1 + len(src))):
            raise RuntimeError(f"shard {g}: senders {src} are not the ranks right after it")
        senders.append((g + 1, g + 1 + len(src)) if src else (0, 0))
    return dest, senders


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
                 rank: int, world: int, group=None, iterative: bool = False):
        import torch
        import torch.distributed as dist

        from .csr5 import TuningParams, csr_to_csr5_shard
        self.torch, self.dist, self.group = torch, dist, group
        self.rank, self.world = rank, world
        self.m, self.n, self.nnz, self.sigma = m, n, nnz, sigma
        view = shard_view(nnz, sigma, rank, world, row_ptr)
        self.active = view is not None
        self.world_eff = effective_world(nnz // (32 * sigma), world, row_ptr, 32 * sigma)
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
        first = (self.a5.info.first_row, int(rank == 0 or self.own[0] == self.a5.info.first_row)) \
            if self.active else (m, 1)
        own = torch.tensor([self.own[0], self.own[1], first[0], first[1]], dtype=torch.int64,
                           device=dev)
        allown = torch.zeros(4 * world, dtype=torch.int64, device=dev)
        all_gather_flat(dist, allown, own, group)
        t = allown.cpu().tolist()
        self.ranges = [(t[4 * g], t[4 * g + 1]) for g in range(world)]
        self.exchange = os.environ.get("CSR5G_EXCHANGE", "p2p")
        self.mailbox = None
        self.mcast = False
        self.iterative = iterative and self.exchange == "p2p"
        if self.iterative and m != n:
            raise ValueError("iterative mode needs a square matrix")
        if self.exchange == "p2p":
            w = self.world_eff
            firsts = [(t[4 * g + 2], t[4 * g + 3]) for g in range(w)]
            self.dest, self.senders = plan_exchange(firsts, self.ranges[:w])
            self._connect(dev)
        elif self.exchange != "collective":
            raise ValueError(f"CSR5G_EXCHANGE={self.exchange}: expected p2p or collective")

    def _connect(self, dev):
        """Mailbox per rank; IPC handles all-gathered once; each rank maps the
        mailboxes it stores into (dest) and acknowledges (senders)."""
        torch, dist = self.torch, self.dist
        L = lib()
        mb = C.c_void_p()
        check(L.csr5g_mailbox_create(dev.index or 0, self.world, self.rank,
                                     self.m if self.iterative else 0, C.byref(mb)))
        self.mailbox = mb
        hbuf = (C.c_uint8 * IPC_HANDLE_BYTES)()
        check(L.csr5g_mailbox_ipc_handle(mb, hbuf))
        mine = torch.tensor(list(hbuf), dtype=torch.uint8, device=dev)
        allh = torch.zeros(IPC_HANDLE_BYTES * self.world, dtype=torch.uint8, device=dev)
        all_gather_flat(dist, allh, mine, self.group)
        allh = allh.cpu().numpy()
        # ranks sharing one GPU must not wait on each other inside a stream:
        # spmv() then separates post and fix-up with host barriers
        uid = torch.tensor(list(torch.cuda.get_device_properties(dev).uuid.bytes), dtype=torch.uint8,
                           device=dev)
        allu = torch.zeros(16 * self.world, dtype=torch.uint8, device=dev)
        all_gather_flat(dist, allu, uid, self.group)
        allu = allu.cpu().numpy().reshape(self.world, 16)
        self.shared_gpu = len({bytes(u) for u in allu}) < self.world
        if self.active:
            d = self.dest[self.rank]
            sb, se = self.senders[self.rank]
            peers = set(([d] if d >= 0 else []) + list(range(sb, se)))
            if self.iterative:  # every active rank stores its rows of the next x here
                peers |= set(range(self.world_eff))
            peers.discard(self.rank)
            for peer in sorted(peers):
                h = allh[IPC_HANDLE_BYTES * peer:IPC_HANDLE_BYTES * (peer + 1)]
                check(L.csr5g_mailbox_open_peer(mb, peer,
                                                (C.c_uint8 * IPC_HANDLE_BYTES)(*h.tolist())))
            check(L.csr5g_mg_bind(self.a5.handle, mb, d, sb, se, self.world_eff))
        self.mcast = self.iterative and self._setup_mcast(dev)

    def _agree(self, dev, ok: bool) -> bool:
        """True when every rank's flag is set (all-gather of one int each)."""
        torch = self.torch
        mine = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        allf = torch.zeros(self.world, dtype=torch.int32, device=dev)
        all_gather_flat(self.dist, allf, mine, self.group)
        return bool(allf.min().item())

    def _setup_mcast(self, dev) -> bool:
        """NVSwitch multicast x buffers for the fused iterative mode (p2p.cu,
        csr5g_mailbox_mcast_*): rank 0 creates the object and exports its
        fabric handle, the other active ranks import it, every active rank adds
        its device, then binds its x ping-pong.  Every step is agreed by all
        ranks; any failure (no multicast, no fabric handles, ranks sharing a
        GPU) leaves the peer-store path.  Opt-in: CSR5G_MCAST=1."""
        torch, L = self.torch, lib()
        # opt-in until it has run on a multi-GPU box: on the one-GPU test box
        # cuMulticastCreate rejects every configuration (tools/mc_probe_raw.py)
        want = os.environ.get("CSR5G_MCAST", "0") == "1" and not self.shared_gpu
        sup = C.c_int32(0)
        if want and self.active:
            want = L.csr5g_mcast_supported(dev.index or 0, C.byref(sup)) == 0 and sup.value == 1
        if not self._agree(dev, want or not self.active):
            return False
        n = self.world_eff
        handle = (C.c_uint8 * 64)()
        ok = True
        if self.rank == 0:
            ok = L.csr5g_mailbox_mcast_create(self.mailbox, n, handle) == 0
        hb = torch.tensor(list(handle), dtype=torch.uint8, device=dev)
        allh = torch.zeros(64 * self.world, dtype=torch.uint8, device=dev)
        all_gather_flat(self.dist, allh, hb, self.group)
        if not self._agree(dev, ok):
            return False
        h0 = (C.c_uint8 * 64)(*allh[:64].cpu().tolist())
        if self.active and self.rank != 0:
            ok = L.csr5g_mailbox_mcast_import(self.mailbox, n, h0) == 0
        if self.active and ok:
            ok = L.csr5g_mailbox_mcast_add(self.mailbox) == 0
        if not self._agree(dev, ok):
            L.csr5g_mailbox_mcast_release(self.mailbox)
            return False
        if self.active:  # every device was added before anyone binds
            ok = L.csr5g_mailbox_mcast_bind(self.mailbox) == 0
        if not self._agree(dev, ok):
            L.csr5g_mailbox_mcast_release(self.mailbox)
            return False
        return True

    def mailbox_errors(self) -> int:
        """Protocol violations seen by this rank's fix-ups (synchronous)."""
        if self.mailbox is None:
            return 0
        e = C.c_uint32()
        check(lib().csr5g_mailbox_errors(self.mailbox, C.byref(e)))
        return e.value

    def close(self):
        if self.mailbox is not None:
            self.torch.cuda.synchronize()
            if self.shared_gpu:  # no rank unmaps a mailbox a peer still writes into
                self.dist.barrier(group=self.group)
            if self.a5 is not None:
                self.a5.release()
                self.a5 = None
            check(lib().csr5g_mailbox_release(self.mailbox))
            self.mailbox = None

    @staticmethod
    def slices_for(nnz: int, sigma: int, rank: int, world: int, row_ptr=None):
        v = shard_view(nnz, sigma, rank, world, row_ptr)
        return (0, 0) if v is None else (v.pos_begin, v.pos_end)

    def spmv(self, x, y, events=None):
        """y[own rows] = (A x)[own rows]; other rows of y are scratch.  `events`
        (csr5.Event pair) brackets this rank's tile kernel."""
        from .csr5 import spmv_csr5, spmv_csr5_evt
        torch = self.torch
        if self.exchange == "p2p":
            return self._spmv_p2p(x, y, events)
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

    def _spmv_p2p(self, x, y, events):
        torch, L = self.torch, lib()
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        ev = (events[0].p, events[1].p) if events is not None else (None, None)
        xp, yp = C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr())
        if not self.shared_gpu:
            if self.active:
                check(L.csr5g_mg_spmv(self.a5.handle, xp, yp, stream, ev[0], ev[1]))
            return y
        # ranks on one GPU: every wait is satisfied before it is enqueued
        if self.active:
            check(L.csr5g_mg_spmv_post(self.a5.handle, xp, yp, stream, ev[0], ev[1]))
        torch.cuda.current_stream().synchronize()
        self.dist.barrier(group=self.group)
        if self.active:
            check(L.csr5g_mg_spmv_fixup(self.a5.handle, yp, stream))
        torch.cuda.current_stream().synchronize()
        self.dist.barrier(group=self.group)
        return y

    def x_buffer(self, which: int):
        """Iterative mode: this rank's x buffer `which` (x_k = x_buffer(k & 1)) as
        a torch view of the mailbox memory (no copy)."""
        p = C.c_void_p()
        check(lib().csr5g_mailbox_vector(self.mailbox, which, C.byref(p)))
        return _device_view(p.value, self.m, self.torch.cuda.current_device())

    def spmv_iter(self, it: int, events=None):
        """Fused iterative step: x_{it+1} = A x_it in the mailbox buffers, every
        rank's owned rows stored into every peer's buffer by the SpMV kernels
        themselves (csr5g_mg_iter).  Returns this rank's x_{it+1} view."""
        torch, L = self.torch, lib()
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        ev = (events[0].p, events[1].p) if events is not None else (None, None)
        if not self.shared_gpu:
            if self.active:
                check(L.csr5g_mg_iter(self.a5.handle, it, stream, ev[0], ev[1]))
            return self.x_buffer(it + 1)
        if self.active:
            check(L.csr5g_mg_iter_post(self.a5.handle, it, stream, ev[0], ev[1]))
        torch.cuda.current_stream().synchronize()
        self.dist.barrier(group=self.group)
        if self.active:
            check(L.csr5g_mg_iter_finish(self.a5.handle, it, stream))
        torch.cuda.current_stream().synchronize()
        self.dist.barrier(group=self.group)
        return self.x_buffer(it + 1)

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
