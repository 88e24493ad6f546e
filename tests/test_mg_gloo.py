"""Multi-rank host logic of the multi-GPU driver (paper_1503_05032_b200.mg),
run as world_size 2 and 3 process groups over gloo on CPU.

Every rank plans its shard with the product's planner (mg.shard_view), builds
the shard's partial result with a CPU emulation of the CUDA shard semantics
(spmv.cu resolve_item / k_fixup: rows owned by the shard holding their first
nonzero; a shard sends at most one partial, for a first row it does not own;
owners add later shards' partials in shard order), exchanges the 16-byte
records with mg.exchange_records, and assembles x for the next iteration with
mg.gather_owned (iterative y -> x mode).  The result must equal the
single-device SpMV on every rank.
"""
import os
import socket
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1503_05032_b200 import mg


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def emulate_shard(row_ptr, col, val, x, m, nnz, sigma, rank, world):
    """CPU restatement of one shard's csr5g_spmv + send record (test side)."""
    B = 32 * sigma
    v = mg.shard_view(nnz, sigma, rank, world, row_ptr)
    pc = nnz // B
    lo, hi = v.pos_begin, v.pos_end
    first_row = int(np.searchsorted(row_ptr, lo, side="right") - 1)
    first_owned = rank == 0 or row_ptr[first_row] >= lo
    if v.tile_end == pc:
        own_end = m
    else:
        nxt = int(np.searchsorted(row_ptr, v.tile_end * B, side="right") - 1)
        own_end = nxt if row_ptr[nxt] >= v.tile_end * B else nxt + 1
    own_begin = 0 if rank == 0 else (first_row if first_owned else first_row + 1)
    y = np.full(m, np.nan)
    # partial sums of the shard's nonzeros per row
    rows = np.searchsorted(row_ptr, np.arange(lo, hi), side="right") - 1
    part = np.zeros(m)
    np.add.at(part, rows, val[lo:hi] * x[col[lo:hi]])
    touched = np.zeros(m, bool)
    touched[rows] = True
    y[own_begin:own_end] = 0.0
    sel = touched.copy()
    sel[:own_begin] = False
    sel[own_end:] = False
    y[sel] = part[sel]
    send = (-1, 0.0)
    if not first_owned:
        send = (first_row, float(part[first_row]))
    last_row = int(rows[-1]) if hi > lo else first_row
    return dict(y=y, send=send, own=(own_begin, own_end), first_row=first_row,
                first_owned=first_owned, last_row=last_row, is_last=v.tile_end == pc)


def pack(rec):
    row, value = rec
    return torch.tensor([row, struct.unpack("<q", struct.pack("<d", value))[0]], dtype=torch.int64)


def unpack(t):
    return int(t[0]), struct.unpack("<d", struct.pack("<q", int(t[1])))[0]


def _worker(rank, world, port, case):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rp, col, val, m, sigma, iters = (case[k] for k in ("rp", "col", "val", "m", "sigma", "iters"))
        nnz = int(rp[-1])
        weff = mg.effective_world(nnz // (32 * sigma), world, rp, 32 * sigma)
        x = np.asarray(case["x"], dtype=np.float64)
        xt = torch.as_tensor(x.copy())
        for _ in range(iters):
            if rank < weff:
                sh = emulate_shard(rp, col, val, xt.numpy(), m, nnz, sigma, rank, weff)
                send = pack(sh["send"])
            else:
                sh = None
                send = pack((-1, 0.0))
            table = mg.exchange_records(dist, send, world)
            y = torch.as_tensor(np.nan_to_num(sh["y"]) if sh else np.zeros(m))
            if sh and not sh["is_last"] and not (not sh["first_owned"] and sh["last_row"] == sh["first_row"]):
                acc = float(y[sh["last_row"]])
                for s in range(rank + 1, weff):  # k_fixup: later shards in order
                    r, v = unpack(table[s])
                    if r != sh["last_row"]:
                        break
                    acc += v
                y[sh["last_row"]] = acc
            own = torch.tensor(list(sh["own"]) if sh else [m, m], dtype=torch.int64)
            owns = [torch.empty_like(own) for _ in range(world)]
            dist.all_gather(owns, own)
            ranges = [(int(o[0]), int(o[1])) for o in owns]
            got = sorted(r for r in ranges if r[1] > r[0])
            assert got[0][0] == 0 and got[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(got, got[1:])), got
            xn = torch.zeros(m, dtype=torch.float64)
            mg.gather_owned(dist, y, xn, ranges, rank)
            ref = np.zeros(m)
            for r in range(m):
                ref[r] = np.dot(val[rp[r]:rp[r + 1]], xt.numpy()[col[rp[r]:rp[r + 1]]])
            np.testing.assert_allclose(xn.numpy(), ref, rtol=1e-12, atol=1e-12)
            xt = xn
    finally:
        dist.destroy_process_group()


def _case(orc, kind, m, n, nnz, seed, frac, sigma, iters=2):
    a = orc.generate_synthetic(kind, m, n, nnz, seed, frac)
    x = orc.rng(seed).random_x(n)
    return dict(rp=a.row_ptr, col=a.col_idx, val=a.val, m=a.m, sigma=sigma, x=x, iters=iters)


def test_shard_edges_avoid_long_rows():
    """An edge inside a long row (three or more parts) moves to the tile where
    the row starts; other edges stay where the equal split puts them."""
    B = 32
    lens = np.full(4000, 3)
    lens[1000] = 300   # long: ~10 tiles
    lens[3000] = 40    # two or three parts
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(rp[-1])
    pc = nnz // B
    for world in (2, 3, 4, 8, 16, 64):
        r = mg.plan_tiles(pc, world, rp, B)
        assert r[0][0] == 0 and r[-1][1] == pc and len(r) <= world
        assert all(a < b for a, b in r)  # no empty shard
        for (_, e), _ in zip(r, r[1:]):
            row = int(np.searchsorted(rp, e * B, side="right") - 1)
            lo, hi = rp[row], rp[row + 1]
            parts = min((hi - 1) // B, pc) - min(lo // B, pc) + 1
            assert lo == e * B or parts < 3, (world, e, row, parts)


def test_plan_tiles_partition():
    for pc in (0, 1, 7, 100, 514517):
        for w in (1, 2, 3, 8):
            r = mg.plan_tiles(pc, w)
            assert r[0][0] == 0 and r[-1][1] == pc
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1
    assert mg.effective_world(3, 8) == 3 and mg.effective_world(0, 8) == 1


def test_plan_exchange_routes_partials_to_owners(orc):
    """mg.plan_exchange (the static routing of the P2P exchange) against the
    CPU emulation of the shard semantics: every non-owned first row goes to
    the shard whose owned range contains it; senders are contiguous."""
    for kind, m, n, nnz, seed, frac, sigma in [(1, 300, 30000, 60000, 3, 0.5, 4),
                                               (2, 5000, 4000, 120000, 4, 0.0, 16),
                                               (0, 2000, 2000, 54000, 5, 0.0, 27),
                                               (1, 300, 30000, 60000, 7, 0.5, 2)]:
        a = orc.generate_synthetic(kind, m, n, nnz, seed, frac)
        x = np.ones(a.n)
        for world in (2, 3, 8, 16):
            w = mg.effective_world(a.nnz // (32 * sigma), world, a.row_ptr, 32 * sigma)
            sh = [emulate_shard(a.row_ptr, a.col_idx, a.val, x, a.m, a.nnz, sigma, g, w)
                  for g in range(w)]
            dest, senders = mg.plan_exchange([(s["first_row"], s["first_owned"]) for s in sh],
                                             [s["own"] for s in sh])
            for g, s in enumerate(sh):
                if s["first_owned"]:
                    assert dest[g] == -1
                else:
                    lo, hi = sh[dest[g]]["own"]
                    assert lo <= s["first_row"] < hi and dest[g] < g
                sb, se = senders[g]
                assert all(dest[r] == g for r in range(sb, se))
                assert sum(d == g for d in dest) == se - sb


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_spmv_gloo(orc, world):
    # square matrices (iterative mode): one long row spanning shards, a skewed
    # matrix with empty rows, a regular one
    cases = [_case(orc, 1, 3000, 3000, 6000, 3, 0.3, 4),
             _case(orc, 2, 900, 900, 12000, 4, 0.0, 5),
             _case(orc, 0, 500, 500, 9000, 5, 0.0, 6)]
    for case in cases:
        mp.spawn(_worker, args=(world, _free_port(), case), nprocs=world, join=True)
