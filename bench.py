#!/usr/bin/env python
"""CSR5 fp64 SpMV benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload st27_200]
    python bench.py --impl reference ...        # the reference's CPU path

One step = one CSR5 SpMV y = A x over the whole matrix (one pass of the hot
path).  At N=1 the workload is BASELINE config 2, the 3D 27-point stencil
200^3 (213.8M nnz, sigma = 27 by the reference rule, 64-bit descriptors).
Under torchrun (N>1) the matrix is tile-range sharded over the ranks with x
replicated; a step includes the boundary-row exchange (NVLink P2P
stores into the owner's mailbox, p2p.cu; no collective).  Default
--scaling weak: the global matrix is N times the 1-GPU one (the stencil N
times deeper along z, graphs log2 N scales larger: R-MAT s24 -> s27 at N=8,
BASELINE config 5), so per-GPU work is fixed; --scaling strong shards the
1-GPU matrix itself.

`value` is GFLOP/s = 2*nnz / t with A and x resident in HBM; t is the max over
ranks of CUDA-event time on the launching stream.  L2 is flushed between timed
calls (2x L2 read outside the events).  `e2e` is the same metric through
the host-buffer call (csr5.spmv_host_batch): per step pinned x H2D + SpMV + y
D2H, pipelined across steps on separate copy engines.  The roofline
figure is for the dominant tile kernel alone (events around it), with the
algorithmic bytes of SURVEY 8(d).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CSR5 fp64 SpMV GFLOP/s + HBM GB/s (% roofline) at 1/2/4/8 B200; conv cost"
UNIT = "GFLOP/s"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str):
    """dram read+write bytes per launch of the tile kernel from the committed
    `ncu --set full` summary (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get(workload, {}).get("k_spmv_dram_bytes")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# --------------------------------------------------------------------------
# the reference's CPU path (oracle/_ref = the unmodified reference library)
# --------------------------------------------------------------------------
def host_matrix(workload: dict):
    """The workload's CSR on the host with the reference's int64 indices.
    Stencils come from the host generator (oracle/testgen.c, no GPU needed);
    the graph workloads are generated on the device and copied back."""
    import numpy as np

    from oracle.oracle import Csr, Oracle, stencil
    if workload["gen"] == "stencil":
        return stencil(Oracle(), workload["kind"], workload["a"], workload.get("layers"))
    from paper_1503_05032_b200.synthetic import make_matrix
    d = make_matrix(workload, "cuda")
    a = Csr(d.m, d.n, d.row_ptr.cpu().numpy(), d.col_idx.cpu().numpy().astype(np.int64),
            d.val.cpu().numpy())
    del d
    return a


def workload_n(workload: dict) -> int:
    if workload["gen"] == "stencil":
        return workload["a"] ** (2 if workload["kind"] == 1 else 1) * workload.get("layers",
                                                                                 workload["a"])
    return 1 << (workload["scale"] if workload["gen"] == "rmat" else workload["log2_m"])


def reference_cpu(workload: dict, x, budget_s: float, omega=4, sigma=16, steps=None, warmup=0,
                  also_w32=False):
    """Time the reference csr5::spmv_csr5 (deterministic) on the host cores.

    steps=None: the bench.cpp:147-160 protocol (samples of `inner` back-to-back
    calls, best sample reported) within ~budget_s.  steps=K: K single calls
    after `warmup` calls (the --impl reference step loop)."""
    import ctypes

    import numpy as np

    from oracle.oracle import Ref
    ref = Ref()
    t0 = time.time()
    a = host_matrix(workload)
    gen_s = time.time() - t0
    h, conv_ms = ref.build_handle(a, omega, sigma)
    dp = ctypes.POINTER(ctypes.c_double)
    xv = ref.L.ref_vec_new(np.ascontiguousarray(x).ctypes.data_as(dp), a.n)
    y = np.zeros(a.m)
    yp = y.ctypes.data_as(dp)
    first = ref.L.ref_time_spmv(h, xv, yp, 0, 1)
    if steps is None:
        inner = max(1, int(0.5 / max(first / 1e3, 1e-6)))
        samples = []
        t_end = time.time() + budget_s
        while (time.time() < t_end or len(samples) < 2) and len(samples) < 10:
            samples.append(ref.L.ref_time_spmv(h, xv, yp, 0, inner))
    else:
        inner = 1
        for _ in range(warmup):
            ref.L.ref_time_spmv(h, xv, yp, 0, 1)
        samples = [ref.L.ref_time_spmv(h, xv, yp, 0, 1) for _ in range(steps)]
    scalar = ref.L.ref_time_csr_scalar(h, xv, yp, 3)
    ref.L.ref_time_spmv(h, xv, yp, 0, 1)  # leave y = the csr5 result
    threads = ref.max_threads()
    w32 = None
    if also_w32:  # the GPU's own omega = 32, sigma = auto on the CPU too
        from oracle.oracle import Oracle
        s32 = Oracle().select_sigma(a.nnz / max(a.m, 1))
        h32, conv32 = ref.build_handle(a, 32, s32)
        y32 = np.zeros(a.m)
        p32 = y32.ctypes.data_as(dp)
        one = ref.L.ref_time_spmv(h32, xv, p32, 0, 1)
        inner32 = max(1, int(0.5 / max(one / 1e3, 1e-6)))
        best = min(ref.L.ref_time_spmv(h32, xv, p32, 0, inner32) for _ in range(3))
        ref.L.ref_free(h32)
        w32 = dict(omega=32, sigma=s32, best_ms=best, conv_ms=conv32, inner=inner32)
    ref.L.ref_vec_free(xv)
    ref.L.ref_free(h)
    return dict(nnz=a.nnz, m=a.m, best_ms=min(samples), mean_ms=sum(samples) / len(samples),
                samples=samples, inner=inner, conv_ms=conv_ms, gen_s=gen_s, threads=threads,
                csr_scalar_ms=scalar, omega=omega, sigma=sigma, y=y, w32=w32)


def est_nnz(wl: dict) -> int:
    from oracle.oracle import stencil_box_size
    if wl["gen"] == "stencil":
        return stencil_box_size(wl["kind"], wl["a"], wl.get("layers", wl["a"]))[1]
    if wl["gen"] == "rmat":
        return wl["edge_factor"] << wl["scale"]
    return int((1 << wl["log2_m"]) * (1 - wl["p_empty"]) * (wl["min_len"] + wl["max_len"]) / 2
               + wl["n_long"] * wl["long_len"])


def mem_available():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except Exception:
        pass
    return None


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    return model, os.cpu_count()


def run_reference(args, workload_name, workload):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    compiled from /root/reference/proj/core/src) on all host threads; rank 0
    only under torchrun."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1503_05032_b200.synthetic import bench_x, scaled_workload
    note = "1-GPU workload"
    if world > 1 and args.scaling == "weak":
        # the same global matrix as our arm, when the host can hold the
        # reference's copies of it (~40 B per nonzero: int64 CSR + Csr5Matrix)
        wl_g = scaled_workload(workload, world)
        need = 40 * est_nnz(wl_g)
        avail = mem_available()
        if avail is None or need < 0.6 * avail:
            workload, note = wl_g, f"global matrix of the {world}-GPU weak-scaling run"
        else:
            note = (f"1-GPU workload: the {world}x matrix needs ~{need / 1e9:.0f} GB of host RAM, "
                    f"{avail / 1e9:.0f} GB available")
    r = reference_cpu(workload, bench_x(workload_n(workload)), 0.0, steps=args.steps,
                      warmup=args.warmup)
    ms = r["mean_ms"]
    gf = 2.0 * r["nnz"] / (ms * 1e6)
    model, ncpu = cpu_info()
    sample = (f"full {workload_name} matrix ({note}, nnz={r['nnz']}), reference csr5::spmv_csr5 "
              f"omega={r['omega']} sigma={r['sigma']} deterministic, one call per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": gf, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name, "desc": workload["desc"], "nnz": r["nnz"],
                   "m": r["m"], "omega": r["omega"], "sigma": r["sigma"], "mode": "deterministic"},
        "cpu_baseline": {"value": gf, "unit": UNIT, "cores": r["threads"], "kind": "reference",
                         "sample": sample, "cpu_model": model, "nproc": ncpu,
                         "conv_ms": r["conv_ms"], "conv_spmv_equiv": r["conv_ms"] / ms,
                         "csr_scalar_gflops": 2.0 * r["nnz"] / (r["csr_scalar_ms"] * 1e6)},
        "e2e": {"value": gf, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def run_ours(args, workload_name, workload):
    import numpy as np
    import torch

    from paper_1503_05032_b200 import csr5, mg
    from paper_1503_05032_b200.synthetic import bench_x
    rank, world, local = dist_env()
    if world > 1:
        # a rank that never sees a peer's flag would block its stream forever:
        # turn such a hang into a loud failure (the whole run takes minutes)
        limit = float(os.environ.get("CSR5G_WATCHDOG_S", "300"))

        def _watchdog():
            time.sleep(limit)
            sys.stderr.write(f"bench.py rank {rank}: no completion after {limit:.0f} s "
                             "(multi-GPU exchange stalled?); aborting\n")
            sys.stderr.flush()
            os._exit(3)

        threading.Thread(target=_watchdog, daemon=True).start()
    if os.environ.get("CSR5G_SHARE_GPU") == "1":  # functional multi-rank check on one GPU
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # NCCL over NVLink; CSR5G_DIST_BACKEND=gloo lets several ranks share one
        # GPU for a functional check of the sharded flow (not a timing)
        backend = os.environ.get("CSR5G_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    from paper_1503_05032_b200.synthetic import WorkloadMatrix, make_matrix, scaled_workload
    if world == 1:
        a = make_matrix(workload, dev)
        m, n, nnz = a.m, a.n, a.nnz
    else:
        # weak: the global matrix is `world` times the 1-GPU one; strong: the
        # 1-GPU matrix itself.  Either way each rank generates the global
        # row_ptr and only its own slice of entries where the generator allows.
        if args.scaling == "weak":
            workload = scaled_workload(workload, world)
        W = WorkloadMatrix(workload, dev)
        m, n, nnz = W.m, W.n, W.nnz
    torch.cuda.synchronize()
    x_host = bench_x(n)
    x = torch.as_tensor(x_host).to(dev)
    y = torch.empty(m, dtype=torch.float64, device=dev)
    sigma = csr5.select_sigma(nnz / m)

    # -- conversion (device-resident CSR -> usable CSR5), timed twice --------
    if world == 1:
        a5 = csr5.csr_to_csr5(a, csr5.TuningParams(sigma=sigma))
        a5.release()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a5 = csr5.csr_to_csr5(a, csr5.TuningParams(sigma=sigma))
        conv_ms = (time.perf_counter() - t0) * 1e3
        info = a5.info
        run = lambda: csr5.spmv_csr5(a5, x, y)  # noqa: E731
    else:
        lo, hi = mg.Csr5Sharded.slices_for(nnz, sigma, rank, world)
        col_s, val_s = W.entries(lo, hi)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sh = mg.Csr5Sharded(W.row_ptr, col_s, val_s, m, n, nnz, sigma, rank, world,
                            iterative=args.iterative and m == n)
        torch.cuda.synchronize()
        conv_ms = (time.perf_counter() - t0) * 1e3
        del col_s, val_s
        a5 = sh.a5
        info = a5.info if a5 is not None else None
        run = lambda: sh.spmv(x, y)  # noqa: E731

    # -- correctness guard before timing (bench.cpp:130-141 analogue) --------
    # y over the rows this rank writes, against cuSPARSE (torch sparse CSR)
    run()
    torch.cuda.synchronize()
    if world == 1:
        own = (0, m)
        rp_own, col_own, val_own = a.row_ptr, a.col_idx, a.val
    else:
        own = sh.own
        rp_own = W.row_ptr[own[0]:own[1] + 1]
        e0, e1 = (int(rp_own[0]), int(rp_own[-1])) if own[1] > own[0] else (0, 0)
        col_own, val_own = W.entries(e0, e1)
        rp_own = rp_own - e0
    err = 0.0
    if own[1] > own[0]:
        A = torch.sparse_csr_tensor(rp_own, col_own.long(), val_own, (own[1] - own[0], n))
        y_chk = (A @ x.unsqueeze(1)).squeeze(1)
        err = ((y[own[0]:own[1]] - y_chk).abs() / y_chk.abs().clamp(min=1.0)).max().item()
        del A, y_chk
    del rp_own, col_own, val_own
    if world > 1:
        W.drop()
    if not err <= 1e-12:
        raise SystemExit(f"correctness guard: max relative error {err} > 1e-12")
    it_ctr = [0]
    if world > 1 and sh.iterative:
        # fused y -> x (p2p.cu): one step from x must leave every active rank
        # with the same x_1, whose owned rows are the y just checked (bit for bit)
        sh.x_buffer(0).copy_(x)
        x1 = sh.spmv_iter(0)
        it_ctr[0] = 1
        torch.cuda.synchronize()
        same = bool(torch.equal(x1[own[0]:own[1]], y[own[0]:own[1]])) if sh.active else True
        h = torch.tensor([int(sh.active), int(same),
                          int(x1.view(torch.int64).sum().item()) if sh.active else 0],
                         dtype=torch.int64, device=dev if dist.get_backend() == "nccl" else "cpu")
        hs = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        act = [v for v in hs if int(v[0])]
        if not all(int(v[1]) for v in act) or len({int(v[2]) for v in act}) != 1:
            raise SystemExit("correctness guard: fused iterative x_1 differs between ranks or from y")
        if sh.mailbox_errors():
            raise SystemExit("correctness guard: P2P mailbox protocol errors")

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64,
                         device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    # L2 flushed between timed calls (a 2x-L2 read outside the events), so no
    # step starts with x or the matrix left in L2 by the previous one; a read
    # leaves clean lines, so the next call pays no write-back for the flush
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    scrub = torch.empty(2 * l2_bytes // 8 + 1, dtype=torch.float64, device=dev)

    for _ in range(args.warmup):
        run()
    steps_ev = [(csr5.Event(), csr5.Event()) for _ in range(args.steps)]
    tk = [(csr5.Event(), csr5.Event()) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    # the steps: the public call alone between the events (iterative mode:
    # plus y -> x, the all-gather of the owned ranges at N>1)
    if args.iterative:
        if m != n:
            raise SystemExit("--iterative needs a square matrix")
        x_keep = x.clone()
        bufs = [x, y]

        def step():
            if world == 1:  # ping-pong: y of this step is x of the next
                csr5.spmv_csr5(a5, bufs[0], bufs[1])
                bufs.reverse()
            elif sh.iterative:  # fused: the SpMV stores y into every rank's next x
                sh.spmv_iter(it_ctr[0])
                it_ctr[0] += 1
            else:
                run()
                sh.gather_y_into_x(y, x)
    else:
        step = run
    for k in range(args.steps):
        if scrub is not None:
            scrub.sum()  # read-only flush: evicts without leaving dirty lines
        steps_ev[k][0].record()
        step()
        steps_ev[k][1].record()
    if args.iterative:
        x.copy_(x_keep)
        del x_keep
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    # the dominant kernel for the roofline: the same steps again with events
    # recorded around the tile kernel on its stream
    for k in range(args.steps):
        if scrub is not None:
            scrub.sum()  # read-only flush: evicts without leaving dirty lines
        if world == 1:
            csr5.spmv_csr5_evt(a5, x, y, tk[k][0], tk[k][1])
        elif a5 is not None:
            sh.spmv(x, y, events=tk[k])
        else:
            run()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = max_over_ranks(sum(b.elapsed_ms(e) for b, e in steps_ev))
    ms = total_ms / args.steps
    tile_all = sorted(b.elapsed_ms(e) for b, e in tk) if a5 is not None else None
    tile_ms = (sum(tile_all) / args.steps) if tile_all else None

    # -- end to end through the host-buffer call ------------------------------
    # Every step moves its own x in from pinned host memory and its y out.
    # N=1: csr5.spmv_host_batch (csr5g_spmv_host_batch), which pipelines step
    # k+1's x H2D and step k's y D2H around SpMV k on separate copy engines.
    # The serial form (H2D, SpMV, D2H back to back on one stream) is reported
    # beside it.  N>1: the serial form through the sharded driver.
    ring = min(args.steps, 4)
    xh = [torch.as_tensor(x_host).pin_memory() for _ in range(ring)]
    yh = [torch.empty(m, dtype=torch.float64).pin_memory() for _ in range(ring)]

    def e2e_serial(k):
        x.copy_(xh[k % ring], non_blocking=True)
        run()
        yh[k % ring].copy_(y, non_blocking=True)

    def e2e_timed(fn):
        e0, e1 = csr5.Event(), csr5.Event()
        torch.cuda.synchronize()
        barrier()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_ms(e1)) / args.steps

    for k in range(args.warmup):
        e2e_serial(k)
    e2e_serial_ms = e2e_timed(lambda: [e2e_serial(k) for k in range(args.steps)])
    e2e_path = "serial: pinned x H2D + spmv + y D2H per step, one stream, CUDA events"
    e2e_ms = e2e_serial_ms
    e2e_trials = None
    pcie_ms = None
    if world == 1:
        xs = [xh[k % ring] for k in range(args.steps)]
        ys = [yh[k % ring] for k in range(args.steps)]
        csr5.spmv_host_batch(a5, xs[:args.warmup], ys[:args.warmup])
        # three runs of the K-step batch, the median reported: a single run
        # is exposed to host-side PCIe hiccups (one default run on a fresh box
        # saw its copies alone 10% slower and the batch 60% slower)
        e2e_trials = sorted(e2e_timed(lambda: csr5.spmv_host_batch(a5, xs, ys)) for _ in range(3))
        e2e_ms = e2e_trials[1]
        e2e_path = ("csr5.spmv_host_batch (csr5g_spmv_host_batch): per step pinned x H2D + SpMV + "
                    "y D2H, x_{k+1} H2D and y_k D2H overlapping SpMV k; CUDA events on the "
                    "caller stream")
        err_h = float(np.max(np.abs(yh[(args.steps - 1) % ring].numpy() - y.cpu().numpy())))
        if err_h != 0.0:
            raise SystemExit(f"host-batch path differs from the device path by {err_h}")
        # the PCIe ceiling of this e2e: the same per-step copies (x in, y out,
        # concurrently on two streams) with no SpMV at all
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        xd2, yd2 = torch.empty_like(x), y.clone()

        def duplex():
            cur = torch.cuda.current_stream()
            s_in.wait_stream(cur)
            s_out.wait_stream(cur)
            for k in range(args.steps):
                with torch.cuda.stream(s_in):
                    xd2.copy_(xh[k % ring], non_blocking=True)
                with torch.cuda.stream(s_out):
                    yh[k % ring].copy_(yd2, non_blocking=True)
            cur.wait_stream(s_in)
            cur.wait_stream(s_out)

        duplex()
        pcie_ms = sorted(e2e_timed(duplex) for _ in range(3))[1]

    # -- iteration scenario (bench.cpp:86-90, 164-175): the GPU plain-CSR
    # baseline beside CSR5, conversion amortised over n solver iterations ----
    iteration = None
    if world == 1:
        from paper_1503_05032_b200.benchmark import iteration_speedup
        # every comparator timed like the CSR5 step: L2 flushed before each call
        # (a read of 2x L2), CUDA events around the call alone
        def timed_flushed(fn, reps=5):
            fn()
            tot = 0.0
            for _ in range(reps):
                scrub.sum()
                b, e = csr5.Event(), csr5.Event()
                b.record()
                fn()
                e.record()
                torch.cuda.synchronize()
                tot += b.elapsed_ms(e)
            return tot / reps

        t_csr = {}
        for k in ("csr-scalar", "csr-segsum"):
            try:
                t_csr[k] = timed_flushed(lambda: csr5.spmv_csr(a, x, y, kernel=k))
            except MemoryError:
                t_csr[k] = None
        # library comparator: cuSPARSE csrmv through torch sparse CSR (int64
        # indices, so it moves 16 B per nonzero to our 12)
        t_lib = None
        try:
            A = torch.sparse_csr_tensor(a.row_ptr, a.col_idx.long(), a.val, (m, n))
            xc = x.unsqueeze(1)
            t_lib = timed_flushed(lambda: A @ xc)
            del A, xc
        except Exception:
            pass
        if t_csr["csr-scalar"]:
            iteration = {"t_cusparse_csrmv_ms": t_lib,"t_csr_scalar_ms": t_csr["csr-scalar"],
                         "t_csr_segsum_ms": t_csr["csr-segsum"], "t_csr5_ms": ms,
                         "t_conv_ms": conv_ms,
                         "speedup_n50": iteration_speedup(t_csr["csr-scalar"], conv_ms, ms, 50),
                         "speedup_n500": iteration_speedup(t_csr["csr-scalar"], conv_ms, ms, 500),
                         "baseline": "GPU csr-scalar (one thread per row), spmv.cpp:139-154"}
        # ingest: device COO -> CSR (csr.cpp:35-72) of this matrix's entries in
        # a random order (sort + duplicate merge + row_ptr)
        try:
            g = torch.Generator(device=dev).manual_seed(1)
            perm = torch.randperm(nnz, device=dev, generator=g)
            rows = torch.repeat_interleave(torch.arange(m, device=dev),
                                           a.row_ptr[1:] - a.row_ptr[:-1])[perm]
            cols = a.col_idx.long()[perm]
            vals = a.val[perm]
            del perm
            csr5.coo_to_csr(rows, cols, vals, m, n, device=dev)  # warm the pool
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            c2 = csr5.coo_to_csr(rows, cols, vals, m, n, device=dev)
            torch.cuda.synchronize()
            ingest_ms = (time.perf_counter() - t0) * 1e3
            same = bool(torch.equal(c2.row_ptr, a.row_ptr) and torch.equal(c2.col_idx, a.col_idx)
                        and torch.equal(c2.val, a.val))
            iteration["ingest"] = {"coo_to_csr_ms": ingest_ms, "entries": nnz,
                                   "order": "random permutation", "equals_generator_csr": same}
            del rows, cols, vals, c2
        except (MemoryError, RuntimeError, TypeError) as e:
            if iteration is not None:
                iteration["ingest"] = {"error": str(e)[:200]}
        # gather ceiling: the same nnz x-gathers alone (torch.index_select over
        # this matrix's col_idx, a library kernel) -- what the x traffic costs
        # without the matrix stream and the reduction
        try:
            idx = a.col_idx.long()
            xs = x.index_select(0, idx)
            iteration["gather_only_ms"] = timed_flushed(
                lambda: torch.index_select(x, 0, idx, out=xs))
            del idx, xs
        except (MemoryError, RuntimeError, TypeError):
            pass
        run()  # leave y = the CSR5 result for the CPU comparison below
        torch.cuda.synchronize()

    flops = 2.0 * nnz
    value = flops / (ms * 1e6)
    peak, peak_src = peaks()
    line = None
    if rank == 0:
        bytes_alg = info.spmv_bytes
        roof = None
        if tile_ms:
            achieved = bytes_alg / (tile_ms * 1e-3) / 1e9
            traffic = ncu_traffic(workload_name)
            if iteration and iteration.get("gather_only_ms"):
                iteration["gather_only_over_kernel"] = iteration["gather_only_ms"] / tile_ms
            roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "kernel": "k_spmv (tile kernel)", "kernel_ms": tile_ms,
                    "kernel_ms_best": tile_all[0],
                    "kernel_ms_median": tile_all[len(tile_all) // 2],
                    "algorithmic_bytes": bytes_alg, "peak_source": peak_src,
                    "frac_of_8TBs_spec": achieved / 8000.0}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                r = reference_cpu(workload, x_host, budget_s=args.cpu_seconds, also_w32=True)
                model, ncpu = cpu_info()
                yr = r.pop("y")
                w32 = r.pop("w32")
                cpu = {"value": 2.0 * r["nnz"] / (r["best_ms"] * 1e6), "unit": UNIT,
                       "cores": r["threads"], "kind": "reference",
                       "sample": (f"full {workload_name} matrix, reference csr5::spmv_csr5 "
                                  f"omega={r['omega']} sigma={r['sigma']} deterministic; best of "
                                  f"{len(r['samples'])} samples x {r['inner']} calls"),
                       "cpu_model": model, "nproc": ncpu, "conv_ms": r["conv_ms"],
                       # the reference's own widths (8 B val + 8 B
                       # col_idx), x and y once; its small metadata excluded
                       "gbs_ref_widths": (16 * r["nnz"] + 8 * (m + n)) / (r["best_ms"] * 1e6),
                       "conv_spmv_equiv": r["conv_ms"] / r["best_ms"],
                       "csr_scalar_gflops": 2.0 * r["nnz"] / (r["csr_scalar_ms"] * 1e6),
                       "y_max_rel_err_vs_gpu": float(np.max(np.abs(yr - y.cpu().numpy()) /
                                                            np.maximum(1.0, np.abs(yr)))),
                       "omega32": {"sigma": w32["sigma"],
                                   "gflops": 2.0 * r["nnz"] / (w32["best_ms"] * 1e6),
                                   "conv_ms": w32["conv_ms"],
                                   "sample": f"best of 3 samples x {w32['inner']} calls"}}
            except Exception as e:  # the CPU number is reported, never gating
                cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                       "sample": f"failed: {e}"}
        launches_per_step = 1
        if world > 1 and sh.active:
            if sh.exchange == "p2p":
                sb, se = sh.senders[sh.rank]
                launches_per_step += int(se > sb) + int(bool(args.iterative and sh.iterative))
            else:
                launches_per_step += 1
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name, "desc": workload["desc"], "m": m, "n": n,
                       "nnz": nnz, "omega": 32, "sigma": sigma, "p": info.p,
                       "desc_word_bits": info.word_bits, "mode": "deterministic",
                       "step": (("iterative: SpMV with y stored into every rank's next x over "
                                 "NVLink (fused, p2p.cu)" if world > 1 and sh.iterative else
                                 "iterative: SpMV + y->x all-gather") if args.iterative else
                                "SpMV (+ boundary exchange at N>1)"),
                       "exchange": (os.environ.get("CSR5G_EXCHANGE", "p2p") if world > 1
                                    else None),
                       "spmv_plan": {"lines_per_gather": round(info.lines_per_gather, 2),
                                     "warps_per_cta": info.warps_per_cta, "stages": info.stages,
                                     "smem_bytes": info.smem_bytes, "x_mode": info.x_mode,
                                     "x_l2_window": info.x_window,
                                     "kernel_variant": ["general", "VR", "NF"][info.kernel_variant]},
                       "parallelism": f"tile-range shards x{world}, x replicated",
                       "l2": (f"L2 flushed between timed calls ({2 * l2_bytes / 1e6:.0f} MB "
                              f"read outside the events); working set "
                              f"{info.spmv_bytes / 1e6:.0f} MB per SpMV"),
                       "x": "mt19937_64(1), 0.5 + (rng()>>11)*2^-53 (bench.cpp:103-105)"},
            "gbs_effective": info.spmv_bytes * world / (ms * 1e-3) / 1e9 if world == 1 else None,
            "roofline": roof,
            "conversion": {"ms": conv_ms, "alloc_ms": info.alloc_ms,
                           "spmv_equiv": conv_ms / ms,
                           "spmv_equiv_excl_alloc": (conv_ms - info.alloc_ms) / ms},
            "cpu_baseline": cpu,
            "iteration": iteration,
            "e2e": {"value": flops / (e2e_ms * 1e6), "unit": UNIT,
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * m,
                    "ms_per_step": e2e_ms, "path": e2e_path,
                    "trials_ms_per_step": e2e_trials,  # N=1: median of three K-step runs
                    "serial_value": flops / (e2e_serial_ms * 1e6),
                    "pcie_duplex_ms_per_step": pcie_ms if world == 1 else None,
                    "frac_of_pcie_duplex": (pcie_ms / e2e_ms) if world == 1 else None,
                    "serial_ms_per_step": e2e_serial_ms},
            # our kernels per step: the SpMV (calibration inside it); at N>1 plus
            # the P2P fix-up on an owner with senders and, fused iterative, the
            # ready signal (collective exchange: plus k_fixup)
            "gpu_launches": args.steps * launches_per_step,
            "clocks": clk,
            "correctness_max_rel_err": err,
        }
        print(json.dumps(line), flush=True)
    a5 = None
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return line


def main():
    from paper_1503_05032_b200.synthetic import WORKLOADS
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="st27_200")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--iterative", action="store_true",
                    help="y -> x mode (square A): each step is SpMV plus the all-gather of y "
                         "into every rank's x (N=1: x and y swap roles every step)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="N>1: weak = the global matrix is N times the 1-GPU workload (stencils "
                         "N times deeper, graphs log2 N scales larger); strong = the same matrix")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, args.workload, wl)
    else:
        run_ours(args, args.workload, wl)


if __name__ == "__main__":
    main()
