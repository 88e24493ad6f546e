#!/usr/bin/env python
"""CSR5 fp64 SpMV benchmark on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload rmat27]
    python bench.py --impl reference ...        # the reference's CPU path

One step = one CSR5 SpMV y = A x over the whole matrix (one pass of the hot
path).  The workload at every N is BASELINE config 5, R-MAT scale 27 edge
factor 16 (2^27 rows, 2.115G nonzeros after de-duplication, vertices
permuted, sigma = 16): the largest single-GPU configuration and the one the
1/2/4/8-GPU curve is quoted on.  Under torchrun (N>1) the matrix is
tile-range sharded over the ranks with x replicated (--scaling strong: the
same global matrix at every N, each rank generating only its slice); a step
includes the boundary-row exchange (NVLink P2P stores into the owner's
mailbox, p2p.cu; no collective).

At N=1 the line also carries `sub_results` for the other BASELINE configs
(27-point stencil 200^3, R-MAT s24, mixed 2^23, 2D Laplacian 1000^2), each
measured the same way with its own roofline, conversion, e2e and CPU
baseline (--sub none skips them).

`value` is GFLOP/s = 2*nnz / t with A and x resident in HBM; t is the max over
ranks of CUDA-event time on the launching stream.  L2 is flushed between timed
calls (2x L2 read outside the events).  `e2e` is the same metric through
the host-buffer call (csr5.spmv_host_batch): per step pinned x H2D + SpMV + y
D2H, pipelined across steps on separate copy engines.  The roofline
figure is for the SpMV's kernels (events around the hot-x staging, when the
plan has one, and the tile kernel), with the algorithmic bytes of SURVEY
8(d); `traffic` is the ncu-measured DRAM bytes of one tile-kernel launch
(profiles/ncu_traffic.json).
"""
from __future__ import annotations

import argparse
import gc
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
DEFAULT_WORKLOAD = "rmat27"
SUB_WORKLOADS = ("st27_200", "rmat24", "mixed23", "lap5_1000")


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


def pin_openmp():
    """SURVEY 8d / BASELINE.md §3: the reference's OpenMP threads pinned one per
    core.  Set before the reference library (and its libgomp) is loaded."""
    os.environ.setdefault("OMP_PLACES", "cores")
    os.environ.setdefault("OMP_PROC_BIND", "close")


# --------------------------------------------------------------------------
# the reference's CPU path (oracle/_ref = the unmodified reference library)
# --------------------------------------------------------------------------
def host_matrix(workload: dict):
    """The workload's CSR on the host with the reference's int64 indices.
    Stencils come from the host generator (oracle/testgen.c, no GPU needed);
    the graph workloads are generated on the device and copied back."""
    import numpy as np
    import torch

    from oracle.oracle import Csr, Oracle, stencil
    if workload["gen"] == "stencil":
        return stencil(Oracle(), workload["kind"], workload["a"], workload.get("layers"))
    from paper_1503_05032_b200.synthetic import make_matrix
    d = make_matrix(workload, "cuda")
    rp = d.row_ptr.cpu().numpy()
    col = np.empty(d.nnz, dtype=np.int64)
    step = 1 << 28  # int32 -> int64 in slices (no whole int32 host copy)
    for lo in range(0, d.nnz, step):
        col[lo:lo + step] = d.col_idx[lo:lo + step].cpu().numpy()
    val = d.val.cpu().numpy()
    m, n = d.m, d.n
    del d
    torch.cuda.empty_cache()
    return Csr(m, n, rp, col, val)


def workload_n(workload: dict) -> int:
    if workload["gen"] == "stencil":
        return workload["a"] ** (2 if workload["kind"] == 1 else 1) * workload.get("layers",
                                                                                 workload["a"])
    return 1 << (workload["scale"] if workload["gen"] == "rmat" else workload["log2_m"])


def reference_cpu(workload: dict, x, budget_s: float, configs=((4, 16),), steps=None, warmup=0):
    """Time the reference csr5::spmv_csr5 (deterministic) on the host cores,
    once per (omega, sigma) in `configs` (sigma 0 = the reference's own
    select_sigma rule).  Handles are built one at a time and the host CSR is
    dropped as soon as the last one exists (R-MAT s27 in the reference's
    int64 form is ~35 GB per copy).

    steps=None: the bench.cpp:147-160 protocol (samples of `inner` back-to-back
    calls, best sample reported) within ~budget_s per config.  steps=K: K single
    calls after `warmup` calls (the --impl reference step loop)."""
    import ctypes

    import numpy as np

    from oracle.oracle import Oracle, Ref
    ref = Ref()
    t0 = time.time()
    a = host_matrix(workload)
    gen_s = time.time() - t0
    m, n, nnz = a.m, a.n, a.nnz
    dp = ctypes.POINTER(ctypes.c_double)
    xv = ref.L.ref_vec_new(np.ascontiguousarray(x).ctypes.data_as(dp), n)
    out = []
    y = np.zeros(m)
    yp = y.ctypes.data_as(dp)
    for ci, (omega, sigma) in enumerate(configs):
        if sigma == 0:
            sigma = Oracle().select_sigma(nnz / max(m, 1))
        h, conv_ms = ref.build_handle(a, omega, sigma)
        if ci == len(configs) - 1:
            a = None  # the handle holds its own copy of the CSR
            gc.collect()
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
        scalar = ref.L.ref_time_csr_scalar(h, xv, yp, 2) if ci == 0 else None
        ref.L.ref_time_spmv(h, xv, yp, 0, 1)  # leave y = the csr5 result
        ref.L.ref_free(h)
        out.append(dict(omega=omega, sigma=sigma, best_ms=min(samples),
                        mean_ms=sum(samples) / len(samples), samples=samples, inner=inner,
                        conv_ms=conv_ms, csr_scalar_ms=scalar))
    ref.L.ref_vec_free(xv)
    return dict(nnz=nnz, m=m, n=n, gen_s=gen_s, threads=ref.max_threads(), runs=out, y=y)


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


def host_fits(wl: dict) -> tuple[bool, str]:
    """Can the host hold the reference's copies of this matrix?  ~56 B per
    nonzero at the peak: the int64 CSR handed over, the reference's own copy
    and the Csr5Matrix being built."""
    need = 56 * est_nnz(wl)
    avail = mem_available()
    if avail is None or need < 0.85 * avail:
        return True, ""
    return False, (f"needs ~{need / 1e9:.0f} GB of host RAM for the reference's copies, "
                   f"{avail / 1e9:.0f} GB available")


def run_reference(args, workload_name, workload):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    compiled from /root/reference/proj/core/src) on all host threads, OpenMP
    pinned; rank 0 only under torchrun.  Both its CPU default (omega=4,
    sigma=16, tuning.hpp:14-15) and the GPU's omega=32 / sigma=auto are
    stepped; `value` is the faster of the two."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1503_05032_b200.synthetic import WORKLOADS, bench_x, scaled_workload
    note = "the benchmark workload"
    if world > 1 and args.scaling == "weak":
        workload, note = scaled_workload(workload, world), f"global matrix of the {world}-GPU run"
    ok, why = host_fits(workload)
    if not ok:  # fall back to the largest graph config the host holds
        workload_name, workload = "rmat24", WORKLOADS["rmat24"]
        note = f"R-MAT s24 instead: {why}"
    r = reference_cpu(workload, bench_x(workload_n(workload)), 0.0,
                      configs=((4, 16), (32, 0)), steps=args.steps, warmup=args.warmup)
    model, ncpu = cpu_info()
    runs = r["runs"]
    gf = [2.0 * r["nnz"] / (q["mean_ms"] * 1e6) for q in runs]
    best = max(range(len(runs)), key=lambda i: gf[i])
    q = runs[best]
    ms = q["mean_ms"]
    sample = (f"full {workload_name} matrix ({note}, nnz={r['nnz']}), reference csr5::spmv_csr5 "
              f"deterministic, one call per step; omega/sigma {runs[0]['omega']}/"
              f"{runs[0]['sigma']} (its CPU default) and {runs[1]['omega']}/{runs[1]['sigma']} "
              f"(the GPU's), the faster reported")
    line = {
        "impl": "reference", "metric": METRIC, "value": gf[best], "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_name, "desc": workload["desc"], "nnz": r["nnz"],
                   "m": r["m"], "omega": q["omega"], "sigma": q["sigma"],
                   "mode": "deterministic"},
        "cpu_baseline": {"value": gf[best], "unit": UNIT, "cores": r["threads"],
                         "kind": "reference", "sample": sample, "cpu_model": model,
                         "nproc": ncpu,
                         "omp": {k: os.environ.get(k) for k in ("OMP_PLACES", "OMP_PROC_BIND")},
                         "runs": [{"omega": p["omega"], "sigma": p["sigma"], "gflops": g,
                                   "ms_per_step": p["mean_ms"], "conv_ms": p["conv_ms"],
                                   "conv_spmv_equiv": p["conv_ms"] / p["mean_ms"]}
                                  for p, g in zip(runs, gf)],
                         "csr_scalar_gflops": 2.0 * r["nnz"] / (runs[0]["csr_scalar_ms"] * 1e6)},
        "e2e": {"value": gf[best], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args, name, wl, x_host, y_gpu):
    """The reference on the host cores of this box, a bounded sample: both
    configurations, best of a few samples each (bench.cpp:147-160)."""
    import numpy as np
    ok, why = host_fits(wl)
    if not ok:
        return {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                "sample": f"skipped: {why}"}
    try:
        budget = args.cpu_seconds if name == args.workload else args.cpu_seconds / 2
        r = reference_cpu(wl, x_host, budget_s=budget, configs=((4, 16), (32, 0)))
    except Exception as e:  # the CPU number is reported, never gating
        return {"value": None, "unit": UNIT, "cores": None, "kind": "reference",
                "sample": f"failed: {e}"}
    model, ncpu = cpu_info()
    yr = r.pop("y")
    d, w32 = r["runs"]
    return {"value": 2.0 * r["nnz"] / (d["best_ms"] * 1e6), "unit": UNIT,
            "cores": r["threads"], "kind": "reference",
            "sample": (f"full {name} matrix, reference csr5::spmv_csr5 omega={d['omega']} "
                       f"sigma={d['sigma']} deterministic; best of {len(d['samples'])} samples "
                       f"x {d['inner']} calls"),
            "cpu_model": model, "nproc": ncpu,
            "omp": {k: os.environ.get(k) for k in ("OMP_PLACES", "OMP_PROC_BIND")},
            "conv_ms": d["conv_ms"],
            # the reference's own widths (8 B val + 8 B col_idx), x
            # and y once; its small metadata excluded
            "gbs_ref_widths": (16 * r["nnz"] + 8 * (r["m"] + r["n"])) / (d["best_ms"] * 1e6),
            "conv_spmv_equiv": d["conv_ms"] / d["best_ms"],
            "csr_scalar_gflops": 2.0 * r["nnz"] / (d["csr_scalar_ms"] * 1e6),
            "y_max_rel_err_vs_gpu": float(np.max(np.abs(yr - y_gpu) /
                                                 np.maximum(1.0, np.abs(yr)))),
            "omega32": {"sigma": w32["sigma"],
                        "gflops": 2.0 * r["nnz"] / (w32["best_ms"] * 1e6),
                        "conv_ms": w32["conv_ms"],
                        "sample": f"best of {len(w32['samples'])} samples x {w32['inner']} calls"}}


# --------------------------------------------------------------------------
# our arm, one GPU
# --------------------------------------------------------------------------
def measure_one(args, name, workload, dev, local):
    """Every measurement of one workload on one GPU: conversion, correctness
    guard, K timed steps, the tile kernel's roofline, e2e through host buffers,
    comparators and the CPU baseline.  Returns the result dict."""
    import numpy as np
    import torch

    from paper_1503_05032_b200 import csr5
    from paper_1503_05032_b200.synthetic import bench_x, make_matrix
    a = make_matrix(workload, dev)
    m, n, nnz = a.m, a.n, a.nnz
    torch.cuda.synchronize()
    x_host = bench_x(n)
    x = torch.as_tensor(x_host).to(dev)
    y = torch.empty(m, dtype=torch.float64, device=dev)
    sigma = csr5.select_sigma(nnz / m)
    big = nnz > 1_000_000_000

    # -- conversion (device-resident CSR -> usable CSR5), timed twice --------
    a5 = csr5.csr_to_csr5(a, csr5.TuningParams(sigma=sigma))
    a5.release()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a5 = csr5.csr_to_csr5(a, csr5.TuningParams(sigma=sigma))
    conv_ms = (time.perf_counter() - t0) * 1e3
    info = a5.info
    run = lambda: csr5.spmv_csr5(a5, x, y)  # noqa: E731

    # -- correctness guard before timing (bench.cpp:130-141 analogue): y
    # against cuSPARSE (torch sparse CSR) --------------------------------------
    run()
    torch.cuda.synchronize()
    A = torch.sparse_csr_tensor(a.row_ptr, a.col_idx.long(), a.val, (m, n))
    y_chk = (A @ x.unsqueeze(1)).squeeze(1)
    err = ((y - y_chk).abs() / y_chk.abs().clamp(min=1.0)).max().item()
    del A, y_chk
    torch.cuda.empty_cache()
    if not err <= 1e-12:
        raise SystemExit(f"{name}: correctness guard: max relative error {err} > 1e-12")

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
    clocks.start()
    time.sleep(0.3)
    if args.iterative:  # ping-pong: y of this step is x of the next
        x_keep = x.clone()
        bufs = [x, y]

        def step():
            csr5.spmv_csr5(a5, bufs[0], bufs[1])
            bufs.reverse()
    else:
        step = run
    for k in range(args.steps):
        scrub.sum()  # read-only flush: evicts without leaving dirty lines
        steps_ev[k][0].record()
        step()
        steps_ev[k][1].record()
    if args.iterative:
        x.copy_(x_keep)
        del x_keep
    torch.cuda.synchronize()
    # the dominant kernel for the roofline: the same steps again with events
    # recorded around the tile kernel on its stream
    for k in range(args.steps):
        scrub.sum()
        csr5.spmv_csr5_evt(a5, x, y, tk[k][0], tk[k][1])
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = sum(b.elapsed_ms(e) for b, e in steps_ev) / args.steps
    tile_all = sorted(b.elapsed_ms(e) for b, e in tk)
    tile_ms = sum(tile_all) / args.steps

    # -- end to end through the host-buffer call ------------------------------
    # Every step moves its own x in from pinned host memory and its y out:
    # csr5.spmv_host_batch (csr5g_spmv_host_batch) pipelines step k+1's x H2D
    # and step k's y D2H around SpMV k on separate copy engines.  The serial
    # form (H2D, SpMV, D2H back to back on one stream) is reported beside it.
    ring = 2 if big else min(args.steps, 4)
    xh = [torch.as_tensor(x_host).pin_memory() for _ in range(ring)]
    yh = [torch.empty(m, dtype=torch.float64).pin_memory() for _ in range(ring)]

    def timed(fn):
        e0, e1 = csr5.Event(), csr5.Event()
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_ms(e1) / args.steps

    def e2e_serial(k):
        x.copy_(xh[k % ring], non_blocking=True)
        run()
        yh[k % ring].copy_(y, non_blocking=True)

    for k in range(min(args.warmup, 2)):
        e2e_serial(k)
    e2e_serial_ms = timed(lambda: [e2e_serial(k) for k in range(args.steps)])
    xs = [xh[k % ring] for k in range(args.steps)]
    ys = [yh[k % ring] for k in range(args.steps)]
    csr5.spmv_host_batch(a5, xs[:2], ys[:2])
    # three runs of the K-step batch, the median reported: a single run is
    # exposed to host-side PCIe hiccups
    e2e_trials = sorted(timed(lambda: csr5.spmv_host_batch(a5, xs, ys)) for _ in range(3))
    e2e_ms = e2e_trials[1]
    x.copy_(xh[0])
    run()
    torch.cuda.synchronize()
    err_h = float((yh[(args.steps - 1) % ring].to(dev) - y).abs().max().item())
    if err_h != 0.0:
        raise SystemExit(f"{name}: host-batch path differs from the device path by {err_h}")
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
    pcie_ms = sorted(timed(duplex) for _ in range(3))[1]
    del xh, yh, xs, ys, xd2, yd2

    # -- iteration scenario (bench.cpp:86-90, 164-175): the GPU plain-CSR
    # baseline beside CSR5, conversion amortised over n solver iterations ----
    from paper_1503_05032_b200.benchmark import iteration_speedup

    def timed_flushed(fn, reps=3):
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
        except (MemoryError, RuntimeError):
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
    torch.cuda.empty_cache()
    iteration = {"t_cusparse_csrmv_ms": t_lib, "t_csr_scalar_ms": t_csr["csr-scalar"],
                 "t_csr_segsum_ms": t_csr["csr-segsum"], "t_csr5_ms": ms, "t_conv_ms": conv_ms,
                 "baseline": "GPU csr-scalar (one thread per row), spmv.cpp:139-154"}
    if t_csr["csr-scalar"]:
        iteration["speedup_n50"] = iteration_speedup(t_csr["csr-scalar"], conv_ms, ms, 50)
        iteration["speedup_n500"] = iteration_speedup(t_csr["csr-scalar"], conv_ms, ms, 500)
    # ingest: device COO -> CSR (csr.cpp:35-72) of this matrix's entries in a
    # random order (sort + duplicate merge + row_ptr); skipped for the 2G-entry
    # graph, whose COO copies would not fit beside the matrix
    if not big:
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
            iteration["ingest"] = {"error": str(e)[:200]}
    # gather ceiling: the same nnz x-gathers alone (torch.index_select over this
    # matrix's col_idx, a library kernel) -- what the x traffic costs without
    # the matrix stream and the reduction
    try:
        idx = a.col_idx.long()
        xs_ = x.index_select(0, idx)
        iteration["gather_only_ms"] = timed_flushed(lambda: torch.index_select(x, 0, idx, out=xs_))
        iteration["gather_only_over_kernel"] = iteration["gather_only_ms"] / tile_ms
        del idx, xs_
    except (MemoryError, RuntimeError, TypeError):
        pass
    torch.cuda.empty_cache()
    run()  # leave y = the CSR5 result for the CPU comparison below
    torch.cuda.synchronize()
    y_host = y.cpu().numpy()
    plan = {"lines_per_gather": round(info.lines_per_gather, 2),
            "warps_per_cta": info.warps_per_cta, "stages": info.stages,
            "smem_bytes": info.smem_bytes, "x_mode": info.x_mode,
            "x_l2_window": info.x_window,
            "kernel_variant": ["general", "VR", "NF"][info.kernel_variant],
            "hot_x_cols": info.hot_cols, "hot_x_sampled_coverage": round(info.hot_coverage, 3)}
    launches_per_step = 2 if info.hot_cols > 0 else 1
    bytes_alg = info.spmv_bytes
    conv_alloc = info.alloc_ms
    p_tiles, word_bits = info.p, info.word_bits
    a5.release()
    del a5, a, x, y, scrub
    gc.collect()
    torch.cuda.empty_cache()

    peak, peak_src = peaks()
    achieved = bytes_alg / (tile_ms * 1e-3) / 1e9
    flops = 2.0 * nnz
    res = {
        "value": flops / (ms * 1e6), "unit": UNIT, "ms_per_step": ms,
        "config": {"workload": name, "desc": workload["desc"], "m": m, "n": n, "nnz": nnz,
                   "omega": 32, "sigma": sigma, "p": p_tiles, "desc_word_bits": word_bits,
                   "mode": "deterministic",
                   "step": "iterative: SpMV, y -> x" if args.iterative else "SpMV",
                   "spmv_plan": plan,
                   "l2": (f"L2 flushed between timed calls ({2 * l2_bytes / 1e6:.0f} MB read "
                          f"outside the events); working set {bytes_alg / 1e6:.0f} MB per SpMV"),
                   "x": "mt19937_64(1), 0.5 + (rng()>>11)*2^-53 (bench.cpp:103-105)"},
        "gbs_effective": bytes_alg / (ms * 1e-3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(name),
                     "kernel": ("k_xhot_fill + k_spmv (hot-x staging and tile kernel)"
                                if launches_per_step == 2 else "k_spmv (tile kernel)"),
                     "kernel_ms": tile_ms,
                     "kernel_ms_best": tile_all[0], "kernel_ms_median": tile_all[len(tile_all) // 2],
                     "algorithmic_bytes": bytes_alg, "peak_source": peak_src,
                     "frac_of_8TBs_spec": achieved / 8000.0},
        "conversion": {"ms": conv_ms, "alloc_ms": conv_alloc, "spmv_equiv": conv_ms / ms,
                       "spmv_equiv_excl_alloc": (conv_ms - conv_alloc) / ms},
        "iteration": iteration,
        "e2e": {"value": flops / (e2e_ms * 1e6), "unit": UNIT,
                "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * m,
                "ms_per_step": e2e_ms,
                "path": ("csr5.spmv_host_batch (csr5g_spmv_host_batch): per step pinned x H2D + "
                         "SpMV + y D2H, x_{k+1} H2D and y_k D2H overlapping SpMV k; CUDA events "
                         "on the caller stream"),
                "trials_ms_per_step": e2e_trials, "serial_value": flops / (e2e_serial_ms * 1e6),
                "serial_ms_per_step": e2e_serial_ms, "pcie_duplex_ms_per_step": pcie_ms,
                "frac_of_pcie_duplex": pcie_ms / e2e_ms},
        # one k_spmv per step (the calibration runs inside it), after the hot
        # columns' x staging (k_xhot_fill) when the plan has one
        "gpu_launches": args.steps * launches_per_step,
        "clocks": clk,
        "correctness_max_rel_err": err,
    }
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline(args, name, workload, x_host, y_host)
    return res


# --------------------------------------------------------------------------
# our arm, N GPUs (one process per GPU)
# --------------------------------------------------------------------------
def measure_sharded(args, name, workload, dev, local, dist, rank, world):
    import torch

    from paper_1503_05032_b200 import csr5, mg
    from paper_1503_05032_b200.synthetic import WorkloadMatrix, bench_x, scaled_workload
    # strong: the same global matrix at every N; weak: `world` times the
    # 1-GPU one.  Either way each rank generates the global row_ptr and only
    # its own slice of entries.
    if args.scaling == "weak":
        workload = scaled_workload(workload, world)
    W = WorkloadMatrix(workload, dev)
    m, n, nnz = W.m, W.n, W.nnz
    torch.cuda.synchronize()
    x_host = bench_x(n)
    x = torch.as_tensor(x_host).to(dev)
    y = torch.empty(m, dtype=torch.float64, device=dev)
    sigma = csr5.select_sigma(nnz / m)
    lo, hi = mg.Csr5Sharded.slices_for(nnz, sigma, rank, world, W.row_ptr)
    col_s, val_s = W.entries(lo, hi)
    # the shard's conversion timed on its second build, as at N = 1 (the first
    # maps the memory pool's pages)
    view = mg.shard_view(nnz, sigma, rank, world, W.row_ptr)
    if view is not None:
        csr5.csr_to_csr5_shard(W.row_ptr, col_s, val_s, m, n, nnz, csr5.TuningParams(sigma=sigma),
                               view.tile_begin, view.tile_end, view.with_tail).release()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sh = mg.Csr5Sharded(W.row_ptr, col_s, val_s, m, n, nnz, sigma, rank, world,
                        iterative=args.iterative and m == n)
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t0) * 1e3
    conv_ms = sh.a5.info.build_ms if sh.a5 is not None else 0.0
    del col_s, val_s
    a5 = sh.a5
    info = a5.info if a5 is not None else None
    run = lambda: sh.spmv(x, y)  # noqa: E731

    # -- correctness guard: this rank's owned rows of y against cuSPARSE ------
    run()
    torch.cuda.synchronize()
    own = sh.own
    err = 0.0
    if own[1] > own[0]:
        rp_own = W.row_ptr[own[0]:own[1] + 1]
        e0, e1 = int(rp_own[0]), int(rp_own[-1])
        col_own, val_own = W.entries(e0, e1)
        A = torch.sparse_csr_tensor(rp_own - e0, col_own.long(), val_own, (own[1] - own[0], n))
        y_chk = (A @ x.unsqueeze(1)).squeeze(1)
        err = ((y[own[0]:own[1]] - y_chk).abs() / y_chk.abs().clamp(min=1.0)).max().item()
        del A, y_chk, rp_own, col_own, val_own
    W.drop()
    torch.cuda.empty_cache()
    if not err <= 1e-12:
        raise SystemExit(f"correctness guard: max relative error {err} > 1e-12")
    it_ctr = [0]
    if sh.iterative:
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

    def max_over_ranks(v: float) -> float:
        t = torch.tensor([v], dtype=torch.float64,
                         device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    scrub = torch.empty(2 * l2_bytes // 8 + 1, dtype=torch.float64, device=dev)
    for _ in range(args.warmup):
        run()
    steps_ev = [(csr5.Event(), csr5.Event()) for _ in range(args.steps)]
    tk = [(csr5.Event(), csr5.Event()) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    if args.iterative:
        def step():
            if sh.iterative:  # fused: the SpMV stores y into every rank's next x
                sh.spmv_iter(it_ctr[0])
                it_ctr[0] += 1
            else:
                run()
                sh.gather_y_into_x(y, x)
    else:
        step = run
    x_keep = x.clone() if args.iterative else None
    for k in range(args.steps):
        scrub.sum()
        steps_ev[k][0].record()
        step()
        steps_ev[k][1].record()
    if x_keep is not None:
        x.copy_(x_keep)
        del x_keep
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        scrub.sum()
        if a5 is not None:
            sh.spmv(x, y, events=tk[k])
        else:
            run()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = max_over_ranks(sum(b.elapsed_ms(e) for b, e in steps_ev)) / args.steps
    tile_ms = (sum(b.elapsed_ms(e) for b, e in tk) / args.steps) if a5 is not None else 0.0
    tile_ms_max = max_over_ranks(tile_ms)

    # -- e2e: the serial form through the sharded driver ----------------------
    ring = 2
    xh = [torch.as_tensor(x_host).pin_memory() for _ in range(ring)]
    yh = [torch.empty(m, dtype=torch.float64).pin_memory() for _ in range(ring)]

    def e2e_serial(k):
        x.copy_(xh[k % ring], non_blocking=True)
        run()
        yh[k % ring][own[0]:own[1]].copy_(y[own[0]:own[1]], non_blocking=True)

    for k in range(min(args.warmup, 2)):
        e2e_serial(k)
    e0, e1 = csr5.Event(), csr5.Event()
    torch.cuda.synchronize()
    dist.barrier()
    e0.record()
    for k in range(args.steps):
        e2e_serial(k)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_ms(e1)) / args.steps
    del xh, yh

    flops = 2.0 * nnz
    peak, peak_src = peaks()
    line = None
    if rank == 0:
        launches = 1 + (1 if info is not None and info.hot_cols > 0 else 0)  # + hot-x staging
        if sh.active:
            if sh.exchange == "p2p":
                sb, se = sh.senders[sh.rank]
                launches += int(se > sb) + int(bool(args.iterative and sh.iterative))
            else:
                launches += 1
        bytes_alg = info.spmv_bytes
        achieved = bytes_alg / (tile_ms * 1e-3) / 1e9 if tile_ms else None
        line = {
            "metric": METRIC, "value": flops / (ms * 1e6), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": name, "desc": workload["desc"], "m": m, "n": n, "nnz": nnz,
                       "omega": 32, "sigma": sigma, "mode": "deterministic",
                       "step": (("iterative: SpMV with y stored into every rank's next x over "
                                 "NVLink (fused, p2p.cu)" if sh.iterative else
                                 "iterative: SpMV + y->x all-gather") if args.iterative else
                                "SpMV + boundary exchange"),
                       "exchange": os.environ.get("CSR5G_EXCHANGE", "p2p"),
                       # NVLink bytes each GPU sends per step (DESIGN §6 model):
                       # the boundary partial (16 B + flags) per shard edge, and in
                       # the fused iterative mode its owned rows of y to every peer
                       # (NVLS multicast: one multimem store per value, replicated
                       # by the switch -- 8 bytes per owned row leave the GPU)
                       "nvls_multicast": bool(getattr(sh, "mcast", False)),
                       "nvlink_out_bytes_per_step_per_gpu": (
                           (8 * (own[1] - own[0]) * (1 if getattr(sh, "mcast", False)
                                                     else world - 1))
                           if args.iterative and sh.iterative else 16 + 8),
                       "parallelism": f"tile-range shards x{world}, x replicated",
                       "l2": f"L2 flushed between timed calls ({2 * l2_bytes / 1e6:.0f} MB read)",
                       "x": "mt19937_64(1), 0.5 + (rng()>>11)*2^-53 (bench.cpp:103-105)"},
            "roofline": ({"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                          "frac": achieved / peak, "traffic": None,
                          "kernel": "k_spmv (rank 0's shard)", "kernel_ms": tile_ms,
                          "kernel_ms_max_over_ranks": tile_ms_max,
                          "algorithmic_bytes": bytes_alg, "peak_source": peak_src}
                         if achieved else None),
            "conversion": {"ms": conv_ms, "spmv_equiv": conv_ms / ms,
                           "what": "rank 0's shard build (second build); setup_ms adds the "
                                   "mailbox / IPC exchange setup",
                           "setup_ms": setup_ms},
            "cpu_baseline": None,
            "e2e": {"value": flops / (e2e_ms * 1e6), "unit": UNIT,
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * (own[1] - own[0]),
                    "ms_per_step": e2e_ms,
                    "path": "serial per rank: pinned x H2D + sharded SpMV + owned y D2H"},
            "gpu_launches": args.steps * launches,
            "clocks": clk,
            "correctness_max_rel_err": err,
        }
    sh.close()
    return line


def run_ours(args, workload_name, workload):
    import torch
    rank, world, local = dist_env()
    if world > 1:
        # a rank that never sees a peer's flag would block its stream forever:
        # turn such a hang into a loud failure (the whole run takes minutes)
        limit = float(os.environ.get("CSR5G_WATCHDOG_S", "600"))

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
    if world == 1:
        from paper_1503_05032_b200.synthetic import WORKLOADS
        res = measure_one(args, workload_name, workload, dev, local)
        line = {"metric": METRIC, "value": res.pop("value"), "unit": UNIT, "n_gpus": 1,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": res.pop("ms_per_step"),
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                "dtype": "f64", "data": "synthetic"}
        line.update(res)
        line["config"]["parallelism"] = "1 GPU (tile-range shards x1)"
        subs = {}
        for w in args.sub:
            if w == workload_name:
                continue
            r = measure_one(args, w, WORKLOADS[w], dev, local)
            r.pop("gpu_launches", None)
            subs[w] = r
        if subs:
            line["sub_results"] = subs
        print(json.dumps(line), flush=True)
        return line
    import torch.distributed as dist
    # NCCL over NVLink; CSR5G_DIST_BACKEND=gloo lets several ranks share one
    # GPU for a functional check of the sharded flow (not a timing)
    backend = os.environ.get("CSR5G_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    line = measure_sharded(args, workload_name, workload, dev, local, dist, rank, world)
    if line is not None:
        print(json.dumps(line), flush=True)
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
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD)
    ap.add_argument("--sub", default=",".join(SUB_WORKLOADS),
                    help="N=1: comma-separated workloads measured as sub_results ('none': skip)")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--iterative", action="store_true",
                    help="y -> x mode (square A): each step is SpMV plus the all-gather of y "
                         "into every rank's x (N=1: x and y swap roles every step)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                    help="N>1: strong = the same global matrix at every N (default); weak = the "
                         "global matrix is N times the 1-GPU workload (stencils N times deeper, "
                         "graphs log2 N scales larger)")
    args = ap.parse_args()
    args.sub = [] if args.sub in ("", "none") else [w for w in args.sub.split(",") if w]
    for w in args.sub:
        if w not in WORKLOADS:
            ap.error(f"--sub: unknown workload {w!r}")
    if args.warmup < 3:
        args.warmup = 3
    pin_openmp()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, args.workload, wl)
    else:
        run_ours(args, args.workload, wl)


if __name__ == "__main__":
    main()
