"""run_benchmark on the GPU: the reference's benchmark harness API
(proj/core/include/csr5/bench.hpp, src/bench.cpp) over the device kernels.

Same names, fields, protocol and errors as the reference:

* kernels csr-scalar / csr-segsum / csr5 (`parse_kernel_list`, bench.cpp:55-72);
* every kernel is checked against the dense-order reference before timing and
  raises `CorrectnessError` with the reference's message when
  `max_relative_error > oracle_tol` (bench.cpp:128-141); `corrupt_for_test`
  perturbs y[0] first, as the reference's test hook does;
* conversion is timed once and shared by every csr5 timing (bench.cpp:107-117);
* `warmup` untimed calls, then `runs` samples each averaging `inner_iters`
  calls; best / avg / GFLOP/s from the best sample (bench.cpp:147-162);
* the iteration scenario: speedup_n50 / speedup_n500 =
  `iteration_speedup(t_csr, t_conv, t_kernel, n)` against csr-scalar, or the
  first kernel when csr-scalar was not requested (bench.cpp:86-90, 164-175);
* `emit_csv`: the fixed header and `std::to_chars(general, 10)` numbers
  (bench.cpp:29-33, 177-195).

GPU differences, all in where the numbers come from rather than what they
mean: samples are CUDA-event times on the launching stream; the dense-order
reference y is the device csr-scalar kernel (one thread per row, row order --
the summation order of dense_spmv_oracle, csr.cpp:85-98); `threads` reports
the device's SM count; x comes from `bench_x(n, x_seed)` (bench.cpp:103-105).
"""
from __future__ import annotations

import enum
import time
from dataclasses import dataclass, field

import torch

from . import csr5
from .synthetic import bench_x


class KernelKind(enum.Enum):
    csr_scalar = "csr-scalar"
    csr_segsum = "csr-segsum"
    csr5 = "csr5"


class CorrectnessError(RuntimeError):
    """bench.hpp:19-24: a kernel disagrees with the dense reference."""


def kernel_name(kind: KernelKind) -> str:
    return kind.value


def parse_kernel_list(text: str) -> list[KernelKind]:
    """bench.cpp:55-72: comma-separated names, in order."""
    kernels = []
    for item in text.split(","):
        if item == "":
            continue  # empty items are skipped (bench.cpp:59)
        try:
            kernels.append(KernelKind(item))
        except ValueError:
            raise ValueError(f"unknown kernel '{item}' (expected csr-scalar, csr-segsum or "
                             f"csr5)") from None
    if not kernels:
        raise ValueError("empty kernel list")
    return kernels


def format_double(v: float) -> str:
    """std::to_chars(v, chars_format::general, 10) == printf("%.10g")."""
    return f"{v:.10g}"


def relative_error(value: float, reference: float) -> float:
    return abs(value - reference) / max(1.0, abs(reference))


def max_relative_error(y: torch.Tensor, reference: torch.Tensor) -> float:
    if y.numel() == 0:
        return 0.0
    return float(((y - reference).abs() / reference.abs().clamp(min=1.0)).max())


def iteration_speedup(t_csr: float, t_pre: float, t_new: float, n: int) -> float:
    """bench.cpp:86-90: n * t_csr / (t_pre + n * t_new)."""
    if t_csr <= 0.0 or t_new <= 0.0 or t_pre < 0.0 or n < 1:
        raise ValueError("iteration_speedup: times must be positive (t_pre >= 0), n >= 1")
    return n * t_csr / (t_pre + n * t_new)


@dataclass
class KernelResult:
    kernel: str
    sample_ms: list[float] = field(default_factory=list)
    best_ms: float = 0.0
    avg_ms: float = 0.0
    gflops: float = 0.0
    conv_ms: float = 0.0
    speedup_n50: float = 0.0
    speedup_n500: float = 0.0


@dataclass
class BenchReport:
    matrix: str
    m: int = 0
    n: int = 0
    nnz: int = 0
    threads: int = 1
    kernels: list[KernelResult] = field(default_factory=list)


@dataclass
class BenchConfig:
    kernels: list[KernelKind] = field(default_factory=lambda: [
        KernelKind.csr_scalar, KernelKind.csr_segsum, KernelKind.csr5])
    runs: int = 10
    inner_iters: int = 1000
    warmup: int = 10
    mode: str = "deterministic"
    params: csr5.TuningParams = field(default_factory=csr5.TuningParams)
    oracle_tol: float = 1e-10
    x_seed: int = 1
    corrupt_for_test: KernelKind | None = None


def run_benchmark(a: csr5.CsrMatrix, name: str, cfg: BenchConfig) -> BenchReport:
    """bench.cpp:92-176 on the device: validate, then time every kernel."""
    if cfg.runs < 1 or cfg.inner_iters < 1 or cfg.warmup < 0:
        raise ValueError("run_benchmark: runs and inner_iters must be >= 1")
    dev = a.row_ptr.device
    props = torch.cuda.get_device_properties(dev)
    report = BenchReport(matrix=name, m=a.m, n=a.n, nnz=a.nnz, threads=props.multi_processor_count)
    x = torch.as_tensor(bench_x(a.n, cfg.x_seed)).to(dev)
    y_ref = csr5.spmv_csr(a, x, kernel="csr-scalar")
    y = torch.zeros(a.m, dtype=torch.float64, device=dev)

    a5, conv_ms = None, 0.0
    if KernelKind.csr5 in cfg.kernels:
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        a5 = csr5.csr_to_csr5(a, cfg.params)
        torch.cuda.synchronize(dev)
        conv_ms = (time.perf_counter() - t0) * 1e3

    try:
        for kind in cfg.kernels:
            if kind == KernelKind.csr5:
                def call():
                    csr5.spmv_csr5(a5, x, y, mode=cfg.mode)
            else:
                def call(k=kind.value):
                    csr5.spmv_csr(a, x, y, kernel=k)
            call()
            if cfg.corrupt_for_test == kind and y.numel() > 0:
                y[0] += 1.0 + y[0].abs()
            err = max_relative_error(y, y_ref)
            if err > cfg.oracle_tol:
                raise CorrectnessError(
                    f"kernel {kind.value} disagrees with the dense reference on '{name}': max "
                    f"relative error {format_double(err)} exceeds {format_double(cfg.oracle_tol)}")
            res = KernelResult(kernel=kind.value,
                               conv_ms=conv_ms if kind == KernelKind.csr5 else 0.0)
            for _ in range(cfg.warmup):
                call()
            for _ in range(cfg.runs):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(cfg.inner_iters):
                    call()
                e1.record()
                e1.synchronize()
                res.sample_ms.append(e0.elapsed_time(e1) / cfg.inner_iters)
            res.best_ms = min(res.sample_ms)
            res.avg_ms = sum(res.sample_ms) / len(res.sample_ms)
            res.gflops = 2.0 * report.nnz / (res.best_ms * 1e6) if res.best_ms > 0.0 else 0.0
            report.kernels.append(res)
    finally:
        if a5 is not None:
            a5.release()

    baseline = next((k for k in report.kernels if k.kernel == "csr-scalar"), None)
    if baseline is None and report.kernels:
        baseline = report.kernels[0]
    for k in report.kernels:
        if baseline is None or baseline.best_ms <= 0.0 or k.best_ms <= 0.0:
            continue
        k.speedup_n50 = iteration_speedup(baseline.best_ms, k.conv_ms, k.best_ms, 50)
        k.speedup_n500 = iteration_speedup(baseline.best_ms, k.conv_ms, k.best_ms, 500)
    return report


CSV_HEADER = "matrix,m,n,nnz,kernel,threads,best_ms,avg_ms,gflops,conv_ms,speedup_n50,speedup_n500"


def emit_csv(report: BenchReport, out=None) -> str:
    """bench.cpp:177-195: the fixed header and one row per kernel.  `out` may
    be a path or a text stream; the CSV text is returned either way."""
    f = format_double
    lines = [CSV_HEADER]
    for k in report.kernels:
        lines.append(",".join([report.matrix, str(report.m), str(report.n), str(report.nnz),
                               k.kernel, str(report.threads), f(k.best_ms), f(k.avg_ms),
                               f(k.gflops), f(k.conv_ms), f(k.speedup_n50), f(k.speedup_n500)]))
    text = "\n".join(lines) + "\n"
    if isinstance(out, str):
        try:
            with open(out, "w") as fh:
                fh.write(text)
        except OSError:
            raise RuntimeError(f"emit_csv: cannot open '{out}'") from None
    elif out is not None:
        out.write(text)
    return text
