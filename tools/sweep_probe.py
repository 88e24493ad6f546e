"""Experiment helper (GPU box): k_spmv time of one workload under a list of
plan knobs, the matrix generated once.  Each configuration is a set of
CSR5G_* environment variables read when the handle's plan is made (NW,
STAGES, BUDGET_KB, XMODE, XWINDOW, VR, NF) or per launch (EARLY); the handle
is rebuilt for every configuration.  L2 scrubbed between calls (as bench.py).
    python tools/sweep_probe.py rmat27 "CSR5G_NW=8" "CSR5G_NW=12 CSR5G_EARLY=0" ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1503_05032_b200 import csr5  # noqa: E402
from paper_1503_05032_b200.synthetic import WORKLOADS, bench_x, make_matrix  # noqa: E402

name, configs = sys.argv[1], sys.argv[2:] or [""]
a = make_matrix(WORKLOADS[name])
x = torch.as_tensor(bench_x(a.n)).cuda()
y = torch.empty(a.m, dtype=torch.float64, device="cuda")
sigma = csr5.select_sigma(a.nnz / a.m)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
scrub = torch.empty(2 * l2 // 8, dtype=torch.float64, device="cuda")
base_env = dict(os.environ)
ref = None
for cfg in configs:
    os.environ.clear()
    os.environ.update(base_env)
    for kv in cfg.split():
        k, v = kv.split("=", 1)
        os.environ[k] = v
    if "L2_FETCH" in os.environ:  # cudaLimitMaxL2FetchGranularity (context-wide)
        import ctypes
        rt = ctypes.CDLL("libcudart.so.12")
        lim = ctypes.c_size_t(int(os.environ["L2_FETCH"]))
        rc = rt.cudaDeviceSetLimit(ctypes.c_int(0x05), lim)
        got = ctypes.c_size_t(0)
        rt.cudaDeviceGetLimit(ctypes.byref(got), ctypes.c_int(0x05))
        print(f"  cudaLimitMaxL2FetchGranularity <- {lim.value}: rc {rc}, now {got.value}", flush=True)
    a5 = csr5.csr_to_csr5(a, csr5.TuningParams(sigma=sigma))
    reps = 10 if a.nnz < 1e9 else 5
    evs = [(csr5.Event(), csr5.Event()) for _ in range(reps)]
    for _ in range(2):
        csr5.spmv_csr5(a5, x, y)
    for e0, e1 in evs:
        scrub.sum()
        csr5.spmv_csr5_evt(a5, x, y, e0, e1)
    torch.cuda.synchronize()
    ms = sorted(e0.elapsed_ms(e1) for e0, e1 in evs)
    if ref is None:
        ref = y.clone()
    ok = bool(((y - ref).abs() <= 1e-12 * ref.abs().clamp(min=1.0)).all())
    i = a5.info
    print(f"{name} [{cfg}] warps {i.warps_per_cta} stages {i.stages} smem {i.smem_bytes} "
          f"variant {i.kernel_variant} xmode {i.x_mode}: mean {sum(ms) / len(ms):.4f} "
          f"median {ms[len(ms) // 2]:.4f} ms  frac {i.spmv_bytes / (sum(ms) / len(ms)) / 1e6 / 6458.4:.3f}"
          f"  same_y {ok}", flush=True)
    a5.release()
