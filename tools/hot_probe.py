"""Experiment helper (GPU box): the hot-column x staging (hotx.cu) under
several build-time knobs on one generated matrix.  Per configuration: build,
10 timed SpMVs (CUDA events around fill + tile kernel, L2 scrubbed between
calls as bench.py does), y compared bit for bit with the first configuration.
    python tools/hot_probe.py rmat24 'CSR5G_HOT=0' '' 'CSR5G_HOT_MB=32' ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1503_05032_b200 import csr5  # noqa: E402
from paper_1503_05032_b200.synthetic import WORKLOADS, bench_x, make_matrix  # noqa: E402

KNOBS = ("CSR5G_HOT", "CSR5G_HOT_MB", "CSR5G_HOT_ORDER", "CSR5G_HOT_L1", "CSR5G_HOT_COLS", "CSR5G_HOT_STRIDE", "CSR5G_HOT_COLD_POL",
         "CSR5G_XMODE", "CSR5G_NW", "CSR5G_BUDGET_KB", "CSR5G_GM", "CSR5G_STAGES")
name, configs = sys.argv[1], sys.argv[2:] or [""]
a = make_matrix(WORKLOADS[name])
x = torch.as_tensor(bench_x(a.n)).cuda()
y = torch.empty(a.m, dtype=torch.float64, device="cuda")
l2 = torch.cuda.get_device_properties(0).L2_cache_size
scrub = torch.empty(2 * l2 // 8, dtype=torch.float64, device="cuda")
sigma = csr5.select_sigma(a.nnz / a.m)
y_first = None
for cfg in configs:
    for k in KNOBS:
        os.environ.pop(k, None)
    for kv in cfg.split():
        k, v = kv.split("=")
        os.environ[k] = v
    a5 = csr5.csr_to_csr5(a, csr5.TuningParams(sigma=sigma))
    evs = [(csr5.Event(), csr5.Event()) for _ in range(10)]
    mode = os.environ.get("PROBE_MODE", "deterministic")
    for _ in range(3):
        csr5.spmv_csr5(a5, x, y, mode=mode)
    noscrub = os.environ.get("PROBE_NOSCRUB") == "1"
    for e0, e1 in evs:
        if not noscrub:
            scrub.sum()
        csr5.spmv_csr5_evt(a5, x, y, e0, e1, mode=mode)
    ts = sorted(e0.elapsed_ms(e1) for e0, e1 in evs)
    ms = sum(ts) / len(ts)
    same = "-"
    if y_first is None:
        y_first = y.clone()
    else:
        same = bool(torch.equal(y.view(torch.int64), y_first.view(torch.int64)))
    i = a5.info
    print(f"{name} [{cfg}] {ms:.4f} ms (min {ts[0]:.4f}) frac {i.spmv_bytes / ms / 1e6 / 6458.4:.3f} "
          f"hot {i.hot_cols} cov {i.hot_coverage:.3f} build {i.build_ms:.1f} ms warps {i.warps_per_cta} "
          f"xmode {i.x_mode} long {i.long_rows} y_same {same}", flush=True)
    a5.release()
