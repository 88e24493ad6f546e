"""Experiment helper (GPU box): k_spmv time of one workload under the current
env knobs (CSR5G_*), CUDA events around the tile kernel, L2 scrubbed between
calls (as bench.py does).
    python tools/plan_probe.py st27_200 [rmat24 ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1503_05032_b200 import csr5  # noqa: E402
from paper_1503_05032_b200.synthetic import WORKLOADS, bench_x, make_matrix  # noqa: E402

for name in sys.argv[1:]:
    a = make_matrix(WORKLOADS[name])
    x = torch.as_tensor(bench_x(a.n)).cuda()
    y = torch.empty(a.m, dtype=torch.float64, device="cuda")
    a5 = csr5.csr_to_csr5(a, csr5.TuningParams(sigma=csr5.select_sigma(a.nnz / a.m)))
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    scrub = torch.empty(2 * l2 // 8, dtype=torch.float64, device="cuda")
    evs = [(csr5.Event(), csr5.Event()) for _ in range(10)]
    for _ in range(3):
        csr5.spmv_csr5(a5, x, y)
    for e0, e1 in evs:
        if scrub is not None:
            scrub.sum()  # read-only flush: evicts without leaving dirty lines
        csr5.spmv_csr5_evt(a5, x, y, e0, e1)
    ms = sum(e0.elapsed_ms(e1) for e0, e1 in evs) / len(evs)
    i = a5.info
    print(name, "warps", i.warps_per_cta, "stages", i.stages, "smem", i.smem_bytes,
          round(ms, 4), "ms frac", round(i.spmv_bytes / ms / 1e6 / 6534.1, 3))
    a5.release()
