"""Experiment helper (GPU box): converter phase times (CSR5G_TRACE=1 adds a
sync per phase) and the untraced build wall time, per workload.
    python tools/conv_trace.py lap5_1000 st27_200"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1503_05032_b200 import csr5  # noqa: E402
from paper_1503_05032_b200.synthetic import WORKLOADS, make_matrix  # noqa: E402

for name in sys.argv[1:]:
    a = make_matrix(WORKLOADS[name])
    sigma = csr5.select_sigma(a.nnz / a.m)
    for _ in range(3):
        csr5.csr_to_csr5(a, csr5.TuningParams(sigma=sigma)).release()
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a5 = csr5.csr_to_csr5(a, csr5.TuningParams(sigma=sigma))
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        a5.release()
    ts.sort()
    print(f"{name} build ms: min {ts[0]:.3f} median {ts[len(ts) // 2]:.3f}", flush=True)
    for mode in ("1", "2"):
        os.environ["CSR5G_TRACE"] = mode
        for _ in range(3):
            csr5.csr_to_csr5(a, csr5.TuningParams(sigma=sigma)).release()
        del os.environ["CSR5G_TRACE"]
