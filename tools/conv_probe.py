import sys, os, time
sys.path.insert(0, '/root/repo')
import torch
from paper_1503_05032_b200 import csr5
from paper_1503_05032_b200.synthetic import WORKLOADS, make_matrix
for name in sys.argv[1:]:
    a = make_matrix(WORKLOADS[name])
    sig = csr5.select_sigma(a.nnz / a.m)
    for i in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        a5 = csr5.csr_to_csr5(a, csr5.TuningParams(sigma=sig))
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(name, i, round((t1 - t0) * 1e3, 3), 'ms alloc', round(a5.info.alloc_ms, 3), flush=True)
        a5.release()
