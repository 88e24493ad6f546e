import sys, os; sys.path.insert(0, '.')
import torch
from paper_1503_05032_b200 import csr5
from paper_1503_05032_b200.synthetic import WORKLOADS, make_matrix, bench_x
for name in sys.argv[1:]:
    a = make_matrix(WORKLOADS[name]); x = torch.as_tensor(bench_x(a.n)).cuda(); y = torch.empty(a.m, dtype=torch.float64, device='cuda')
    a5 = csr5.csr_to_csr5(a, csr5.TuningParams(sigma=csr5.select_sigma(a.nnz / a.m)))
    evs = [(csr5.Event(), csr5.Event()) for _ in range(10)]
    for _ in range(3): csr5.spmv_csr5(a5, x, y)
    for e0, e1 in evs: csr5.spmv_csr5_evt(a5, x, y, e0, e1)
    ms = sum(e0.elapsed_ms(e1) for e0, e1 in evs) / len(evs)
    print(name, os.environ.get("CSR5G_XMODE", "-"), a5.info.warps_per_cta, a5.info.stages, round(ms, 4), "ms frac", round(a5.info.spmv_bytes / ms / 1e6 / 6534.1, 3))
    a5.release()
