"""Experiment helper (GPU box): the same x gathers of one workload issued by
different kernels, for ncu to compare DRAM bytes, L2 hit rate and time:
  1. the CSR5 SpMV (k_spmv),
  2. torch.index_select over col_idx in CSR (row-major) order,
  3. torch.index_select over col_idx in the CSR5 (tile-transposed) order,
  4. cuSPARSE csrmv (torch sparse CSR).
L2 scrubbed before each (a 2x L2 read).  Prints CUDA-event times; run under
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,\
lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,dram__sectors_read.sum \
      -k regex:"k_spmv|index|csrmv|Csr|spmv" python tools/gather_compare.py rmat27
for the counters."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1503_05032_b200 import csr5  # noqa: E402
from paper_1503_05032_b200.synthetic import WORKLOADS, bench_x, make_matrix  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "rmat24"
a = make_matrix(WORKLOADS[name])
x = torch.as_tensor(bench_x(a.n)).cuda()
y = torch.empty(a.m, dtype=torch.float64, device="cuda")
sigma = csr5.select_sigma(a.nnz / a.m)
a5 = csr5.csr_to_csr5(a, csr5.TuningParams(sigma=sigma))
l2 = torch.cuda.get_device_properties(0).L2_cache_size
scrub = torch.empty(2 * l2 // 8, dtype=torch.float64, device="cuda")
idx = a.col_idx.long()
B = 32 * sigma
pc = a.nnz // B
idx_t = torch.cat([idx[:pc * B].view(pc, 32, sigma).transpose(1, 2).reshape(-1), idx[pc * B:]])
out = torch.empty(a.nnz, dtype=torch.float64, device="cuda")


def timed(label, fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        scrub.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name} {label}: {min(ts):.3f} ms (best of {reps})", flush=True)


timed("csr5 spmv", lambda: csr5.spmv_csr5(a5, x, y))
timed("index_select csr order", lambda: torch.index_select(x, 0, idx, out=out))
timed("index_select csr5 order", lambda: torch.index_select(x, 0, idx_t, out=out))
del idx_t
A = torch.sparse_csr_tensor(a.row_ptr, idx, a.val, (a.m, a.n))
xc = x.unsqueeze(1)
timed("cusparse csrmv", lambda: A @ xc)
