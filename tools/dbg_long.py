import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle.oracle import Oracle
from paper_1503_05032_b200 import csr5
orc = Oracle()
rng = np.random.default_rng(5)
bad = 0
for trial in range(300):
    m = int(rng.integers(1, 150)); n = int(rng.integers(1, 150)); nnz = int(rng.integers(0, 4000))
    sigma = int(rng.choice([1, 2, 4, 12, 16, 27, 48]))
    rows = rng.integers(0, m, nnz); cols = rng.integers(0, n, nnz)
    a = orc.coo_to_csr(rows.tolist(), cols.tolist(), rng.uniform(0.5, 1.5, nnz).tolist(), m, n)
    x = orc.rng(trial).random_x(n)
    d = csr5.CsrMatrix.from_host(a.m, a.n, a.row_ptr, a.col_idx.astype(np.int32), a.val)
    a5 = csr5.csr_to_csr5(d, csr5.TuningParams(sigma=sigma))
    yr = orc.spmv(a, x, 32, sigma)
    for mode in ("deterministic", "atomic"):
      y = csr5.spmv_csr5(a5, torch.as_tensor(x).cuda(), mode=mode).cpu().numpy()
      err = np.abs(y - yr) / np.maximum(1, np.abs(yr))
      if err.max() > 1e-12:
        bad += 1
        B = 32 * sigma; pc = a.nnz // B
        rp = a.row_ptr
        w = np.flatnonzero(err > 1e-12)
        info = a5.info
        print(f"{mode} trial {trial} m={m} n={n} nnz={a.nnz} sigma={sigma} pc={pc} tail={a.nnz % B} long_rows={info.long_rows} warps={info.spmv_warps} variant={info.kernel_variant}")
        for r in w[:6]:
            f, l = min(rp[r] // B, pc), min((rp[r + 1] - 1) // B, pc)
            print(f"   row {r}: y={y[r]:.6f} ref={yr[r]:.6f} len={rp[r+1]-rp[r]} parts {f}..{l} ({l - f + 1})")
    a5.release()
    if bad > 8: break
print("bad", bad)
