// synth.cu -- synthetic stencil matrices generated on the device (bench and
// test inputs for BASELINE configs 1 and 2).  Rows are grid points in
// lexicographic order, columns sorted ascending, so the CSR is canonical
// (csr.cpp:9-33).  Diagonal 4 / 26, off-diagonal -1.
#include <cub/cub.cuh>

#include "internal.cuh"

namespace csr5g {
namespace {

__device__ __forceinline__ int64_t nb(int64_t i, int64_t a) {
  return (a == 1) ? 1 : 3 - (i == 0) - (i == a - 1);
}

__global__ void k_count(int kind, int64_t a, int64_t m, int64_t* __restrict__ cnt) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  int64_t c;
  if (kind == 0) {
    const int64_t iy = r / a, ix = r - iy * a;
    c = 1 + (iy > 0) + (ix > 0) + (ix < a - 1) + (iy < a - 1);
  } else {
    const int64_t z = r / (a * a), rem = r - z * a * a, y = rem / a, x = rem - y * a;
    c = nb(x, a) * nb(y, a) * nb(z, a);
  }
  cnt[r] = c;
}

__global__ void k_fill(int kind, int64_t a, int64_t m, const int64_t* __restrict__ rp,
                       int32_t* __restrict__ col, double* __restrict__ val) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  int64_t q = rp[r];
  if (kind == 0) {
    const int64_t iy = r / a, ix = r - iy * a;
    const int64_t cand[5] = {r - a, r - 1, r, r + 1, r + a};
    const bool ok[5] = {iy > 0, ix > 0, true, ix < a - 1, iy < a - 1};
    for (int k = 0; k < 5; ++k)
      if (ok[k]) {
        col[q] = (int32_t)cand[k];
        val[q] = cand[k] == r ? 4.0 : -1.0;
        ++q;
      }
  } else {
    const int64_t z = r / (a * a), rem = r - z * a * a, y = rem / a, x = rem - y * a;
    for (int dz = -1; dz <= 1; ++dz) {
      if (z + dz < 0 || z + dz >= a) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        if (y + dy < 0 || y + dy >= a) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          if (x + dx < 0 || x + dx >= a) continue;
          const int64_t c = r + dz * a * a + dy * a + dx;
          col[q] = (int32_t)c;
          val[q] = (dz == 0 && dy == 0 && dx == 0) ? 26.0 : -1.0;
          ++q;
        }
      }
    }
  }
}

}  // namespace
}  // namespace csr5g

using namespace csr5g;

extern "C" {

int csr5g_stencil_size(int32_t kind, int64_t a, int64_t* m, int64_t* nnz) {
  if (a < 1 || (kind != 0 && kind != 1) || !m || !nnz)
    return fail(CSR5G_EINVAL, "csr5g: stencil kind must be 0 or 1 and a >= 1");
  if (kind == 0) {
    *m = a * a;
    *nnz = a == 1 ? 1 : 5 * a * a - 4 * a;
  } else {
    *m = a * a * a;
    const int64_t s = a == 1 ? 1 : 3 * a - 2;
    *nnz = s * s * s;
  }
  return CSR5G_OK;
}

int csr5g_stencil_fill(int32_t kind, int64_t a, int64_t* d_row_ptr, int32_t* d_col_idx,
                       double* d_val, void* stream_v) {
  int64_t m = 0, nnz = 0;
  int rc = csr5g_stencil_size(kind, a, &m, &nnz);
  if (rc) return rc;
  if (m >= (int64_t(1) << 31)) return fail(CSR5G_ERANGE, "csr5g: stencil too large");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  int64_t* cnt = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  CSR5G_CUDA(cudaMallocAsync(&cnt, sizeof(int64_t) * m, stream));
  k_count<<<(unsigned)((m + 255) / 256), 256, 0, stream>>>(kind, a, m, cnt);
  CSR5G_CUDA(cudaGetLastError());
  CSR5G_CUDA(cudaMemsetAsync(d_row_ptr, 0, sizeof(int64_t), stream));
  CSR5G_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, d_row_ptr + 1, (int)m, stream));
  CSR5G_CUDA(cudaMallocAsync(&tmp, tb, stream));
  CSR5G_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, cnt, d_row_ptr + 1, (int)m, stream));
  k_fill<<<(unsigned)((m + 255) / 256), 256, 0, stream>>>(kind, a, m, d_row_ptr, d_col_idx, d_val);
  CSR5G_CUDA(cudaGetLastError());
  CSR5G_CUDA(cudaFreeAsync(tmp, stream));
  CSR5G_CUDA(cudaFreeAsync(cnt, stream));
  return CSR5G_OK;
}

}  // extern "C"
