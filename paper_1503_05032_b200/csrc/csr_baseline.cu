// csr_baseline.cu -- the plain-CSR kernels the reference benchmarks CSR5
// against (spmv.cpp:139-209), on the device, for the iteration scenario of
// run_benchmark (bench.cpp:86-90, 164-173: speedup_n50 / speedup_n500 need
// t_csr) and as the harness's dense-order check.
//
//  csr-scalar  one thread per row, `sum += val * x[col]` in row order -- the
//              reference's spmv_csr_scalar and, being sequential per row, the
//              summation order of dense_spmv_oracle (csr.cpp:85-98).
//  csr-segsum  products val * x[col] into a buffer, then the segmented sum
//              over the rows (spmv_csr_segsum: bit flags at row starts +
//              serial_segmented_sum); empty rows 0.  Each segment is summed
//              serially in order, as serial_segmented_sum does, one thread per
//              row over the product buffer.
// Both read the caller's device CSR (int64 row_ptr, int32 col_idx) as is.
#include <algorithm>

#include "internal.cuh"

namespace csr5g {
namespace {

__global__ void k_csr_scalar(int64_t m, const int64_t* __restrict__ rp,
                             const int32_t* __restrict__ col, const double* __restrict__ val,
                             const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t q = rp[r]; q < rp[r + 1]; ++q) s = fma(val[q], x[col[q]], s);
    y[r] = s;
  }
}

__global__ void k_products(int64_t nnz, const int32_t* __restrict__ col,
                           const double* __restrict__ val, const double* __restrict__ x,
                           double* __restrict__ prod) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz;
       q += (int64_t)gridDim.x * blockDim.x)
    prod[q] = val[q] * x[col[q]];
}

// serial sum of each row's segment of the product buffer
__global__ void k_segment_sums(int64_t m, const int64_t* __restrict__ rp,
                               const double* __restrict__ prod, double* __restrict__ y) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t q = rp[r]; q < rp[r + 1]; ++q) s += prod[q];
    y[r] = s;
  }
}

}  // namespace

int csr_spmv(int device, int kernel, int64_t m, int64_t n, int64_t nnz, const int64_t* rp,
             const int32_t* col, const double* val, const double* x, double* y,
             cudaStream_t stream) {
  CSR5G_CUDA(cudaSetDevice(device));
  if (m == 0) return CSR5G_OK;
  int sms = 0;
  CSR5G_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  if (kernel == CSR5G_CSR_SCALAR) {
    const int64_t blocks = std::min<int64_t>((m + 255) / 256, (int64_t)sms * 8);
    k_csr_scalar<<<(unsigned)blocks, 256, 0, stream>>>(m, rp, col, val, x, y);
    CSR5G_CUDA(cudaGetLastError());
    return CSR5G_OK;
  }
  // csr-segsum
  if (nnz == 0) {
    CSR5G_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * m, stream));
    return CSR5G_OK;
  }
  double* prod = nullptr;
  CSR5G_CUDA(cudaMallocAsync(&prod, sizeof(double) * nnz, stream));
  const int64_t blocks = std::min<int64_t>((nnz + 255) / 256, (int64_t)sms * 16);
  k_products<<<(unsigned)blocks, 256, 0, stream>>>(nnz, col, val, x, prod);
  CSR5G_CUDA(cudaGetLastError());
  const int64_t rblocks = std::min<int64_t>((m + 255) / 256, (int64_t)sms * 8);
  k_segment_sums<<<(unsigned)rblocks, 256, 0, stream>>>(m, rp, prod, y);
  CSR5G_CUDA(cudaGetLastError());
  CSR5G_CUDA(cudaFreeAsync(prod, stream));
  return CSR5G_OK;
}

}  // namespace csr5g
