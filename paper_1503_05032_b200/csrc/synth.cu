// synth.cu -- synthetic stencil matrices generated on the device (bench and
// test inputs for BASELINE configs 1 and 2).  Rows are grid points in
// lexicographic order, columns sorted ascending, so the CSR is canonical
// (csr.cpp:9-33).  Diagonal 4 / 26, off-diagonal -1.
#include <cub/cub.cuh>

#include <random>

#include "internal.cuh"

namespace csr5g {
namespace {

// neighbours of coordinate i along an axis of extent e (itself included)
__device__ __forceinline__ int64_t nb(int64_t i, int64_t e) {
  return (e == 1) ? 1 : 3 - (i == 0) - (i == e - 1);
}

// Grid: a columns per line (x), a lines per plane (y, 3D only) and `layers`
// along the outermost axis (y in 2D, z in 3D); layers = a is the cube/square.
__global__ void k_count(int kind, int64_t a, int64_t layers, int64_t m, int64_t* __restrict__ cnt) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  int64_t c;
  if (kind == 0) {
    const int64_t iy = r / a, ix = r - iy * a;
    c = 1 + (iy > 0) + (ix > 0) + (ix < a - 1) + (iy < layers - 1);
  } else {
    const int64_t z = r / (a * a), rem = r - z * a * a, y = rem / a, x = rem - y * a;
    c = nb(x, a) * nb(y, a) * nb(z, layers);
  }
  cnt[r] = c;
}

// Writes the entries of row r whose global positions fall in [lo, hi) to
// col/val at position - lo (lo = 0, hi = nnz: the whole matrix).
__global__ void k_fill(int kind, int64_t a, int64_t layers, int64_t m,
                       const int64_t* __restrict__ rp, int64_t lo, int64_t hi,
                       int32_t* __restrict__ col, double* __restrict__ val) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  int64_t q = rp[r];
  if (rp[r + 1] <= lo || q >= hi) return;
  auto put = [&](int64_t c, double v) {
    if (q >= lo && q < hi) {
      col[q - lo] = (int32_t)c;
      val[q - lo] = v;
    }
    ++q;
  };
  if (kind == 0) {
    const int64_t iy = r / a, ix = r - iy * a;
    if (iy > 0) put(r - a, -1.0);
    if (ix > 0) put(r - 1, -1.0);
    put(r, 4.0);
    if (ix < a - 1) put(r + 1, -1.0);
    if (iy < layers - 1) put(r + a, -1.0);
  } else {
    const int64_t z = r / (a * a), rem = r - z * a * a, y = rem / a, x = rem - y * a;
    for (int dz = -1; dz <= 1; ++dz) {
      if (z + dz < 0 || z + dz >= layers) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        if (y + dy < 0 || y + dy >= a) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          if (x + dx < 0 || x + dx >= a) continue;
          put(r + dz * a * a + dy * a + dx, (dz == 0 && dy == 0 && dx == 0) ? 26.0 : -1.0);
        }
      }
    }
  }
}

}  // namespace
}  // namespace csr5g

using namespace csr5g;

extern "C" {

int csr5g_stencil_box_size(int32_t kind, int64_t a, int64_t layers, int64_t* m, int64_t* nnz) {
  if (a < 1 || layers < 1 || (kind != 0 && kind != 1) || !m || !nnz)
    return fail(CSR5G_EINVAL, "csr5g: stencil kind must be 0 or 1 and a, layers >= 1");
  // per-axis neighbour sums: an axis of extent e contributes 3e - 2 (e > 1)
  auto ax = [](int64_t e) { return e == 1 ? int64_t(1) : 3 * e - 2; };
  if (kind == 0) {
    *m = a * layers;
    *nnz = a * layers + 2 * (a - 1) * layers + 2 * (layers - 1) * a;
  } else {
    *m = a * a * layers;
    *nnz = ax(a) * ax(a) * ax(layers);
  }
  return CSR5G_OK;
}

int csr5g_stencil_size(int32_t kind, int64_t a, int64_t* m, int64_t* nnz) {
  return csr5g_stencil_box_size(kind, a, a, m, nnz);
}

int csr5g_stencil_box_fill(int32_t kind, int64_t a, int64_t layers, int64_t pos_begin,
                           int64_t pos_end, int64_t* d_row_ptr, int32_t* d_col_idx,
                           double* d_val, void* stream_v) {
  int64_t m = 0, nnz = 0;
  int rc = csr5g_stencil_box_size(kind, a, layers, &m, &nnz);
  if (rc) return rc;
  if (m >= (int64_t(1) << 31)) return fail(CSR5G_ERANGE, "csr5g: stencil too large");
  if (pos_begin < 0 || pos_end < pos_begin || pos_end > nnz)
    return fail(CSR5G_EINVAL, "csr5g: stencil slice out of range");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  int64_t* cnt = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  CSR5G_CUDA(cudaMallocAsync(&cnt, sizeof(int64_t) * m, stream));
  k_count<<<(unsigned)((m + 255) / 256), 256, 0, stream>>>(kind, a, layers, m, cnt);
  CSR5G_CUDA(cudaGetLastError());
  CSR5G_CUDA(cudaMemsetAsync(d_row_ptr, 0, sizeof(int64_t), stream));
  CSR5G_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, d_row_ptr + 1, (int)m, stream));
  CSR5G_CUDA(cudaMallocAsync(&tmp, tb, stream));
  CSR5G_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, cnt, d_row_ptr + 1, (int)m, stream));
  if (pos_end > pos_begin) {
    k_fill<<<(unsigned)((m + 255) / 256), 256, 0, stream>>>(kind, a, layers, m, d_row_ptr,
                                                           pos_begin, pos_end, d_col_idx, d_val);
    CSR5G_CUDA(cudaGetLastError());
  }
  CSR5G_CUDA(cudaFreeAsync(tmp, stream));
  CSR5G_CUDA(cudaFreeAsync(cnt, stream));
  return CSR5G_OK;
}

int csr5g_stencil_fill(int32_t kind, int64_t a, int64_t* d_row_ptr, int32_t* d_col_idx,
                       double* d_val, void* stream_v) {
  int64_t m = 0, nnz = 0;
  int rc = csr5g_stencil_box_size(kind, a, a, &m, &nnz);
  if (rc) return rc;
  return csr5g_stencil_box_fill(kind, a, a, 0, nnz, d_row_ptr, d_col_idx, d_val, stream_v);
}

// The benchmark's x (bench.cpp:103-105): std::mt19937_64(seed), x_i = 0.5 +
// (rng() >> 11) * 2^-53, on the host (the engine is sequential; 134M values
// for R-MAT s27 take ~1 s here against ~30 s vectorised in numpy).
int csr5g_bench_x(int64_t n, uint64_t seed, double* h_x) {
  if (n < 0 || (n > 0 && !h_x)) return fail(CSR5G_EINVAL, "csr5g: bad bench_x arguments");
  std::mt19937_64 rng(seed);
  for (int64_t i = 0; i < n; ++i) h_x[i] = 0.5 + (double)(rng() >> 11) * 0x1.0p-53;
  return CSR5G_OK;
}

}  // extern "C"
