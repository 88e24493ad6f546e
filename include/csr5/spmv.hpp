// csr5/spmv.hpp -- drop-in for the reference's spmv.hpp (spmv.cpp:17-298).
// Every kernel runs on the GPU: spmv_csr5 through the CSR5 tile kernel
// (k_spmv, calibration inside), the CSR baselines through csr_baseline.cu,
// spmv_csr5_tile through the tile kernel's trace instantiation.  Host vectors
// are staged through the library's pipeline (csr5g_spmv_host); for
// device-resident x / y use csr5/gpu.hpp.
#pragma once

#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "csr5/csr.hpp"
#include "csr5/format.hpp"

namespace csr5 {

/// spmv.hpp:9-16.  deterministic: the shared rows' partials are combined in
/// a fixed order (bit-identical across runs); atomic: fp64 atomics.
enum class SpmvMode { deterministic, atomic };

/// One partial sum leaving a tile (spmv.hpp:18-25).
struct TileContribution {
  index_t row = 0;
  double value = 0.0;
  bool accumulate = false;
};

/// Per-worker scratch of the reference's CPU tile kernel (spmv.hpp:27-38).
/// Kept for source compatibility: the GPU kernel's scratch lives in
/// registers and shared memory, so nothing here is read.
struct SpmvWorkspace {
  std::vector<double> tmp;
  std::vector<double> last_tmp;
  std::vector<double> scan_scratch;
  std::vector<index_t> seg_offset;
  std::vector<index_t> blue_head;
  std::vector<std::uint8_t> has_head;

  void resize(index_t omega) {
    const auto w = static_cast<std::size_t>(omega);
    tmp.resize(w);
    last_tmp.resize(w);
    scan_scratch.resize(w);
    seg_offset.resize(w);
    blue_head.resize(w);
    has_head.resize(w);
  }
};

namespace detail {
inline void check_x(index_t n, std::size_t len) {  // spmv.cpp:17-21
  if (static_cast<index_t>(len) != n)
    throw std::invalid_argument("spmv: x has length " + std::to_string(len) + ", expected " +
                                std::to_string(n));
}
inline void check_y(index_t m, std::size_t len) {  // spmv.cpp:23-27
  if (static_cast<index_t>(len) != m)
    throw std::invalid_argument("spmv: y has length " + std::to_string(len) + ", expected " +
                                std::to_string(m));
}
inline void csr_kernel(int kernel, const CsrMatrix& a, const DenseVector& x, std::span<double> y) {
  check_x(a.n, x.size());
  check_y(a.m, y.size());
  check(csr5g_csr_spmv_host(-1, kernel, a.m, a.n, a.nnz(), a.row_ptr.data(), a.col_idx.data(),
                            a.val.data(), x.data(), y.data()));
}
}  // namespace detail

/// Row-parallel CSR kernel (spmv.cpp:139-154): one GPU thread per row.
inline void spmv_csr_scalar(const CsrMatrix& a, const DenseVector& x, std::span<double> y) {
  detail::csr_kernel(CSR5G_CSR_SCALAR, a, x, y);
}
inline DenseVector spmv_csr_scalar(const CsrMatrix& a, const DenseVector& x) {
  DenseVector y(static_cast<std::size_t>(a.m));
  spmv_csr_scalar(a, x, y);
  return y;
}

/// CSR via products + segmented sum (spmv.cpp:156-209), on the GPU.
inline void spmv_csr_segsum(const CsrMatrix& a, const DenseVector& x, std::span<double> y) {
  detail::csr_kernel(CSR5G_CSR_SEGSUM, a, x, y);
}
inline DenseVector spmv_csr_segsum(const CsrMatrix& a, const DenseVector& x) {
  DenseVector y(static_cast<std::size_t>(a.m));
  spmv_csr_segsum(a, x, y);
  return y;
}

/// Contributions of one complete tile in the reference's emission order
/// (spmv.cpp:211-222): the sealed segments column by column, top to bottom,
/// then the bottom piece of every head-bearing column after the fast
/// segmented sum.  Computed by the GPU tile kernel itself (its trace
/// instantiation, csr5g_spmv_tile), so the per-tile values are the ones the
/// SpMV combines.
inline std::vector<TileContribution> spmv_csr5_tile(const Csr5Matrix& a5, index_t tid,
                                                    const DenseVector& x, SpmvWorkspace& ws) {
  (void)ws;
  if (tid < 0 || tid >= a5.p_complete)
    throw std::invalid_argument("spmv_csr5_tile: tile " + std::to_string(tid) +
                                " is not a complete tile");
  detail::check_x(a5.n, x.size());
  const std::size_t cap = static_cast<std::size_t>(a5.omega() * a5.sigma()) + 1;
  std::vector<std::int64_t> rows(cap);
  std::vector<double> vals(cap);
  std::vector<std::uint8_t> acc(cap);
  std::int64_t count = 0;
  detail::check(csr5g_spmv_tile(a5.handle(), tid, x.data(), rows.data(), vals.data(), acc.data(),
                                static_cast<std::int64_t>(cap), &count));
  std::vector<TileContribution> out(static_cast<std::size_t>(count));
  for (std::size_t k = 0; k < out.size(); ++k) out[k] = {rows[k], vals[k], acc[k] != 0};
  return out;
}

/// spmv.cpp:224-298: y fully overwritten; host x / y staged to the device.
inline void spmv_csr5(const Csr5Matrix& a5, const DenseVector& x, std::span<double> y,
                      SpmvMode mode = SpmvMode::deterministic) {
  detail::check_x(a5.n, x.size());
  detail::check_y(a5.m, y.size());
  if (a5.m == 0) return;
  detail::check(csr5g_spmv_host(a5.handle(), x.data(), y.data(),
                                mode == SpmvMode::atomic ? CSR5G_MODE_ATOMIC
                                                         : CSR5G_MODE_DETERMINISTIC));
}
inline DenseVector spmv_csr5(const Csr5Matrix& a5, const DenseVector& x,
                             SpmvMode mode = SpmvMode::deterministic) {
  DenseVector y(static_cast<std::size_t>(a5.m));
  spmv_csr5(a5, x, std::span<double>(y), mode);
  return y;
}

}  // namespace csr5
