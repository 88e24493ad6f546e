// csr5/gpu.hpp -- GPU-only additions to the csr5:: drop-in (not in the
// reference): SpMV on device-resident vectors (the fast path, no staging) and
// a batch of host vectors through the pipelined entry point.
#pragma once

#include <vector>

#include "csr5/spmv.hpp"

namespace csr5 {

/// y = A x with x, y device pointers on `stream` (a cudaStream_t, or nullptr
/// for the legacy default stream); stream-ordered, no synchronisation.
inline void spmv_csr5_device(const Csr5Matrix& a5, const double* d_x, double* d_y,
                             SpmvMode mode = SpmvMode::deterministic, void* stream = nullptr) {
  detail::check(csr5g_spmv(a5.handle(), d_x, d_y,
                           mode == SpmvMode::atomic ? CSR5G_MODE_ATOMIC : CSR5G_MODE_DETERMINISTIC,
                           stream));
}

/// y_k = A x_k for host vectors (csr5g_spmv_host_batch): x_{k+1} H2D and y_k
/// D2H overlap SpMV k on the two copy engines; returns when all are done.
inline void spmv_csr5_batch(const Csr5Matrix& a5, const std::vector<const double*>& xs,
                            const std::vector<double*>& ys,
                            SpmvMode mode = SpmvMode::deterministic) {
  if (xs.size() != ys.size())
    throw std::invalid_argument("spmv: " + std::to_string(xs.size()) + " x vectors but " +
                                std::to_string(ys.size()) + " y vectors");
  detail::check(csr5g_spmv_host_batch(
      a5.handle(), xs.data(), ys.data(), static_cast<std::int64_t>(xs.size()),
      mode == SpmvMode::atomic ? CSR5G_MODE_ATOMIC : CSR5G_MODE_DETERMINISTIC, nullptr));
  detail::check(csr5g_stream_synchronize(nullptr));
}

}  // namespace csr5
