// csr5g.hpp -- C++ drop-in for the reference's csr5:: hot-path API, over the
// C ABI of libcsr5g.so (include/csr5g.h).  Header-only; link -lcsr5g.
//
// reference (proj/core/include/csr5)        here (namespace csr5g)
// -----------------------------------------  ----------------------------------
// TuningParams            tuning.hpp:13-24    TuningParams (omega = 32, sigma 0 = auto)
// CsrMatrix               csr.hpp:25-35       CsrMatrix (same fields, int64 indices)
// DenseVector             csr.hpp:19          DenseVector
// SpmvMode                spmv.hpp:16         SpmvMode
// Csr5Matrix              format.hpp:130-176  Csr5Matrix (move-only RAII device handle)
// csr_to_csr5             format.hpp:182      csr_to_csr5
// spmv_csr5 (x2)          spmv.hpp:58-61      spmv_csr5 (x2; + a device-pointer overload)
// csr5_to_csr             format.hpp:186      csr5_to_csr
// dump_format             format.hpp:190      dump_format
// select_sigma            tuning.hpp:29       select_sigma
// CooEntry, coo_to_csr    csr.hpp             CooEntry, coo_to_csr (sorted + summed on the GPU)
// read_matrix_market,     matrix_market.hpp   read_matrix_market, load_matrix_market
//   load_matrix_market
// (host-vector batch)                         spmv_csr5_batch (pipelined H2D/SpMV/D2H)
//
// Errors are rethrown as the reference's exception types with the library's
// message: CSR5G_EINVAL -> std::invalid_argument, CSR5G_ERANGE ->
// std::out_of_range, everything else -> std::runtime_error.  The reference's
// argument-check messages ("spmv: x has length N, expected M", the tuning and
// layout messages) are reproduced verbatim.
#pragma once

#include <cstdint>
#include <ostream>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "csr5g.h"

namespace csr5g {

using index_t = std::int64_t;
using DenseVector = std::vector<double>;

enum class SpmvMode { deterministic = CSR5G_MODE_DETERMINISTIC, atomic = CSR5G_MODE_ATOMIC };

struct TuningParams {
  index_t omega = 32;  // one warp lane per tile column (GPU)
  index_t sigma = 0;   // 0: select_sigma(nnz/m, <r,s,t,u>) like `spmv-bench --sigma auto`
  index_t r = 4;
  index_t s = 32;
  index_t t = 256;
  index_t u = 4;
};

struct CsrMatrix {
  index_t m = 0;
  index_t n = 0;
  std::vector<index_t> row_ptr;
  std::vector<index_t> col_idx;
  std::vector<double> val;
  index_t nnz() const { return row_ptr.empty() ? 0 : row_ptr.back(); }
  bool operator==(const CsrMatrix&) const = default;
};

inline void check(int rc) {
  if (rc == CSR5G_OK) return;
  const std::string msg = csr5g_last_error();
  if (rc == CSR5G_EINVAL) throw std::invalid_argument(msg);
  if (rc == CSR5G_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

inline index_t select_sigma(double nnz_per_row, const TuningParams& b = {}) {
  index_t out = 0;
  check(csr5g_select_sigma(nnz_per_row, b.r, b.s, b.t, b.u, &out));
  return out;
}

class Csr5Matrix {
 public:
  Csr5Matrix() = default;
  explicit Csr5Matrix(csr5g_matrix h) : h_(h) { check(csr5g_info_get(h_, &info_)); }
  Csr5Matrix(const Csr5Matrix&) = delete;
  Csr5Matrix& operator=(const Csr5Matrix&) = delete;
  Csr5Matrix(Csr5Matrix&& o) noexcept : h_(std::exchange(o.h_, nullptr)), info_(o.info_) {}
  Csr5Matrix& operator=(Csr5Matrix&& o) noexcept {
    if (this != &o) {
      reset();
      h_ = std::exchange(o.h_, nullptr);
      info_ = o.info_;
    }
    return *this;
  }
  ~Csr5Matrix() { reset(); }

  void reset() {
    if (h_) csr5g_release(h_);
    h_ = nullptr;
  }
  csr5g_matrix handle() const { return h_; }
  const csr5g_info& info() const { return info_; }

  // reference field names (format.hpp:130-176)
  index_t m() const { return info_.m; }
  index_t n() const { return info_.n; }
  index_t nnz() const { return info_.nnz; }
  index_t omega() const { return info_.omega; }
  index_t sigma() const { return info_.sigma; }
  index_t p() const { return info_.p; }
  index_t p_complete() const { return info_.p_complete; }
  index_t tail_len() const { return info_.tail_len; }
  std::size_t metadata_bytes() const { return (std::size_t)info_.metadata_bytes; }

  // Every array widened to the reference's 64-bit types.
  struct Arrays {
    std::vector<std::uint64_t> tile_ptr, tile_desc;
    std::vector<index_t> empty_offset_ptr, empty_offset, col_idx;
    std::vector<double> val;
  };
  Arrays export_arrays() const {
    Arrays a;
    const index_t pcs = info_.tile_end - info_.tile_begin;
    a.tile_ptr.resize((std::size_t)info_.tile_ptr_len);
    a.tile_desc.resize((std::size_t)(pcs * info_.omega));
    a.empty_offset_ptr.resize((std::size_t)(pcs + 1));
    a.empty_offset.resize((std::size_t)info_.empty_offset_len);
    a.col_idx.resize((std::size_t)info_.nnz_held);
    a.val.resize((std::size_t)info_.nnz_held);
    check(csr5g_export(h_, a.tile_ptr.data(), a.tile_desc.data(), a.empty_offset_ptr.data(),
                       a.empty_offset.data(), a.col_idx.data(), a.val.data()));
    return a;
  }

 private:
  csr5g_matrix h_ = nullptr;
  csr5g_info info_{};
};

// format.cpp:165-252 -- the host CSR is staged to `device`, converted there.
inline Csr5Matrix csr_to_csr5(const CsrMatrix& a, const TuningParams& params = {},
                              int device = 0) {
  if (static_cast<index_t>(a.row_ptr.size()) != a.m + 1)
    throw std::runtime_error("csr: row_ptr has size " + std::to_string(a.row_ptr.size()) +
                             ", expected " + std::to_string(a.m + 1));
  if (static_cast<index_t>(a.col_idx.size()) != a.nnz() ||
      static_cast<index_t>(a.val.size()) != a.nnz())
    throw std::runtime_error("csr: col_idx/val size does not match row_ptr[m]");
  const csr5g_params p{params.omega, params.sigma, params.r, params.s, params.t, params.u};
  csr5g_matrix h = nullptr;
  check(csr5g_build_host(device, a.m, a.n, a.nnz(), a.row_ptr.data(), a.col_idx.data(),
                         a.val.data(), &p, &h));
  return Csr5Matrix(h);
}

// spmv.cpp:224-298 with the reference's argument checks (spmv.cpp:17-27).
inline void spmv_csr5(const Csr5Matrix& a5, const DenseVector& x, std::span<double> y,
                      SpmvMode mode = SpmvMode::deterministic) {
  if (static_cast<index_t>(x.size()) != a5.n())
    throw std::invalid_argument("spmv: x has length " + std::to_string(x.size()) +
                                ", expected " + std::to_string(a5.n()));
  if (static_cast<index_t>(y.size()) != a5.m())
    throw std::invalid_argument("spmv: y has length " + std::to_string(y.size()) +
                                ", expected " + std::to_string(a5.m()));
  check(csr5g_spmv_host(a5.handle(), x.data(), y.data(), static_cast<int32_t>(mode)));
}

inline DenseVector spmv_csr5(const Csr5Matrix& a5, const DenseVector& x,
                             SpmvMode mode = SpmvMode::deterministic) {
  DenseVector y(static_cast<std::size_t>(a5.m()));
  spmv_csr5(a5, x, std::span<double>(y), mode);
  return y;
}

// Device-resident overload (the fast path): x, y are device pointers,
// stream a cudaStream_t; stream-ordered, no synchronisation.
inline void spmv_csr5(const Csr5Matrix& a5, const double* d_x, double* d_y, SpmvMode mode,
                      void* stream) {
  check(csr5g_spmv(a5.handle(), d_x, d_y, static_cast<int32_t>(mode), stream));
}

// format.cpp:254-265: undo the tile transposition; row_ptr is unchanged by the
// format, so the caller passes the one it built from.
inline CsrMatrix csr5_to_csr(const Csr5Matrix& a5, std::vector<index_t> row_ptr) {
  CsrMatrix a;
  a.m = a5.m();
  a.n = a5.n();
  a.row_ptr = std::move(row_ptr);
  a.col_idx.resize((std::size_t)a5.info().nnz_held);
  a.val.resize((std::size_t)a5.info().nnz_held);
  check(csr5g_to_csr_host(a5.handle(), a.col_idx.data(), a.val.data()));
  return a;
}

// format.cpp:267-305 text dump (same layout), read back from the device.
inline void dump_format(const Csr5Matrix& a5, std::ostream& out) {
  const csr5g_info& i = a5.info();
  const auto ar = a5.export_arrays();
  const index_t om = i.omega, sg = i.sigma;
  const int yb = i.y_offset_bits, sb = i.seg_offset_bits;
  out << "csr5 m=" << i.m << " n=" << i.n << " nnz=" << i.nnz << " omega=" << om
      << " sigma=" << sg << " tiles=" << i.p << " complete=" << i.p_complete
      << " tail=" << i.tail_len << " tile_ptr_bits=" << i.tile_ptr_bits
      << " desc_word_bits=" << i.word_bits << " metadata_bytes=" << i.metadata_bytes
      << " empty_offset_entries=" << i.empty_offset_len << '\n';
  for (index_t k = 0; k + 1 < i.tile_ptr_len; ++k) {
    const index_t tid = i.tile_begin + k;
    const std::uint64_t raw = ar.tile_ptr[(std::size_t)k];
    const bool empty = (raw >> 31) & 1u;
    out << "tile " << tid << ": row=" << (raw & 0x7fffffffu) << " empty=" << (empty ? 1 : 0);
    if (tid >= i.p_complete) {
      out << " tail nnz=" << i.tail_len << '\n';
      continue;
    }
    const std::uint64_t ym = (std::uint64_t{1} << yb) - 1, smask = (std::uint64_t{1} << sb) - 1;
    out << " y_offset=[";
    for (index_t c = 0; c < om; ++c)
      out << (c ? "," : "") << ((ar.tile_desc[(std::size_t)(k * om + c)] >> (sb + sg)) & ym);
    out << "] seg_offset=[";
    for (index_t c = 0; c < om; ++c)
      out << (c ? "," : "") << ((ar.tile_desc[(std::size_t)(k * om + c)] >> sg) & smask);
    out << "] bit_flag=[";
    for (index_t c = 0; c < om; ++c) {
      if (c) out << ",";
      for (index_t j = 0; j < sg; ++j)
        out << (((ar.tile_desc[(std::size_t)(k * om + c)] >> (sg - 1 - j)) & 1u) ? '1' : '0');
    }
    out << "]";
    if (empty) {
      out << " empty_offset=[";
      for (index_t e = ar.empty_offset_ptr[(std::size_t)k]; e < ar.empty_offset_ptr[(std::size_t)k + 1];
           ++e)
        out << (e != ar.empty_offset_ptr[(std::size_t)k] ? "," : "") << ar.empty_offset[(std::size_t)e];
      out << "]";
    }
    out << '\n';
  }
}

// y_k = A x_k for a batch of host vectors (csr5g_spmv_host_batch): x_{k+1}
// H2D and y_k D2H overlap SpMV k; synchronises before returning.  Pinned
// (cudaHostAlloc'd) vectors overlap fully; pageable ones still work.
inline void spmv_csr5_batch(const Csr5Matrix& a5, const std::vector<const double*>& xs,
                            const std::vector<double*>& ys,
                            SpmvMode mode = SpmvMode::deterministic) {
  if (xs.size() != ys.size())
    throw std::invalid_argument("spmv: " + std::to_string(xs.size()) + " x vectors but " +
                                std::to_string(ys.size()) + " y vectors");
  check(csr5g_spmv_host_batch(a5.handle(), xs.data(), ys.data(), (int64_t)xs.size(),
                              static_cast<int32_t>(mode), nullptr));
  check(csr5g_stream_synchronize(nullptr));
}

struct CooEntry {
  index_t row;
  index_t col;
  double value;
};

struct MatrixMarketData {
  std::vector<CooEntry> entries;
  index_t m = 0;
  index_t n = 0;
};

// csr.cpp:35-72: sorted by (row, col), duplicates summed in input order (on
// `device`); out-of-range entries throw std::invalid_argument.
inline CsrMatrix coo_to_csr(const std::vector<CooEntry>& entries, index_t m, index_t n,
                            int device = 0) {
  std::vector<index_t> r(entries.size()), c(entries.size());
  std::vector<double> v(entries.size());
  for (std::size_t k = 0; k < entries.size(); ++k) {
    r[k] = entries[k].row;
    c[k] = entries[k].col;
    v[k] = entries[k].value;
  }
  CsrMatrix a;
  a.m = m;
  a.n = n;
  a.row_ptr.resize(static_cast<std::size_t>(m < 0 ? 0 : m) + 1);
  a.col_idx.resize(entries.size());
  a.val.resize(entries.size());
  index_t nnz = 0;
  check(csr5g_coo_to_csr_host(device, m, n, (int64_t)entries.size(), r.data(), c.data(),
                              v.data(), a.row_ptr.data(), a.col_idx.data(), a.val.data(), &nnz));
  a.col_idx.resize((std::size_t)nnz);
  a.val.resize((std::size_t)nnz);
  return a;
}

// matrix_market.cpp:38-96; parse errors throw std::runtime_error with the
// reference's text.
inline MatrixMarketData read_matrix_market(const std::string& path) {
  csr5g_coo h = nullptr;
  int64_t m = 0, n = 0, k = 0;
  check(csr5g_mm_read(path.c_str(), &h, &m, &n, &k));
  std::vector<index_t> r((std::size_t)k), c((std::size_t)k);
  std::vector<double> v((std::size_t)k);
  const int rc = csr5g_coo_get(h, r.data(), c.data(), v.data());
  csr5g_coo_release(h);
  check(rc);
  MatrixMarketData d;
  d.m = m;
  d.n = n;
  d.entries.resize((std::size_t)k);
  for (std::size_t q = 0; q < (std::size_t)k; ++q) d.entries[q] = {r[q], c[q], v[q]};
  return d;
}

inline CsrMatrix load_matrix_market(const std::string& path, int device = 0) {
  const MatrixMarketData d = read_matrix_market(path);
  return coo_to_csr(d.entries, d.m, d.n, device);
}

}  // namespace csr5g
