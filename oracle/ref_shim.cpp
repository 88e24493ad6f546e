// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles the reference sources
// where they lie (/root/reference/proj/core/src/*.cpp) together with this
// file into oracle/_ref/libcsr5ref.so.  Tests use it to pin the C oracle
// (csr5_oracle.c) and to regenerate golden fixtures; bench.py --impl
// reference uses it as the reference's own CPU implementation.  The
// product never loads it.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <new>
#include <sstream>
#include <span>
#include <string>
#include <vector>

#include "csr5/bench.hpp"
#include "csr5/csr.hpp"
#include "csr5/format.hpp"
#include "csr5/matrix_market.hpp"
#include "csr5/spmv.hpp"
#include "csr5/synthetic.hpp"
#include "csr5/tuning.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 3;
  return 2;
}

struct RefHandle {
  csr5::Csr5Matrix a5;
  csr5::CsrMatrix a;  // kept for csr-scalar timing
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void ref_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

// csr_to_csr5 (format.hpp:182).  Copies the caller's CSR into reference
// types first (not timed by callers that use ref_build_timed).
int ref_build(int64_t m, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
              const double* val, int64_t omega, int64_t sigma, int64_t r, int64_t s, int64_t t,
              int64_t u, int parallel, void** out, double* conv_ms) {
  try {
    auto* h = new RefHandle();
    h->a.m = m;
    h->a.n = n;
    h->a.row_ptr.assign(row_ptr, row_ptr + m + 1);
    const int64_t nnz = row_ptr[m];
    h->a.col_idx.assign(col_idx, col_idx + nnz);
    h->a.val.assign(val, val + nnz);
    csr5::TuningParams p{.omega = omega, .sigma = sigma, .r = r, .s = s, .t = t, .u = u};
    const auto t0 = std::chrono::steady_clock::now();
    try {
      h->a5 = csr5::csr_to_csr5(h->a, p, parallel != 0);
    } catch (...) {
      delete h;
      throw;
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (conv_ms) *conv_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    *out = h;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_free(void* hv) { delete static_cast<RefHandle*>(hv); }

// Sizes: p, pc, tail, tile_ptr_bits, word_bits, eo count, y_bits, seg_bits.
void ref_info(void* hv, int64_t* out8) {
  const auto& a5 = static_cast<RefHandle*>(hv)->a5;
  out8[0] = a5.p;
  out8[1] = a5.p_complete;
  out8[2] = a5.tail_len;
  out8[3] = a5.tile_ptr_bits;
  out8[4] = a5.layout.word_bits;
  out8[5] = static_cast<int64_t>(a5.empty_offset.size());
  out8[6] = a5.layout.y_offset_bits;
  out8[7] = a5.layout.seg_offset_bits;
}

int64_t ref_metadata_bytes(void* hv) {
  return static_cast<int64_t>(static_cast<RefHandle*>(hv)->a5.metadata_bytes());
}

void ref_export(void* hv, uint64_t* tile_ptr, uint64_t* tile_desc, int64_t* eo_ptr, int64_t* eo,
                int64_t* col_idx, double* val) {
  const auto& a5 = static_cast<RefHandle*>(hv)->a5;
  for (std::size_t i = 0; i < a5.tile_ptr.size(); ++i) tile_ptr[i] = a5.tile_ptr[i];
  for (std::size_t i = 0; i < a5.tile_desc.size(); ++i) tile_desc[i] = a5.tile_desc[i];
  std::memcpy(eo_ptr, a5.empty_offset_ptr.data(), a5.empty_offset_ptr.size() * sizeof(int64_t));
  std::memcpy(eo, a5.empty_offset.data(), a5.empty_offset.size() * sizeof(int64_t));
  std::memcpy(col_idx, a5.col_idx.data(), a5.col_idx.size() * sizeof(int64_t));
  std::memcpy(val, a5.val.data(), a5.val.size() * sizeof(double));
}

// dump_format (format.hpp:190): the reference's text dump into buf (at most
// cap bytes); returns the full length.
int64_t ref_dump_format(void* hv, char* buf, int64_t cap) {
  std::ostringstream out;
  csr5::dump_format(static_cast<RefHandle*>(hv)->a5, out);
  const std::string t = out.str();
  if (buf && cap > 0) std::memcpy(buf, t.data(), std::min<size_t>(t.size(), (size_t)cap));
  return static_cast<int64_t>(t.size());
}

// spmv_csr5 (spmv.hpp:58); mode 0 deterministic, 1 atomic.
int ref_spmv(void* hv, const double* x, double* y, int mode) {
  try {
    const auto& a5 = static_cast<RefHandle*>(hv)->a5;
    csr5::DenseVector xv(x, x + a5.n);
    csr5::spmv_csr5(a5, xv, std::span<double>(y, static_cast<std::size_t>(a5.m)),
                    mode ? csr5::SpmvMode::atomic : csr5::SpmvMode::deterministic);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// spmv_csr5 on a prebuilt x vector (no copy in the timed path).
struct RefVec {
  csr5::DenseVector v;
};
void* ref_vec_new(const double* x, int64_t n) { return new RefVec{csr5::DenseVector(x, x + n)}; }
void ref_vec_free(void* v) { delete static_cast<RefVec*>(v); }

// Times `iters` back-to-back spmv_csr5 calls (bench.cpp:147-160 protocol:
// one sample = the mean of `iters` calls); returns ms per call.
double ref_time_spmv(void* hv, void* xv, double* y, int mode, int iters) {
  const auto& a5 = static_cast<RefHandle*>(hv)->a5;
  const auto& x = static_cast<RefVec*>(xv)->v;
  std::span<double> ys(y, static_cast<std::size_t>(a5.m));
  const auto m = mode ? csr5::SpmvMode::atomic : csr5::SpmvMode::deterministic;
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) csr5::spmv_csr5(a5, x, ys, m);
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(t1 - t0).count() / iters;
}

double ref_time_csr_scalar(void* hv, void* xv, double* y, int iters) {
  const auto& a = static_cast<RefHandle*>(hv)->a;
  const auto& x = static_cast<RefVec*>(xv)->v;
  std::span<double> ys(y, static_cast<std::size_t>(a.m));
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) csr5::spmv_csr_scalar(a, x, ys);
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(t1 - t0).count() / iters;
}

// spmv_csr5_tile (spmv.hpp:53) -> count, or -1 when cap is too small.
int64_t ref_tile_contrib(void* hv, int64_t tid, const double* x, int64_t* rows, double* vals,
                         uint8_t* acc, int64_t cap) {
  try {
    const auto& a5 = static_cast<RefHandle*>(hv)->a5;
    csr5::DenseVector xv(x, x + a5.n);
    csr5::SpmvWorkspace ws;
    const auto c = csr5::spmv_csr5_tile(a5, tid, xv, ws);
    if (static_cast<int64_t>(c.size()) > cap) return -1;
    for (std::size_t k = 0; k < c.size(); ++k) {
      rows[k] = c[k].row;
      vals[k] = c[k].value;
      acc[k] = c[k].accumulate ? 1 : 0;
    }
    return static_cast<int64_t>(c.size());
  } catch (const std::exception& e) {
    fail(e);
    return -2;
  }
}

// csr5_to_csr (format.hpp:186) -> the recovered col_idx / val.
int ref_to_csr(void* hv, int64_t* col_idx, double* val) {
  try {
    const auto a = csr5::csr5_to_csr(static_cast<RefHandle*>(hv)->a5);
    std::memcpy(col_idx, a.col_idx.data(), a.col_idx.size() * sizeof(int64_t));
    std::memcpy(val, a.val.data(), a.val.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// dense_spmv_oracle (csr.hpp:51)
void ref_dense_spmv(int64_t m, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                    const double* val, const double* x, double* y) {
  csr5::CsrMatrix a;
  a.m = m;
  a.n = n;
  a.row_ptr.assign(row_ptr, row_ptr + m + 1);
  a.col_idx.assign(col_idx, col_idx + row_ptr[m]);
  a.val.assign(val, val + row_ptr[m]);
  const auto y2 = csr5::dense_spmv_oracle(a, csr5::DenseVector(x, x + n));
  std::memcpy(y, y2.data(), y2.size() * sizeof(double));
}

// select_sigma (tuning.hpp:29)
int ref_select_sigma(double npr, int64_t r, int64_t s, int64_t t, int64_t u, int64_t* out) {
  try {
    csr5::TuningParams p{.r = r, .s = s, .t = t, .u = u};
    *out = csr5::select_sigma(npr, p);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// generate_synthetic (synthetic.hpp:26): returns a malloc'd-by-new buffer
// handle; use ref_csr_get to copy out and ref_csr_free to release.
void* ref_generate(int kind, int64_t m, int64_t n, int64_t nnz, uint64_t seed, double frac,
                   int* rc) {
  try {
    auto* a = new csr5::CsrMatrix(csr5::generate_synthetic(
        static_cast<csr5::SyntheticKind>(kind), m, n, nnz, seed, frac));
    *rc = 0;
    return a;
  } catch (const std::exception& e) {
    *rc = fail(e);
    return nullptr;
  }
}
int64_t ref_csr_nnz(void* a) { return static_cast<csr5::CsrMatrix*>(a)->nnz(); }
void ref_csr_get(void* av, int64_t* row_ptr, int64_t* col_idx, double* val) {
  const auto* a = static_cast<csr5::CsrMatrix*>(av);
  std::memcpy(row_ptr, a->row_ptr.data(), a->row_ptr.size() * sizeof(int64_t));
  std::memcpy(col_idx, a->col_idx.data(), a->col_idx.size() * sizeof(int64_t));
  std::memcpy(val, a->val.data(), a->val.size() * sizeof(double));
}
void ref_csr_free(void* a) { delete static_cast<csr5::CsrMatrix*>(a); }

// bench.cpp:55-72 parse_kernel_list: kinds (0 csr-scalar, 1 csr-segsum,
// 2 csr5) into out[cap]; returns the count, or -(status) on an exception.
int ref_parse_kernels(const char* text, int* out, int cap) {
  try {
    const auto v = csr5::parse_kernel_list(text);
    int k = 0;
    for (auto kind : v)
      if (k < cap) out[k++] = static_cast<int>(kind);
    return static_cast<int>(v.size());
  } catch (const std::exception& e) {
    return -fail(e);
  }
}

// bench.cpp:86-90 iteration_speedup.
int ref_iteration_speedup(double t_csr, double t_pre, double t_new, int64_t n, double* out) {
  try {
    *out = csr5::iteration_speedup(t_csr, t_pre, t_new, n);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// bench.cpp:177-186 emit_csv over a report assembled from plain arrays
// (kernel names separated by '\n'); the CSV text goes to out[cap].
int64_t ref_emit_csv(const char* matrix, int64_t m, int64_t n, int64_t nnz, int threads,
                     int nk, const char* kernel_names, const double* best, const double* avg,
                     const double* gflops, const double* conv, const double* s50,
                     const double* s500, char* out, int64_t cap) {
  csr5::BenchReport r;
  r.matrix = matrix;
  r.m = m;
  r.n = n;
  r.nnz = nnz;
  r.threads = threads;
  std::stringstream names(kernel_names);
  for (int i = 0; i < nk; ++i) {
    csr5::KernelResult k;
    std::getline(names, k.kernel, '\n');
    k.best_ms = best[i];
    k.avg_ms = avg[i];
    k.gflops = gflops[i];
    k.conv_ms = conv[i];
    k.speedup_n50 = s50[i];
    k.speedup_n500 = s500[i];
    r.kernels.push_back(k);
  }
  std::ostringstream os;
  csr5::emit_csv(r, os);
  const std::string t = os.str();
  if ((int64_t)t.size() + 1 <= cap) std::memcpy(out, t.c_str(), t.size() + 1);
  return (int64_t)t.size();
}

// matrix_market.cpp:38-96 read_matrix_market: entries into a handle.
int ref_mm_read(const char* path, int64_t* m, int64_t* n, int64_t* count, void** out) {
  try {
    auto* d = new csr5::MatrixMarketData(csr5::read_matrix_market(std::string(path)));
    *m = d->m;
    *n = d->n;
    *count = (int64_t)d->entries.size();
    *out = d;
    return 0;
  } catch (const std::exception& e) {
    *out = nullptr;
    return fail(e);
  }
}
void ref_mm_get(void* h, int64_t* rows, int64_t* cols, double* vals) {
  const auto* d = static_cast<csr5::MatrixMarketData*>(h);
  for (size_t k = 0; k < d->entries.size(); ++k) {
    rows[k] = d->entries[k].row;
    cols[k] = d->entries[k].col;
    vals[k] = d->entries[k].value;
  }
}
void ref_mm_free(void* h) { delete static_cast<csr5::MatrixMarketData*>(h); }

// csr.cpp:35-72 coo_to_csr -> a CsrMatrix handle (ref_csr_nnz / ref_csr_get).
int ref_coo_to_csr(int64_t m, int64_t n, int64_t count, const int64_t* rows, const int64_t* cols,
                   const double* vals, void** out) {
  try {
    std::vector<csr5::CooEntry> e((size_t)count);
    for (int64_t k = 0; k < count; ++k) e[(size_t)k] = {rows[k], cols[k], vals[k]};
    *out = new csr5::CsrMatrix(csr5::coo_to_csr(std::move(e), m, n));
    return 0;
  } catch (const std::exception& ex) {
    *out = nullptr;
    return fail(ex);
  }
}

}  // extern "C"
