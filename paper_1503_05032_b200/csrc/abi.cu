// abi.cu -- the extern "C" boundary (include/csr5g.h).  Argument checking and
// error text follow the reference (tuning.cpp, descriptor.cpp, spmv.cpp:17-27);
// everything else forwards to convert.cu / spmv.cu.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

namespace csr5g {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& msg) { g_error = msg; }

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
            ") in " + what;
  cudaGetLastError();  // do not leak a non-sticky error into the next call
  return e == cudaErrorMemoryAllocation ? CSR5G_ENOMEM : CSR5G_ECUDA;
}

}  // namespace csr5g

using namespace csr5g;

namespace csr5g {
// device < 0: the calling thread's current CUDA device (the reference's API
// has no device argument)
int resolve_device(int* device) {
  int ndev = 0;
  CSR5G_CUDA(cudaGetDeviceCount(&ndev));
  if (*device < 0) CSR5G_CUDA(cudaGetDevice(device));
  if (*device >= ndev) return fail(CSR5G_ECUDA, "csr5g: no such CUDA device");
  return CSR5G_OK;
}
}  // namespace csr5g

struct csr5g_matrix_s {
  Handle* h;
};

extern "C" {

const char* csr5g_last_error(void) { return g_error.c_str(); }

const char* csr5g_version(void) { return "csr5g 0.1 sm_100a"; }

int csr5g_select_sigma(double nnz_per_row, int64_t r, int64_t s, int64_t t, int64_t u,
                       int64_t* out) {
  if (!out) return fail(CSR5G_EINVAL, "csr5g: out is NULL");
  if (!(r <= s && s <= t)) return fail(CSR5G_EINVAL, "select_sigma: bounds must satisfy r <= s <= t");
  if (nnz_per_row <= (double)r)
    *out = r;
  else if (nnz_per_row <= (double)s)
    *out = (int64_t)std::llround(nnz_per_row);
  else if (nnz_per_row <= (double)t)
    *out = s;
  else
    *out = u;
  return CSR5G_OK;
}

int csr5g_layout(int64_t omega, int64_t sigma, int32_t* yb, int32_t* sb, int32_t* wb) {
  if (omega < 1 || sigma < 1)
    return fail(CSR5G_EINVAL, "descriptor layout: omega and sigma must be >= 1");
  auto ceil_log2 = [](int64_t v) {
    const uint64_t x = (uint64_t)v - 1;
    return x ? 64 - __builtin_clzll(x) : 0;
  };
  const int y = ceil_log2(omega * sigma), s = ceil_log2(omega);
  const int64_t total = y + s + sigma;
  if (total > 64)
    return fail(CSR5G_EINVAL, "descriptor layout: " + std::to_string(total) +
                                  " bits per column exceed a 64-bit word; choose a smaller sigma");
  if (yb) *yb = y;
  if (sb) *sb = s;
  if (wb) *wb = total <= 32 ? 32 : 64;
  return CSR5G_OK;
}

static int wrap_build(int device, int64_t m, int64_t n, int64_t nnz, const int64_t* rp,
                      const int32_t* ci, const double* va, const csr5g_params* params, int64_t tb,
                      int64_t te, bool shard, int with_tail, void* stream, csr5g_matrix* out) {
  if (!out) return fail(CSR5G_EINVAL, "csr5g: out is NULL");
  *out = nullptr;
  Handle* h = nullptr;
  const int rc = build_handle(device, m, n, nnz, rp, ci, va, params, tb, te, shard, with_tail,
                              static_cast<cudaStream_t>(stream), &h);
  if (rc) return rc;
  *out = new csr5g_matrix_s{h};
  return CSR5G_OK;
}

int csr5g_build(int device, int64_t m, int64_t n, int64_t nnz, const int64_t* d_row_ptr,
                const int32_t* d_col_idx, const double* d_val, const csr5g_params* params,
                void* stream, csr5g_matrix* out) {
  return wrap_build(device, m, n, nnz, d_row_ptr, d_col_idx, d_val, params, 0, 0, false, 0, stream,
                    out);
}

int csr5g_build_shard(int device, int64_t m, int64_t n, int64_t nnz, const int64_t* d_row_ptr,
                      const int32_t* d_col_idx, const double* d_val, const csr5g_params* params,
                      int64_t tile_begin, int64_t tile_end, int32_t with_tail, void* stream,
                      csr5g_matrix* out) {
  return wrap_build(device, m, n, nnz, d_row_ptr, d_col_idx, d_val, params, tile_begin, tile_end,
                    true, with_tail, stream, out);
}

int csr5g_info_get(csr5g_matrix h, csr5g_info* out) {
  if (!h || !out) return fail(CSR5G_EINVAL, "csr5g: NULL handle");
  *out = h->h->info;
  return CSR5G_OK;
}

int csr5g_export(csr5g_matrix hm, uint64_t* h_tile_ptr, uint64_t* h_tile_desc, int64_t* h_eo_ptr,
                 int64_t* h_eo, int64_t* h_col_idx, double* h_val) {
  if (!hm) return fail(CSR5G_EINVAL, "csr5g: NULL handle");
  Handle* h = hm->h;
  CSR5G_CUDA(cudaSetDevice(h->device));
  CSR5G_CUDA(cudaDeviceSynchronize());
  const csr5g_info& in = h->info;
  const int64_t pcs = h->pcs;
  if (h_tile_ptr) {
    CSR5G_CUDA(cudaMemcpy(h_tile_ptr, h->tile_ptr, sizeof(uint32_t) * in.tile_ptr_len,
                          cudaMemcpyDeviceToHost));
    auto* w32 = reinterpret_cast<uint32_t*>(h_tile_ptr);
    for (int64_t i = in.tile_ptr_len - 1; i >= 0; --i) h_tile_ptr[i] = w32[i];
  }
  if (h_tile_desc) {
    const int64_t cnt = pcs * kOmega;
    if (h->wide) {
      CSR5G_CUDA(cudaMemcpy(h_tile_desc, h->desc, sizeof(uint64_t) * cnt, cudaMemcpyDeviceToHost));
    } else {
      CSR5G_CUDA(cudaMemcpy(h_tile_desc, h->desc, sizeof(uint32_t) * cnt, cudaMemcpyDeviceToHost));
      auto* w32 = reinterpret_cast<uint32_t*>(h_tile_desc);
      for (int64_t i = cnt - 1; i >= 0; --i) h_tile_desc[i] = w32[i];
    }
  }
  if (h_eo_ptr)
    CSR5G_CUDA(cudaMemcpy(h_eo_ptr, h->eo_ptr, sizeof(int64_t) * (pcs + 1), cudaMemcpyDeviceToHost));
  if (h_eo) {
    CSR5G_CUDA(cudaMemcpy(h_eo, h->eo, sizeof(int32_t) * in.empty_offset_len, cudaMemcpyDeviceToHost));
    auto* w32 = reinterpret_cast<int32_t*>(h_eo);
    for (int64_t i = in.empty_offset_len - 1; i >= 0; --i) h_eo[i] = w32[i];
  }
  if (h_col_idx) {
    CSR5G_CUDA(cudaMemcpy(h_col_idx, h->col, sizeof(int32_t) * in.nnz_held, cudaMemcpyDeviceToHost));
    auto* w32 = reinterpret_cast<int32_t*>(h_col_idx);
    for (int64_t i = in.nnz_held - 1; i >= 0; --i) h_col_idx[i] = w32[i];
  }
  if (h_val)
    CSR5G_CUDA(cudaMemcpy(h_val, h->val, sizeof(double) * in.nnz_held, cudaMemcpyDeviceToHost));
  return CSR5G_OK;
}

int csr5g_spmv(csr5g_matrix h, const double* d_x, double* d_y, int32_t mode, void* stream) {
  return csr5g_spmv_evt(h, d_x, d_y, mode, stream, nullptr, nullptr);
}

int csr5g_spmv_evt(csr5g_matrix h, const double* d_x, double* d_y, int32_t mode, void* stream,
                   void* ev0, void* ev1) {
  if (!h) return fail(CSR5G_EINVAL, "csr5g: NULL handle");
  if (mode != CSR5G_MODE_DETERMINISTIC && mode != CSR5G_MODE_ATOMIC)
    return fail(CSR5G_EINVAL, "csr5g: unknown spmv mode " + std::to_string(mode));
  if (h->h->info.m > 0 && !d_y) return fail(CSR5G_EINVAL, "spmv: y is NULL");
  if (h->h->info.n > 0 && !d_x) return fail(CSR5G_EINVAL, "spmv: x is NULL");
  return launch_spmv(h->h, d_x, d_y, mode, static_cast<cudaStream_t>(stream),
                     static_cast<cudaEvent_t>(ev0), static_cast<cudaEvent_t>(ev1));
}

int csr5g_shard_send_record(csr5g_matrix h, csr5g_partial** d_send) {
  if (!h || !d_send) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  *d_send = h->h->send;
  return CSR5G_OK;
}

int csr5g_set_send_buffer(csr5g_matrix h, csr5g_partial* d_send) {
  if (!h) return fail(CSR5G_EINVAL, "csr5g: NULL handle");
  h->h->send_ext = d_send;
  return CSR5G_OK;
}

int csr5g_fixup(csr5g_matrix h, const csr5g_partial* d_all, int32_t world, int32_t rank,
                double* d_y, void* stream) {
  if (!h || !d_all || !d_y) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  if (rank < 0 || rank >= world) return fail(CSR5G_EINVAL, "csr5g: rank outside [0, world)");
  return launch_fixup(h->h, d_all, world, rank, d_y, static_cast<cudaStream_t>(stream));
}

int csr5g_to_csr(csr5g_matrix h, int32_t* d_col_idx, double* d_val, void* stream) {
  if (!h) return fail(CSR5G_EINVAL, "csr5g: NULL handle");
  if (h->h->info.nnz_held > 0 && (!d_col_idx || !d_val))
    return fail(CSR5G_EINVAL, "csr5g: NULL output");
  return launch_to_csr(h->h, d_col_idx, d_val, static_cast<cudaStream_t>(stream));
}

int csr5g_build_host(int device, int64_t m, int64_t n, int64_t nnz, const int64_t* h_row_ptr,
                     const int64_t* h_col_idx, const double* h_val, const csr5g_params* params,
                     csr5g_matrix* out) {
  if (!out) return fail(CSR5G_EINVAL, "csr5g: out is NULL");
  *out = nullptr;
  if (m < 0 || n < 0 || nnz < 0) return fail(CSR5G_EINVAL, "csr: negative dimension");
  if (n >= (int64_t(1) << 31))
    return fail(CSR5G_ERANGE, "csr5g: n >= 2^31 columns does not fit the int32 col_idx");
  if (m > 0 && !h_row_ptr) return fail(CSR5G_EINVAL, "csr5g: row_ptr is NULL");
  if (m > 0 && h_row_ptr[m] != nnz)
    return fail(CSR5G_EINVAL, "csr: col_idx/val size does not match row_ptr[m]");
  if (int rc = resolve_device(&device)) return rc;
  CSR5G_CUDA(cudaSetDevice(device));
  std::vector<int32_t> c32((size_t)nnz);
  for (int64_t i = 0; i < nnz; ++i) c32[(size_t)i] = (int32_t)h_col_idx[i];
  int64_t* d_rp = nullptr;
  int32_t* d_ci = nullptr;
  double* d_va = nullptr;
  auto done = [&](int rc) {
    cudaFree(d_rp);
    cudaFree(d_ci);
    cudaFree(d_va);
    return rc;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&d_rp, sizeof(int64_t) * (m + 1))) != cudaSuccess ||
      (e = cudaMalloc(&d_ci, sizeof(int32_t) * std::max<int64_t>(nnz, 1))) != cudaSuccess ||
      (e = cudaMalloc(&d_va, sizeof(double) * std::max<int64_t>(nnz, 1))) != cudaSuccess)
    return done(cuda_fail(e, "cudaMalloc(staging)"));
  if (m > 0 && (e = cudaMemcpy(d_rp, h_row_ptr, sizeof(int64_t) * (m + 1),
                               cudaMemcpyHostToDevice)) != cudaSuccess)
    return done(cuda_fail(e, "cudaMemcpy(row_ptr)"));
  if (nnz > 0 && ((e = cudaMemcpy(d_ci, c32.data(), sizeof(int32_t) * nnz,
                                  cudaMemcpyHostToDevice)) != cudaSuccess ||
                  (e = cudaMemcpy(d_va, h_val, sizeof(double) * nnz, cudaMemcpyHostToDevice)) !=
                      cudaSuccess))
    return done(cuda_fail(e, "cudaMemcpy(col_idx/val)"));
  return done(csr5g_build(device, m, n, nnz, d_rp, d_ci, d_va, params, nullptr, out));
}

static int check_mode(int32_t mode) {
  if (mode != CSR5G_MODE_DETERMINISTIC && mode != CSR5G_MODE_ATOMIC)
    return fail(CSR5G_EINVAL, "csr5g: unknown spmv mode " + std::to_string(mode));
  return CSR5G_OK;
}

int csr5g_spmv_host(csr5g_matrix h, const double* h_x, double* h_y, int32_t mode) {
  if (!h) return fail(CSR5G_EINVAL, "csr5g: NULL handle");
  const csr5g_info& in = h->h->info;
  if (in.m > 0 && !h_y) return fail(CSR5G_EINVAL, "spmv: y is NULL");
  if (in.n > 0 && !h_x) return fail(CSR5G_EINVAL, "spmv: x is NULL");
  if (int rc = check_mode(mode)) return rc;
  int rc = spmv_host_batch(h->h, &h_x, &h_y, 1, mode, nullptr);
  if (rc) return rc;
  CSR5G_CUDA(cudaStreamSynchronize(nullptr));
  return CSR5G_OK;
}

int csr5g_spmv_host_batch(csr5g_matrix h, const double* const* h_xs, double* const* h_ys,
                          int64_t count, int32_t mode, void* stream) {
  if (!h) return fail(CSR5G_EINVAL, "csr5g: NULL handle");
  if (count < 0) return fail(CSR5G_EINVAL, "csr5g: negative batch count");
  if (count == 0) return CSR5G_OK;
  if (!h_xs || !h_ys) return fail(CSR5G_EINVAL, "csr5g: NULL vector list");
  const csr5g_info& in = h->h->info;
  for (int64_t k = 0; k < count; ++k) {
    if (in.m > 0 && !h_ys[k]) return fail(CSR5G_EINVAL, "spmv: y is NULL");
    if (in.n > 0 && !h_xs[k]) return fail(CSR5G_EINVAL, "spmv: x is NULL");
  }
  if (int rc = check_mode(mode)) return rc;
  return spmv_host_batch(h->h, h_xs, h_ys, count, mode, static_cast<cudaStream_t>(stream));
}

int csr5g_csr_spmv(int device, int32_t kernel, int64_t m, int64_t n, int64_t nnz,
                   const int64_t* d_row_ptr, const int32_t* d_col_idx, const double* d_val,
                   const double* d_x, double* d_y, void* stream) {
  if (kernel != CSR5G_CSR_SCALAR && kernel != CSR5G_CSR_SEGSUM)
    return fail(CSR5G_EINVAL, "csr5g: unknown CSR kernel " + std::to_string(kernel));
  if (m < 0 || n < 0 || nnz < 0) return fail(CSR5G_EINVAL, "csr: negative dimension");
  if (m > 0 && (!d_row_ptr || !d_y)) return fail(CSR5G_EINVAL, "spmv: row_ptr or y is NULL");
  if (nnz > 0 && (!d_col_idx || !d_val || !d_x))
    return fail(CSR5G_EINVAL, "spmv: col_idx, val or x is NULL");
  if (m >= (int64_t(1) << 31))
    return fail(CSR5G_ERANGE, "csr5g: m >= 2^31 rows is unsupported");
  return csr_spmv(device, kernel, m, n, nnz, d_row_ptr, d_col_idx, d_val, d_x, d_y,
                  static_cast<cudaStream_t>(stream));
}

int csr5g_csr_spmv_host(int device, int32_t kernel, int64_t m, int64_t n, int64_t nnz,
                        const int64_t* h_row_ptr, const int64_t* h_col_idx, const double* h_val,
                        const double* h_x, double* h_y) {
  if (m < 0 || n < 0 || nnz < 0) return fail(CSR5G_EINVAL, "csr: negative dimension");
  if (m > 0 && (!h_row_ptr || !h_y)) return fail(CSR5G_EINVAL, "spmv: row_ptr or y is NULL");
  if (nnz > 0 && (!h_col_idx || !h_val || !h_x))
    return fail(CSR5G_EINVAL, "spmv: col_idx, val or x is NULL");
  if (m > 0 && h_row_ptr[m] != nnz)
    return fail(CSR5G_EINVAL, "csr: col_idx/val size does not match row_ptr[m]");
  if (n >= (int64_t(1) << 31))
    return fail(CSR5G_ERANGE, "csr5g: n >= 2^31 columns does not fit the int32 col_idx");
  if (int rc = resolve_device(&device)) return rc;
  CSR5G_CUDA(cudaSetDevice(device));
  std::vector<int32_t> c32((size_t)nnz);
  for (int64_t i = 0; i < nnz; ++i) c32[(size_t)i] = (int32_t)h_col_idx[i];
  int64_t* d_rp = nullptr;
  int32_t* d_ci = nullptr;
  double *d_va = nullptr, *d_x = nullptr, *d_y = nullptr;
  auto done = [&](int rc) {
    for (void* q : {(void*)d_rp, (void*)d_ci, (void*)d_va, (void*)d_x, (void*)d_y}) cudaFree(q);
    return rc;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&d_rp, sizeof(int64_t) * (m + 1))) != cudaSuccess ||
      (e = cudaMalloc(&d_ci, sizeof(int32_t) * std::max<int64_t>(nnz, 1))) != cudaSuccess ||
      (e = cudaMalloc(&d_va, sizeof(double) * std::max<int64_t>(nnz, 1))) != cudaSuccess ||
      (e = cudaMalloc(&d_x, sizeof(double) * std::max<int64_t>(n, 1))) != cudaSuccess ||
      (e = cudaMalloc(&d_y, sizeof(double) * std::max<int64_t>(m, 1))) != cudaSuccess)
    return done(cuda_fail(e, "cudaMalloc(csr staging)"));
  if ((m > 0 && (e = cudaMemcpy(d_rp, h_row_ptr, sizeof(int64_t) * (m + 1),
                                cudaMemcpyHostToDevice)) != cudaSuccess) ||
      (nnz > 0 && ((e = cudaMemcpy(d_ci, c32.data(), sizeof(int32_t) * nnz,
                                   cudaMemcpyHostToDevice)) != cudaSuccess ||
                   (e = cudaMemcpy(d_va, h_val, sizeof(double) * nnz, cudaMemcpyHostToDevice)) !=
                       cudaSuccess)) ||
      (n > 0 && (e = cudaMemcpy(d_x, h_x, sizeof(double) * n, cudaMemcpyHostToDevice)) !=
                    cudaSuccess))
    return done(cuda_fail(e, "cudaMemcpy(csr staging)"));
  int rc = csr5g_csr_spmv(device, kernel, m, n, nnz, d_rp, d_ci, d_va, d_x, d_y, nullptr);
  if (rc) return done(rc);
  if (m > 0 && (e = cudaMemcpy(h_y, d_y, sizeof(double) * m, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return done(cuda_fail(e, "cudaMemcpy(y)"));
  return done(CSR5G_OK);
}

int csr5g_spmv_tile(csr5g_matrix hm, int64_t tid, const double* h_x, int64_t* h_rows,
                    double* h_vals, uint8_t* h_acc, int64_t cap, int64_t* count) {
  if (!hm || !count) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  Handle* h = hm->h;
  const csr5g_info& in = h->info;
  if (tid < in.tile_begin || tid >= in.tile_end)
    return fail(CSR5G_EINVAL, "spmv_csr5_tile: tile " + std::to_string(tid) +
                                  " is not a complete tile");
  if (in.n > 0 && !h_x) return fail(CSR5G_EINVAL, "csr5g: x is NULL");
  const int64_t k = tid - in.tile_begin, B = h->B;
  CSR5G_CUDA(cudaSetDevice(h->device));
  double *d_x = nullptr, *d_vals = nullptr;
  int64_t* d_rows = nullptr;
  int32_t* d_count = nullptr;
  auto done = [&](int rc) {
    for (void* q : {(void*)d_x, (void*)d_vals, (void*)d_rows, (void*)d_count}) cudaFree(q);
    return rc;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&d_x, sizeof(double) * std::max<int64_t>(in.n, 1))) != cudaSuccess ||
      (e = cudaMalloc(&d_vals, sizeof(double) * B)) != cudaSuccess ||
      (e = cudaMalloc(&d_rows, sizeof(int64_t) * B)) != cudaSuccess ||
      (e = cudaMalloc(&d_count, sizeof(int32_t))) != cudaSuccess)
    return done(cuda_fail(e, "cudaMalloc(tile trace)"));
  if (in.n > 0 && (e = cudaMemcpy(d_x, h_x, sizeof(double) * in.n, cudaMemcpyHostToDevice)) !=
                      cudaSuccess)
    return done(cuda_fail(e, "cudaMemcpy(x)"));
  if (int rc = launch_tile_trace(h, k, d_x, d_rows, d_vals, d_count, nullptr)) return done(rc);
  int32_t H = 0;
  if ((e = cudaMemcpy(&H, d_count, sizeof H, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return done(cuda_fail(e, "tile trace"));
  std::vector<int64_t> rows((size_t)H);
  std::vector<double> vals((size_t)H);
  std::vector<uint64_t> words(kOmega);
  const size_t wb = h->wide ? 8 : 4;
  std::vector<unsigned char> raw(kOmega * wb);
  if ((e = cudaMemcpy(rows.data(), d_rows, sizeof(int64_t) * H, cudaMemcpyDeviceToHost)) !=
          cudaSuccess ||
      (e = cudaMemcpy(vals.data(), d_vals, sizeof(double) * H, cudaMemcpyDeviceToHost)) !=
          cudaSuccess ||
      (e = cudaMemcpy(raw.data(), static_cast<const unsigned char*>(h->desc) + k * kOmega * wb,
                      kOmega * wb, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return done(cuda_fail(e, "tile trace"));
  for (int i = 0; i < kOmega; ++i) {
    uint64_t w = 0;
    std::memcpy(&w, raw.data() + i * wb, wb);
    words[i] = w;
  }
  if (cap < H) return done(fail(CSR5G_EINVAL, "csr5g: tile contribution buffer too small"));
  // the reference's emission order (spmv.cpp:61-105): per column, the
  // segments sealed inside it top to bottom (accumulate only for head 0),
  // then every head-bearing column's bottom piece (accumulate)
  const int sigma = (int)in.sigma;
  const uint64_t fmask = sigma >= 64 ? ~0ull : (1ull << sigma) - 1;
  int64_t q = 0;
  auto emit = [&](int64_t head, bool acc) {
    if (h_rows) h_rows[q] = rows[(size_t)head];
    if (h_vals) h_vals[q] = vals[(size_t)head];
    if (h_acc) h_acc[q] = acc ? 1 : 0;
    ++q;
  };
  for (int pass = 0; pass < 2; ++pass)
    for (int i = 0; i < kOmega; ++i) {
      const int64_t y = (int64_t)(words[i] >> (kSegBits + sigma));
      const int cnt = __builtin_popcountll(words[i] & fmask);
      if (pass == 0)
        for (int s = 0; s + 1 < cnt; ++s) emit(y + s, y + s == 0);
      else if (cnt > 0)
        emit(y + cnt - 1, true);
    }
  *count = q;
  return done(q == H ? CSR5G_OK : fail(CSR5G_ERUNTIME, "csr5g: tile trace head count mismatch"));
}

int csr5g_export_row_ptr(csr5g_matrix hm, int64_t* h_row_ptr) {
  if (!hm || !h_row_ptr) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  Handle* h = hm->h;
  CSR5G_CUDA(cudaSetDevice(h->device));
  CSR5G_CUDA(cudaDeviceSynchronize());
  if (h->info.m == 0) {
    h_row_ptr[0] = 0;
    return CSR5G_OK;
  }
  CSR5G_CUDA(cudaMemcpy(h_row_ptr, h->row_ptr, sizeof(int64_t) * (h->info.m + 1),
                        cudaMemcpyDeviceToHost));
  return CSR5G_OK;
}

int csr5g_to_csr_host(csr5g_matrix h, int64_t* h_col_idx, double* h_val) {
  if (!h) return fail(CSR5G_EINVAL, "csr5g: NULL handle");
  const int64_t nz = h->h->info.nnz_held;
  CSR5G_CUDA(cudaSetDevice(h->h->device));
  int32_t* dc = nullptr;
  double* dv = nullptr;
  auto done = [&](int rc) {
    cudaFree(dc);
    cudaFree(dv);
    return rc;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&dc, sizeof(int32_t) * std::max<int64_t>(nz, 1))) != cudaSuccess ||
      (e = cudaMalloc(&dv, sizeof(double) * std::max<int64_t>(nz, 1))) != cudaSuccess)
    return done(cuda_fail(e, "cudaMalloc(csr)"));
  int rc = csr5g_to_csr(h, dc, dv, nullptr);
  if (rc) return done(rc);
  std::vector<int32_t> c32((size_t)nz);
  if (nz > 0 && ((e = cudaMemcpy(c32.data(), dc, sizeof(int32_t) * nz, cudaMemcpyDeviceToHost)) !=
                     cudaSuccess ||
                 (e = cudaMemcpy(h_val, dv, sizeof(double) * nz, cudaMemcpyDeviceToHost)) !=
                     cudaSuccess))
    return done(cuda_fail(e, "cudaMemcpy(csr)"));
  for (int64_t i = 0; i < nz; ++i) h_col_idx[i] = c32[(size_t)i];
  return done(CSR5G_OK);
}

int csr5g_release(csr5g_matrix h) {
  if (!h) return CSR5G_OK;
  free_handle(h->h);
  delete h;
  return CSR5G_OK;
}

int csr5g_event_create(void** ev) {
  if (!ev) return fail(CSR5G_EINVAL, "csr5g: NULL event");
  cudaEvent_t e;
  CSR5G_CUDA(cudaEventCreate(&e));
  *ev = e;
  return CSR5G_OK;
}

int csr5g_event_record(void* ev, void* stream) {
  CSR5G_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), static_cast<cudaStream_t>(stream)));
  return CSR5G_OK;
}

int csr5g_event_elapsed_ms(void* a, void* b, float* ms) {
  CSR5G_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(b)));
  CSR5G_CUDA(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(a), static_cast<cudaEvent_t>(b)));
  return CSR5G_OK;
}

int csr5g_event_destroy(void* ev) {
  CSR5G_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(ev)));
  return CSR5G_OK;
}

int csr5g_stream_synchronize(void* stream) {
  CSR5G_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return CSR5G_OK;
}

}  // extern "C"
