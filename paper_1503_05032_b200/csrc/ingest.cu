// ingest.cu -- matrices from files: the Matrix Market reader (host) and the
// COO -> CSR conversion (device).
//
// Reader (matrix_market.cpp:38-103): ASCII coordinate files with field real /
// integer / pattern and symmetry general / symmetric; banner, size line and
// entries are tokenised with the C++ stream extractors, so what parses, what
// is rejected and the "matrix market: line N: ..." texts are the reference's.
// Symmetric files are expanded while reading (mirror entry right after its
// source, diagonal once); indices become 0-based.
//
// COO -> CSR (csr.cpp:35-72) on the device:
//   1. bounds: the first out-of-range entry (atomicMin over its position)
//      raises the reference's std::invalid_argument text;
//   2. a stable radix sort of (row << 31 | col) keys carrying the values, so
//      duplicates keep their input order;
//   3. run heads (key changes) compacted by a scan; each head sums its run
//      left to right from 0.0 -- the reference's `sum += value` order, so the
//      summed values are bit-identical;
//   4. row_ptr from per-row counts (atomics) and an inclusive scan.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "internal.cuh"

struct csr5g_coo_s {
  int64_t m = 0, n = 0;
  std::vector<int64_t> rows, cols;
  std::vector<double> vals;
};

namespace csr5g {
namespace {

std::string lowercase(std::string s) {
  for (char& c : s) c = (char)std::tolower((unsigned char)c);
  return s;
}

struct LineReader {
  std::istream& in;
  size_t line = 0;
  // next line holding data: skips blank lines and '%' comments, drops a '\r'
  bool data(std::string& s) {
    while (std::getline(in, s)) {
      ++line;
      if (!s.empty() && s.back() == '\r') s.pop_back();
      const size_t p = s.find_first_not_of(" \t");
      if (p != std::string::npos && s[p] != '%') return true;
    }
    return false;
  }
};

struct MmError {
  std::string msg;
};

[[noreturn]] void at_line(size_t line, const std::string& what) {
  throw MmError{"matrix market: line " + std::to_string(line) + ": " + what};
}

void parse_mm(std::istream& in, csr5g_coo_s& out) {
  LineReader rd{in};
  std::string s;
  if (!std::getline(in, s)) throw MmError{"matrix market: empty input"};
  rd.line = 1;
  if (!s.empty() && s.back() == '\r') s.pop_back();
  std::string tok[5];
  {
    std::istringstream hs(s);
    for (auto& t : tok) hs >> t;
  }
  const std::string object = tok[1];
  const std::string fmt = lowercase(tok[2]), field = lowercase(tok[3]), sym = lowercase(tok[4]);
  if (lowercase(tok[0]) != "%%matrixmarket") at_line(1, "missing %%MatrixMarket banner");
  if (lowercase(object) != "matrix") at_line(1, "unsupported object '" + object + "'");
  if (fmt != "coordinate")
    at_line(1, "unsupported format '" + fmt + "' (only coordinate is supported)");
  if (field == "complex") at_line(1, "complex field is not supported");
  if (field != "real" && field != "integer" && field != "pattern")
    at_line(1, "unsupported field '" + field + "'");
  if (sym != "general" && sym != "symmetric") at_line(1, "unsupported symmetry '" + sym + "'");

  if (!rd.data(s)) throw MmError{"matrix market: missing size line"};
  int64_t m = 0, n = 0, declared = 0;
  {
    std::istringstream ss(s);
    if (!(ss >> m >> n >> declared) || m < 0 || n < 0 || declared < 0)
      at_line(rd.line, "malformed size line '" + s + "'");
  }
  const bool pattern = field == "pattern", symmetric = sym == "symmetric";
  out.m = m;
  out.n = n;
  const size_t cap = (size_t)(symmetric ? 2 * declared : declared);
  out.rows.reserve(cap);
  out.cols.reserve(cap);
  out.vals.reserve(cap);
  for (int64_t k = 0; k < declared; ++k) {
    if (!rd.data(s))
      throw MmError{"matrix market: expected " + std::to_string(declared) + " entries, got " +
                    std::to_string(k)};
    std::istringstream es(s);
    int64_t r = 0, c = 0;
    double v = 1.0;
    if (!(es >> r >> c)) at_line(rd.line, "malformed entry '" + s + "'");
    if (!pattern && !(es >> v)) at_line(rd.line, "missing value in entry '" + s + "'");
    if (r < 1 || r > m || c < 1 || c > n)
      at_line(rd.line, "index (" + std::to_string(r) + ", " + std::to_string(c) + ") outside " +
                           std::to_string(m) + "x" + std::to_string(n));
    out.rows.push_back(r - 1);
    out.cols.push_back(c - 1);
    out.vals.push_back(v);
    if (symmetric && r != c) {
      out.rows.push_back(c - 1);
      out.cols.push_back(r - 1);
      out.vals.push_back(v);
    }
  }
}

// ---- device COO -> CSR ---------------------------------------------------------
__global__ void k_first_bad(int64_t count, const int64_t* __restrict__ rows,
                            const int64_t* __restrict__ cols, int64_t m, int64_t n,
                            unsigned long long* __restrict__ first) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows[k], c = cols[k];
    if (r < 0 || r >= m || c < 0 || c >= n) atomicMin(first, (unsigned long long)k);
  }
}

__global__ void k_keys(int64_t count, const int64_t* __restrict__ rows,
                       const int64_t* __restrict__ cols, uint64_t* __restrict__ keys) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x)
    keys[k] = ((uint64_t)rows[k] << 31) | (uint64_t)cols[k];
}

__global__ void k_heads(int64_t count, const uint64_t* __restrict__ keys,
                        int64_t* __restrict__ head) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x)
    head[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0;
}

// pos = inclusive scan of head: a head at k writes unique entry pos[k] - 1
__global__ void k_runs(int64_t count, const uint64_t* __restrict__ keys,
                       const double* __restrict__ vals, const int64_t* __restrict__ pos,
                       int32_t* __restrict__ col_out, double* __restrict__ val_out,
                       unsigned long long* __restrict__ row_cnt) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < count;
       k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[k];
    if (k > 0 && keys[k - 1] == key) continue;
    double s = 0.0;
    for (int64_t j = k; j < count && keys[j] == key; ++j) s += vals[j];
    const int64_t u = pos[k] - 1;
    col_out[u] = (int32_t)(key & 0x7fffffffu);
    val_out[u] = s;
    atomicAdd(row_cnt + (key >> 31), 1ull);
  }
}

}  // namespace
}  // namespace csr5g

using namespace csr5g;

extern "C" {

int csr5g_mm_read(const char* path, csr5g_coo* out, int64_t* m, int64_t* n, int64_t* count) {
  if (!path || !out || !m || !n || !count) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  *out = nullptr;
  std::ifstream in(path);
  if (!in) return fail(CSR5G_ERUNTIME, std::string("matrix market: cannot open '") + path + "'");
  auto* c = new csr5g_coo_s;
  try {
    parse_mm(in, *c);
  } catch (const MmError& e) {
    delete c;
    return fail(CSR5G_ERUNTIME, e.msg);
  } catch (const std::bad_alloc&) {
    delete c;
    return fail(CSR5G_ENOMEM, "matrix market: out of host memory");
  }
  *out = c;
  *m = c->m;
  *n = c->n;
  *count = (int64_t)c->rows.size();
  return CSR5G_OK;
}

int csr5g_mm_parse(const char* text, int64_t len, csr5g_coo* out, int64_t* m, int64_t* n,
                   int64_t* count) {
  if ((!text && len > 0) || len < 0 || !out || !m || !n || !count)
    return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  *out = nullptr;
  std::istringstream in(std::string(text ? text : "", (size_t)len));
  auto* c = new csr5g_coo_s;
  try {
    parse_mm(in, *c);
  } catch (const MmError& e) {
    delete c;
    return fail(CSR5G_ERUNTIME, e.msg);
  } catch (const std::bad_alloc&) {
    delete c;
    return fail(CSR5G_ENOMEM, "matrix market: out of host memory");
  }
  *out = c;
  *m = c->m;
  *n = c->n;
  *count = (int64_t)c->rows.size();
  return CSR5G_OK;
}

int csr5g_coo_get(csr5g_coo c, int64_t* h_rows, int64_t* h_cols, double* h_vals) {
  if (!c) return fail(CSR5G_EINVAL, "csr5g: NULL COO");
  if (h_rows) std::copy(c->rows.begin(), c->rows.end(), h_rows);
  if (h_cols) std::copy(c->cols.begin(), c->cols.end(), h_cols);
  if (h_vals) std::copy(c->vals.begin(), c->vals.end(), h_vals);
  return CSR5G_OK;
}

int csr5g_coo_release(csr5g_coo c) {
  delete c;
  return CSR5G_OK;
}

int csr5g_coo_to_csr(int device, int64_t m, int64_t n, int64_t count, const int64_t* d_rows,
                     const int64_t* d_cols, const double* d_vals, int64_t* d_row_ptr,
                     int32_t* d_col_idx, double* d_val, int64_t* nnz, void* stream_v) {
  if (!nnz) return fail(CSR5G_EINVAL, "csr5g: nnz is NULL");
  *nnz = 0;
  if (m < 0 || n < 0 || count < 0) return fail(CSR5G_EINVAL, "csr: negative dimension");
  if (m >= (int64_t(1) << 31) || n >= (int64_t(1) << 31))
    return fail(CSR5G_ERANGE, "csr5g: m or n >= 2^31 does not fit the device CSR");
  if (!d_row_ptr || (count > 0 && (!d_rows || !d_cols || !d_vals || !d_col_idx || !d_val)))
    return fail(CSR5G_EINVAL, "csr5g: NULL device buffer");
  if (int rc = resolve_device(&device)) return rc;
  CSR5G_CUDA(cudaSetDevice(device));
  cudaStream_t st = static_cast<cudaStream_t>(stream_v);
  int sms = 148;
  CSR5G_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  auto grid = [&](int64_t work) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, (int64_t)sms * 16));
  };
  // scratch: first-bad + row counts (m+1, as u64) + keys x2 + values x2 + heads + pos + CUB
  unsigned long long* first = nullptr;
  unsigned long long* cnt = nullptr;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  double* v1 = nullptr;
  int64_t *head = nullptr, *pos = nullptr;
  void* tmp = nullptr;
  auto done = [&](int rc) {
    for (void* p : {(void*)first, (void*)cnt, (void*)k0, (void*)k1, (void*)v1,
                    (void*)head, (void*)pos, tmp})
      if (p) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    return rc;
  };
#define CK(call)                                         \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return done(cuda_fail(e_, #call)); \
  } while (0)
  CK(cudaMallocAsync(&first, sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), st));
  if (count > 0) {
    k_first_bad<<<grid(count), 256, 0, st>>>(count, d_rows, d_cols, m, n, first);
    CK(cudaGetLastError());
  }
  unsigned long long bad = ~0ull;
  CK(cudaMemcpyAsync(&bad, first, sizeof bad, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (bad != ~0ull) {
    int64_t r = 0, c = 0;
    CK(cudaMemcpy(&r, d_rows + bad, sizeof r, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&c, d_cols + bad, sizeof c, cudaMemcpyDeviceToHost));
    return done(fail(CSR5G_EINVAL, "coo entry " + std::to_string(bad) + " out of bounds: (" +
                                       std::to_string(r) + ", " + std::to_string(c) +
                                       ") for a " + std::to_string(m) + "x" + std::to_string(n) +
                                       " matrix"));
  }
  CK(cudaMallocAsync(&cnt, sizeof(unsigned long long) * (m + 1), st));
  CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * (m + 1), st));
  int64_t uniq = 0;
  if (count > 0) {
    CK(cudaMallocAsync(&k0, sizeof(uint64_t) * count, st));
    CK(cudaMallocAsync(&k1, sizeof(uint64_t) * count, st));
    CK(cudaMallocAsync(&v1, sizeof(double) * count, st));
    CK(cudaMallocAsync(&head, sizeof(int64_t) * count, st));
    CK(cudaMallocAsync(&pos, sizeof(int64_t) * count, st));
    k_keys<<<grid(count), 256, 0, st>>>(count, d_rows, d_cols, k0);
    CK(cudaGetLastError());
    int end_bit = 31;
    while (end_bit < 64 && (m - 1) >> (end_bit - 31)) ++end_bit;
    size_t tb = 0, tb2 = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, d_vals, v1, count, 0, end_bit, st));
    CK(cub::DeviceScan::InclusiveSum(nullptr, tb2, head, pos, count, st));
    tb = std::max(tb, tb2);
    CK(cudaMallocAsync(&tmp, tb, st));
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, d_vals, v1, count, 0, end_bit, st));
    k_heads<<<grid(count), 256, 0, st>>>(count, k1, head);
    CK(cudaGetLastError());
    CK(cub::DeviceScan::InclusiveSum(tmp, tb, head, pos, count, st));
    k_runs<<<grid(count), 256, 0, st>>>(count, k1, v1, pos, d_col_idx, d_val, cnt + 1);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&uniq, pos + count - 1, sizeof uniq, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(tmp, st));
    tmp = nullptr;
  }
  // row_ptr[0] = 0, row_ptr[r + 1] = row_ptr[r] + count(r)
  size_t tb = 0;
  CK(cub::DeviceScan::InclusiveSum(nullptr, tb, cnt, reinterpret_cast<unsigned long long*>(d_row_ptr),
                                   m + 1, st));
  CK(cudaMallocAsync(&tmp, tb, st));
  CK(cub::DeviceScan::InclusiveSum(tmp, tb, cnt, reinterpret_cast<unsigned long long*>(d_row_ptr),
                                   m + 1, st));
#undef CK
  int rc = done(CSR5G_OK);
  if (rc == CSR5G_OK) *nnz = uniq;
  return rc;
}

int csr5g_coo_to_csr_host(int device, int64_t m, int64_t n, int64_t count, const int64_t* h_rows,
                          const int64_t* h_cols, const double* h_vals, int64_t* h_row_ptr,
                          int64_t* h_col_idx, double* h_val, int64_t* nnz) {
  if (!nnz || !h_row_ptr || (count > 0 && (!h_rows || !h_cols || !h_vals || !h_col_idx || !h_val)))
    return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  *nnz = 0;
  if (m < 0 || n < 0 || count < 0) return fail(CSR5G_EINVAL, "csr: negative dimension");
  if (int rc = resolve_device(&device)) return rc;
  CSR5G_CUDA(cudaSetDevice(device));
  const size_t k = (size_t)std::max<int64_t>(count, 1);
  int64_t *dr = nullptr, *dc = nullptr, *drp = nullptr;
  double *dv = nullptr, *dov = nullptr;
  int32_t* doc = nullptr;
  auto done = [&](int rc) {
    for (void* p : {(void*)dr, (void*)dc, (void*)drp, (void*)dv, (void*)dov, (void*)doc})
      if (p) cudaFree(p);
    return rc;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&dr, 8 * k)) || (e = cudaMalloc(&dc, 8 * k)) || (e = cudaMalloc(&dv, 8 * k)) ||
      (e = cudaMalloc(&drp, 8 * (size_t)(m + 1))) || (e = cudaMalloc(&doc, 4 * k)) ||
      (e = cudaMalloc(&dov, 8 * k)))
    return done(cuda_fail(e, "cudaMalloc(coo)"));
  if (count > 0 && ((e = cudaMemcpy(dr, h_rows, 8 * count, cudaMemcpyHostToDevice)) ||
                    (e = cudaMemcpy(dc, h_cols, 8 * count, cudaMemcpyHostToDevice)) ||
                    (e = cudaMemcpy(dv, h_vals, 8 * count, cudaMemcpyHostToDevice))))
    return done(cuda_fail(e, "cudaMemcpy(coo)"));
  int rc = csr5g_coo_to_csr(device, m, n, count, dr, dc, dv, drp, doc, dov, nnz, nullptr);
  if (rc) return done(rc);
  std::vector<int32_t> cols((size_t)*nnz);
  if ((e = cudaMemcpy(h_row_ptr, drp, 8 * (size_t)(m + 1), cudaMemcpyDeviceToHost)) ||
      (*nnz && ((e = cudaMemcpy(cols.data(), doc, 4 * (size_t)*nnz, cudaMemcpyDeviceToHost)) ||
                (e = cudaMemcpy(h_val, dov, 8 * (size_t)*nnz, cudaMemcpyDeviceToHost)))))
    return done(cuda_fail(e, "cudaMemcpy(csr)"));
  for (size_t q = 0; q < cols.size(); ++q) h_col_idx[q] = cols[q];
  return done(CSR5G_OK);
}

}  // extern "C"
