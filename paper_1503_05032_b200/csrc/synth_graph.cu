// synth_graph.cu -- irregular synthetic matrices on the device (BASELINE
// configs 3-5).  Counter-based hashing (splitmix64 keyed by index), so a given
// (kind, size, seed) is the same matrix on every GPU and every run.
//
//  R-MAT (Chakrabarti et al.; Graph500 parameters a,b,c,d = .57,.19,.19,.05):
//    edge e picks one quadrant per level from a 16-bit draw; vertex ids are
//    optionally relabelled by a keyed bijection on `scale` bits (Graph500
//    permutes vertices); (row, col) keys are radix-sorted and de-duplicated
//    (CUB), values U[0.5, 1.5).
//  Mixed skew: m = n = 2^k, each row empty with
//    probability p_empty, `n_long` rows of exactly `long_len` nonzeros at
//    evenly spaced columns (synthetic.cpp:50-52), the others U[min_len,
//    max_len] distinct random columns (one per equal-width stratum, so
//    sorted and distinct by construction), values U[0.5, 1.5).
#include <cub/cub.cuh>

#include <new>

#include "internal.cuh"

namespace csr5g {
namespace {

__host__ __device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ double unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

// keyed bijection on `bits`-bit integers (odd multiply mod 2^bits + xorshift)
__device__ __forceinline__ uint64_t permute_bits(uint64_t x, int bits, uint64_t key) {
  const uint64_t mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
  const int s1 = (bits + 1) / 2 > 0 ? (bits + 1) / 2 : 1;
  for (int r = 0; r < 3; ++r) {
    const uint64_t k = splitmix(key + r);
    x = (x * (k | 1ull) + (k >> 17)) & mask;
    x ^= x >> s1;
  }
  return x & mask;
}

__global__ void k_rmat_edges(uint64_t E, int scale, uint64_t seed, int permute,
                             uint64_t* __restrict__ keys) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  // Graph500 thresholds on 16-bit draws: a=.57, a+b=.76, a+b+c=.95
  const uint32_t ta = 37355, tab = 49807, tabc = 62259;
  uint64_t u = 0, v = 0, h = 0;
  for (int lvl = 0; lvl < scale; ++lvl) {
    if ((lvl & 3) == 0) h = splitmix(seed ^ splitmix(e * 7 + (uint64_t)(lvl >> 2)));
    const uint32_t r = (uint32_t)(h & 0xffff);
    h >>= 16;
    const uint32_t bu = r >= tab, bv = (r >= ta && r < tab) || r >= tabc;
    u = (u << 1) | bu;
    v = (v << 1) | bv;
  }
  if (permute) {
    u = permute_bits(u, scale, seed * 31 + 1);
    v = permute_bits(v, scale, seed * 31 + 1);
  }
  keys[e] = (u << 32) | v;
}

// row_ptr[r] = first key index with row >= r (r in [0, m])
__global__ void k_keys_row_ptr(const uint64_t* __restrict__ keys, int64_t nnz, int64_t m,
                               int64_t* __restrict__ row_ptr) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r > m) return;
  const uint64_t target = (uint64_t)r << 32;
  int64_t lo = 0, hi = nnz;
  while (lo < hi) {
    const int64_t mid = lo + ((hi - lo) >> 1);
    if (keys[mid] < target)
      lo = mid + 1;
    else
      hi = mid;
  }
  row_ptr[r] = lo;
}

__global__ void k_keys_fill(const uint64_t* __restrict__ keys, int64_t nnz, uint64_t seed,
                            int32_t* __restrict__ col, double* __restrict__ val) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  const uint64_t k = keys[i];
  col[i] = (int32_t)(k & 0xffffffffu);
  val[i] = 0.5 + unit(splitmix(seed * 0x51ED27 + k));
}

struct MixedSpec {
  int64_t m, n, long_len;
  int32_t n_long, min_len, max_len;
  double p_empty;
  uint64_t seed;
};

__device__ __forceinline__ int64_t mixed_long_row(const MixedSpec& s, int64_t r) {
  // long rows at (k+1) * m / (n_long+1); returns k or -1
  for (int k = 0; k < s.n_long; ++k)
    if (r == (int64_t)(k + 1) * s.m / (s.n_long + 1)) return k;
  return -1;
}

__global__ void k_mixed_len(MixedSpec s, int64_t* __restrict__ len) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= s.m) return;
  int64_t l;
  if (mixed_long_row(s, r) >= 0) {
    l = s.long_len;
  } else {
    const uint64_t h = splitmix(s.seed ^ splitmix((uint64_t)r));
    if (unit(h) < s.p_empty)
      l = 0;
    else
      l = s.min_len + (int64_t)(splitmix(h) % (uint64_t)(s.max_len - s.min_len + 1));
  }
  len[r] = l;
}

__global__ void k_mixed_fill_short(MixedSpec s, const int64_t* __restrict__ rp,
                                   int32_t* __restrict__ col, double* __restrict__ val) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= s.m || mixed_long_row(s, r) >= 0) return;
  const int64_t b = rp[r], l = rp[r + 1] - b;
  for (int64_t j = 0; j < l; ++j) {
    const int64_t lo = j * s.n / l, hi = (j + 1) * s.n / l;
    const uint64_t h = splitmix(s.seed * 0x9E37 + splitmix((uint64_t)r * 64 + (uint64_t)j));
    col[b + j] = (int32_t)(lo + (int64_t)(h % (uint64_t)(hi - lo)));
    val[b + j] = 0.5 + unit(splitmix(h));
  }
}

__global__ void k_mixed_fill_long(MixedSpec s, const int64_t* __restrict__ rp,
                                  int32_t* __restrict__ col, double* __restrict__ val) {
  const int k = blockIdx.y;
  const int64_t r = (int64_t)(k + 1) * s.m / (s.n_long + 1);
  const int64_t b = rp[r], l = s.long_len;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < l;
       j += (int64_t)gridDim.x * blockDim.x) {
    col[b + j] = (int32_t)(j * s.n / l);
    val[b + j] = 0.5 + unit(splitmix(s.seed * 0x2545F + splitmix((uint64_t)r * 0x100000 + j)));
  }
}

}  // namespace
}  // namespace csr5g

using namespace csr5g;

struct csr5g_gen_s {
  int kind = 0;  // 0 = keys (R-MAT), 1 = mixed
  int64_t m = 0, n = 0, nnz = 0;
  uint64_t seed = 0;
  uint64_t* keys = nullptr;  // R-MAT: sorted unique (row << 32 | col)
  int64_t* len = nullptr;    // mixed: row lengths
  MixedSpec spec{};
};

extern "C" {

int csr5g_rmat_create(int32_t scale, int32_t edge_factor, uint64_t seed, int32_t permute,
                      void* stream_v, csr5g_gen* out, int64_t* m, int64_t* nnz) {
  if (scale < 1 || scale > 30 || edge_factor < 1 || !out || !m || !nnz)
    return fail(CSR5G_EINVAL, "csr5g: R-MAT needs 1 <= scale <= 30 and edge_factor >= 1");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  const uint64_t E = (uint64_t)edge_factor << scale;
  auto* g = new (std::nothrow) csr5g_gen_s();
  if (!g) return fail(CSR5G_ENOMEM, "csr5g: host allocation failed");
  g->kind = 0;
  g->m = g->n = int64_t(1) << scale;
  g->seed = seed;
  uint64_t *k0 = nullptr, *k1 = nullptr;
  void* tmp = nullptr;
  int* nsel = nullptr;
  auto bail = [&](int rc) {
    cudaFree(k0);
    cudaFree(k1);
    cudaFree(tmp);
    cudaFree(nsel);
    if (g->keys) cudaFree(g->keys);
    delete g;
    return rc;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&k0, E * 8)) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(keys)"));
  if ((e = cudaMalloc(&k1, E * 8)) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(keys)"));
  if ((e = cudaMalloc(&nsel, sizeof(int64_t))) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc"));
  k_rmat_edges<<<(unsigned)((E + 255) / 256), 256, 0, stream>>>(E, scale, seed, permute, k0);
  if ((e = cudaGetLastError()) != cudaSuccess) return bail(cuda_fail(e, "k_rmat_edges"));
  size_t sb = 0, ub = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, sb, k0, k1, (int64_t)E, 0, 32 + scale, stream);
  cub::DeviceSelect::Unique(nullptr, ub, k1, k0, reinterpret_cast<int64_t*>(nsel), (int64_t)E, stream);
  if ((e = cudaMalloc(&tmp, std::max(sb, ub))) != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(tmp)"));
  if ((e = cub::DeviceRadixSort::SortKeys(tmp, sb, k0, k1, (int64_t)E, 0, 32 + scale, stream)) != cudaSuccess)
    return bail(cuda_fail(e, "SortKeys"));
  if ((e = cub::DeviceSelect::Unique(tmp, ub, k1, k0, reinterpret_cast<int64_t*>(nsel), (int64_t)E,
                                     stream)) != cudaSuccess)
    return bail(cuda_fail(e, "Unique"));
  int64_t cnt = 0;
  if ((e = cudaMemcpyAsync(&cnt, nsel, sizeof cnt, cudaMemcpyDeviceToHost, stream)) != cudaSuccess ||
      (e = cudaStreamSynchronize(stream)) != cudaSuccess)
    return bail(cuda_fail(e, "R-MAT count"));
  cudaFree(k1);
  k1 = nullptr;
  cudaFree(tmp);
  tmp = nullptr;
  cudaFree(nsel);
  nsel = nullptr;
  g->keys = k0;
  k0 = nullptr;
  g->nnz = cnt;
  *out = g;
  *m = g->m;
  *nnz = cnt;
  return CSR5G_OK;
}

int csr5g_mixed_create(int32_t log2_m, double p_empty, int32_t n_long, int64_t long_len,
                       int32_t min_len, int32_t max_len, uint64_t seed, void* stream_v,
                       csr5g_gen* out, int64_t* m, int64_t* nnz) {
  if (log2_m < 4 || log2_m > 30 || min_len < 1 || max_len < min_len || n_long < 0 || !out)
    return fail(CSR5G_EINVAL, "csr5g: bad mixed-matrix parameters");
  const int64_t mm = int64_t(1) << log2_m;
  if (long_len > mm || max_len > mm) return fail(CSR5G_EINVAL, "csr5g: rows longer than n");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  auto* g = new (std::nothrow) csr5g_gen_s();
  if (!g) return fail(CSR5G_ENOMEM, "csr5g: host allocation failed");
  g->kind = 1;
  g->m = g->n = mm;
  g->seed = seed;
  g->spec = MixedSpec{mm, mm, long_len, n_long, min_len, max_len, p_empty, seed};
  cudaError_t e = cudaMalloc(&g->len, sizeof(int64_t) * (mm + 1));
  if (e != cudaSuccess) {
    delete g;
    return cuda_fail(e, "cudaMalloc(len)");
  }
  k_mixed_len<<<(unsigned)((mm + 255) / 256), 256, 0, stream>>>(g->spec, g->len);
  int64_t* tot = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cub::DeviceReduce::Sum(nullptr, tb, g->len, tot, mm, stream);
  cudaMalloc(&tmp, tb);
  cudaMalloc(&tot, sizeof(int64_t));
  cub::DeviceReduce::Sum(tmp, tb, g->len, tot, mm, stream);
  int64_t cnt = 0;
  cudaMemcpyAsync(&cnt, tot, sizeof cnt, cudaMemcpyDeviceToHost, stream);
  e = cudaStreamSynchronize(stream);
  cudaFree(tmp);
  cudaFree(tot);
  if (e != cudaSuccess) {
    cudaFree(g->len);
    delete g;
    return cuda_fail(e, "mixed lengths");
  }
  g->nnz = cnt;
  *out = g;
  *m = mm;
  *nnz = cnt;
  return CSR5G_OK;
}

int csr5g_gen_fill(csr5g_gen g, int64_t* d_row_ptr, int32_t* d_col_idx, double* d_val,
                   void* stream_v) {
  if (!g) return fail(CSR5G_EINVAL, "csr5g: NULL generator");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  if (g->kind == 0) {
    k_keys_row_ptr<<<(unsigned)((g->m + 256) / 256), 256, 0, stream>>>(g->keys, g->nnz, g->m,
                                                                          d_row_ptr);
    k_keys_fill<<<(unsigned)((g->nnz + 255) / 256), 256, 0, stream>>>(g->keys, g->nnz, g->seed,
                                                                       d_col_idx, d_val);
  } else {
    void* tmp = nullptr;
    size_t tb = 0;
    CSR5G_CUDA(cudaMemsetAsync(d_row_ptr, 0, sizeof(int64_t), stream));
    cub::DeviceScan::InclusiveSum(nullptr, tb, g->len, d_row_ptr + 1, g->m, stream);
    CSR5G_CUDA(cudaMallocAsync(&tmp, tb, stream));
    CSR5G_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, g->len, d_row_ptr + 1, g->m, stream));
    CSR5G_CUDA(cudaFreeAsync(tmp, stream));
    k_mixed_fill_short<<<(unsigned)((g->m + 255) / 256), 256, 0, stream>>>(g->spec, d_row_ptr,
                                                                            d_col_idx, d_val);
    if (g->spec.n_long > 0)
      k_mixed_fill_long<<<dim3(64, g->spec.n_long), 256, 0, stream>>>(g->spec, d_row_ptr, d_col_idx,
                                                                      d_val);
  }
  CSR5G_CUDA(cudaGetLastError());
  return CSR5G_OK;
}

int csr5g_gen_release(csr5g_gen g) {
  if (!g) return CSR5G_OK;
  cudaFree(g->keys);
  cudaFree(g->len);
  delete g;
  return CSR5G_OK;
}

}  // extern "C"
