// synth_graph.cu -- irregular synthetic matrices on the device (BASELINE
// configs 3-5).  Counter-based hashing (splitmix64 keyed by index), so a given
// (kind, size, seed) is the same matrix on every GPU and every run.
//
//  R-MAT (Chakrabarti et al.; Graph500 parameters a,b,c,d = .57,.19,.19,.05):
//    edge e picks one quadrant per level from a 16-bit draw; vertex ids are
//    optionally relabelled by a keyed bijection on `scale` bits (Graph500
//    permutes vertices); (row, col) keys are radix-sorted and de-duplicated
//    (CUB), values U[0.5, 1.5).  Rows are cut into blocks of at most 2^28 raw
//    edges (a histogram pass); a block's entries are regenerated from the
//    edge counter whenever needed (all edges generated, the block's rows
//    kept, sorted, de-duplicated), so the whole edge list never sits in
//    memory (R-MAT s27: 2^31 edges) and a rank can fill just its slice of
//    entries (csr5g_gen_fill_range).
//  Mixed skew: m = n = 2^k, each row empty with
//    probability p_empty, `n_long` rows of exactly `long_len` nonzeros at
//    evenly spaced columns (synthetic.cpp:50-52), the others U[min_len,
//    max_len] distinct random columns (one per equal-width stratum, so
//    sorted and distinct by construction), values U[0.5, 1.5).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <new>
#include <vector>

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

// One R-MAT edge: `scale` quadrant choices from 16-bit draws, then the
// optional keyed relabelling of both endpoints.
__device__ __forceinline__ void rmat_edge(uint64_t e, int scale, uint64_t seed, int permute,
                                          uint64_t& u, uint64_t& v) {
  // Graph500 thresholds on 16-bit draws: a=.57, a+b=.76, a+b+c=.95
  const uint32_t ta = 37355, tab = 49807, tabc = 62259;
  uint64_t h = 0;
  u = v = 0;
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
}

constexpr int kHistBins = 1024;

// edges per row bin (row >> shift), to cut the rows into blocks of bounded
// edge count
__global__ void k_rmat_hist(uint64_t E, int scale, uint64_t seed, int permute, int shift,
                            unsigned long long* __restrict__ hist) {
  __shared__ unsigned int sh[kHistBins];
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += stride) {
    uint64_t u, v;
    rmat_edge(e, scale, seed, permute, u, v);
    atomicAdd(&sh[u >> shift], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, (unsigned long long)sh[i]);
}

// the (row << 32 | col) keys of the edges whose row lies in [row_lo, row_hi),
// compacted in arbitrary order (sorted afterwards)
__global__ void k_rmat_select(uint64_t E, int scale, uint64_t seed, int permute, uint64_t row_lo,
                              uint64_t row_hi, uint64_t* __restrict__ out,
                              unsigned long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < E; base += stride) {
    const uint64_t e = base + threadIdx.x;
    uint64_t u = 0, v = 0;
    bool take = false;
    if (e < E) {
      rmat_edge(e, scale, seed, permute, u, v);
      take = u >= row_lo && u < row_hi;
    }
    const uint32_t mask = __ballot_sync(kFull, take);
    if (!mask) continue;
    const int leader = __ffs(mask) - 1;
    unsigned long long b = 0;
    if (lane == leader) b = atomicAdd(cnt, (unsigned long long)__popc(mask));
    b = __shfl_sync(kFull, b, leader);
    if (take) out[b + __popc(mask & ((1u << lane) - 1))] = (u << 32) | v;
  }
}

// row_ptr[r] = base + (first key index with row >= r), r in [row_lo, row_hi)
__global__ void k_keys_row_ptr(const uint64_t* __restrict__ keys, int64_t nk, int64_t row_lo,
                               int64_t row_hi, int64_t base, int64_t* __restrict__ row_ptr) {
  const int64_t r = row_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= row_hi) return;
  const uint64_t target = (uint64_t)r << 32;
  int64_t lo = 0, hi = nk;
  while (lo < hi) {
    const int64_t mid = lo + ((hi - lo) >> 1);
    if (keys[mid] < target)
      lo = mid + 1;
    else
      hi = mid;
  }
  row_ptr[r] = base + lo;
}

// entries of a block (its sorted unique keys, global positions base + i) that
// fall in [lo, hi), written at position - lo
__global__ void k_keys_fill(const uint64_t* __restrict__ keys, int64_t nk, int64_t base, int64_t lo,
                            int64_t hi, uint64_t seed, int32_t* __restrict__ col,
                            double* __restrict__ val) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nk) return;
  const int64_t pos = base + i;
  if (pos < lo || pos >= hi) return;
  const uint64_t k = keys[i];
  col[pos - lo] = (int32_t)(k & 0xffffffffu);
  val[pos - lo] = 0.5 + unit(splitmix(seed * 0x51ED27 + k));
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

__global__ void k_mixed_fill_short(MixedSpec s, const int64_t* __restrict__ rp, int64_t lo,
                                   int64_t hi, int32_t* __restrict__ col, double* __restrict__ val) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= s.m || mixed_long_row(s, r) >= 0) return;
  const int64_t b = rp[r], l = rp[r + 1] - b;
  if (b + l <= lo || b >= hi) return;
  for (int64_t j = 0; j < l; ++j) {
    const int64_t q = b + j;
    if (q < lo || q >= hi) continue;
    const int64_t c0 = j * s.n / l, c1 = (j + 1) * s.n / l;
    const uint64_t h = splitmix(s.seed * 0x9E37 + splitmix((uint64_t)r * 64 + (uint64_t)j));
    col[q - lo] = (int32_t)(c0 + (int64_t)(h % (uint64_t)(c1 - c0)));
    val[q - lo] = 0.5 + unit(splitmix(h));
  }
}

__global__ void k_mixed_fill_long(MixedSpec s, const int64_t* __restrict__ rp, int64_t lo,
                                  int64_t hi, int32_t* __restrict__ col, double* __restrict__ val) {
  const int k = blockIdx.y;
  const int64_t r = (int64_t)(k + 1) * s.m / (s.n_long + 1);
  const int64_t b = rp[r], l = s.long_len;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < l;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = b + j;
    if (q < lo || q >= hi) continue;
    col[q - lo] = (int32_t)(j * s.n / l);
    val[q - lo] = 0.5 + unit(splitmix(s.seed * 0x2545F + splitmix((uint64_t)r * 0x100000 + j)));
  }
}

}  // namespace
}  // namespace csr5g

using namespace csr5g;

struct csr5g_gen_s {
  int kind = 0;  // 0 = R-MAT, 1 = mixed
  int64_t m = 0, n = 0, nnz = 0;
  uint64_t seed = 0;
  // R-MAT: rows are cut into blocks of bounded edge count; a block's entries
  // are its edges' sorted unique keys, regenerated whenever they are needed
  int scale = 0, permute = 0;
  uint64_t E = 0;
  int64_t* row_ptr = nullptr;       // device, m + 1 (deduplicated)
  std::vector<int64_t> blk_row;     // block b holds rows [blk_row[b], blk_row[b+1])
  std::vector<int64_t> blk_pos;     // ... and global positions [blk_pos[b], blk_pos[b+1])
  uint64_t blk_cap = 0;             // most raw edges in one block
  int64_t* len = nullptr;           // mixed: row lengths
  MixedSpec spec{};
};

namespace {

// Raw edges per block: large enough that few passes are needed, small enough
// that the key buffers (2 x 8 B per edge + sort scratch) stay a few GB.
// CSR5G_GEN_BLOCK_EDGES overrides it (tests force many blocks on small graphs).
uint64_t block_edges() {
  static const uint64_t v = [] {
    const char* e = std::getenv("CSR5G_GEN_BLOCK_EDGES");
    return e ? std::max<uint64_t>(1, std::strtoull(e, nullptr, 10)) : uint64_t(1) << 28;
  }();
  return v;
}

// Scratch of one block pass: two key arrays (sort ping-pong) and the CUB
// temporary storage, sized for the largest block.
struct KeyScratch {
  uint64_t* k0 = nullptr;
  uint64_t* k1 = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  unsigned long long* cnt = nullptr;  // [0] selected edges, [1] unique keys
  ~KeyScratch() {
    cudaFree(k0);
    cudaFree(k1);
    cudaFree(tmp);
    cudaFree(cnt);
  }
  int init(uint64_t cap, int scale, cudaStream_t stream) {
    CSR5G_CUDA(cudaMalloc(&k0, std::max<uint64_t>(cap, 1) * 8));
    CSR5G_CUDA(cudaMalloc(&k1, std::max<uint64_t>(cap, 1) * 8));
    CSR5G_CUDA(cudaMalloc(&cnt, 2 * sizeof(unsigned long long)));
    size_t sb = 0, ub = 0;
    CSR5G_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, sb, k0, k1, (int64_t)cap, 0, 32 + scale,
                                              stream));
    CSR5G_CUDA(cub::DeviceSelect::Unique(nullptr, ub, k1, k0,
                                         reinterpret_cast<int64_t*>(cnt + 1), (int64_t)cap, stream));
    tmp_bytes = std::max(sb, ub);
    CSR5G_CUDA(cudaMalloc(&tmp, tmp_bytes));
    return CSR5G_OK;
  }
};

unsigned grid_for(int device_sms, uint64_t work) {
  const uint64_t want = (work + 255) / 256;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)device_sms * 16));
}

// Block b's sorted unique keys into s.k0; returns their count.
int rmat_block_keys(const csr5g_gen_s* g, size_t b, KeyScratch& s, int sms, cudaStream_t stream,
                    int64_t* nk) {
  CSR5G_CUDA(cudaMemsetAsync(s.cnt, 0, 2 * sizeof(unsigned long long), stream));
  k_rmat_select<<<grid_for(sms, g->E), 256, 0, stream>>>(
      g->E, g->scale, g->seed, g->permute, (uint64_t)g->blk_row[b], (uint64_t)g->blk_row[b + 1],
      s.k0, s.cnt);
  CSR5G_CUDA(cudaGetLastError());
  unsigned long long sel = 0;
  CSR5G_CUDA(cudaMemcpyAsync(&sel, s.cnt, sizeof sel, cudaMemcpyDeviceToHost, stream));
  CSR5G_CUDA(cudaStreamSynchronize(stream));
  size_t sb = s.tmp_bytes;
  CSR5G_CUDA(cub::DeviceRadixSort::SortKeys(s.tmp, sb, s.k0, s.k1, (int64_t)sel, 0, 32 + g->scale,
                                            stream));
  size_t ub = s.tmp_bytes;
  CSR5G_CUDA(cub::DeviceSelect::Unique(s.tmp, ub, s.k1, s.k0, reinterpret_cast<int64_t*>(s.cnt + 1),
                                       (int64_t)sel, stream));
  unsigned long long u = 0;
  CSR5G_CUDA(cudaMemcpyAsync(&u, s.cnt + 1, sizeof u, cudaMemcpyDeviceToHost, stream));
  CSR5G_CUDA(cudaStreamSynchronize(stream));
  *nk = (int64_t)u;
  return CSR5G_OK;
}

int sm_count(int* sms) {
  int dev = 0;
  CSR5G_CUDA(cudaGetDevice(&dev));
  CSR5G_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
  return CSR5G_OK;
}

// R-MAT entries at global positions [lo, hi) (and, if asked, the row_ptr)
int rmat_fill(const csr5g_gen_s* g, int64_t lo, int64_t hi, int64_t* d_row_ptr, int32_t* d_col,
              double* d_val, cudaStream_t stream) {
  if (d_row_ptr)
    CSR5G_CUDA(cudaMemcpyAsync(d_row_ptr, g->row_ptr, sizeof(int64_t) * (g->m + 1),
                               cudaMemcpyDeviceToDevice, stream));
  if (hi <= lo) return CSR5G_OK;
  int sms = 0;
  if (int rc = sm_count(&sms)) return rc;
  KeyScratch s;
  if (int rc = s.init(g->blk_cap, g->scale, stream)) return rc;
  for (size_t b = 0; b + 1 < g->blk_row.size(); ++b) {
    const int64_t p0 = g->blk_pos[b], p1 = g->blk_pos[b + 1];
    if (p1 <= lo || p0 >= hi || p1 == p0) continue;
    int64_t nk = 0;
    if (int rc = rmat_block_keys(g, b, s, sms, stream, &nk)) return rc;
    if (nk != p1 - p0) return fail(CSR5G_ERUNTIME, "csr5g: R-MAT block regenerated differently");
    k_keys_fill<<<(unsigned)((nk + 255) / 256), 256, 0, stream>>>(s.k0, nk, p0, lo, hi, g->seed,
                                                                  d_col, d_val);
    CSR5G_CUDA(cudaGetLastError());
  }
  CSR5G_CUDA(cudaStreamSynchronize(stream));  // the scratch is freed on return
  return CSR5G_OK;
}

int mixed_fill(const csr5g_gen_s* g, int64_t lo, int64_t hi, int64_t* d_row_ptr, int32_t* d_col,
               double* d_val, cudaStream_t stream) {
  int64_t* rp = d_row_ptr;
  if (!rp) CSR5G_CUDA(cudaMallocAsync(&rp, sizeof(int64_t) * (g->m + 1), stream));
  void* tmp = nullptr;
  size_t tb = 0;
  cudaError_t e = cudaMemsetAsync(rp, 0, sizeof(int64_t), stream);
  if (e == cudaSuccess) e = cub::DeviceScan::InclusiveSum(nullptr, tb, g->len, rp + 1, g->m, stream);
  if (e == cudaSuccess) e = cudaMallocAsync(&tmp, tb, stream);
  if (e == cudaSuccess) e = cub::DeviceScan::InclusiveSum(tmp, tb, g->len, rp + 1, g->m, stream);
  if (tmp) cudaFreeAsync(tmp, stream);
  if (e == cudaSuccess && hi > lo) {
    k_mixed_fill_short<<<(unsigned)((g->m + 255) / 256), 256, 0, stream>>>(g->spec, rp, lo, hi,
                                                                            d_col, d_val);
    if (g->spec.n_long > 0)
      k_mixed_fill_long<<<dim3(64, g->spec.n_long), 256, 0, stream>>>(g->spec, rp, lo, hi, d_col,
                                                                      d_val);
    e = cudaGetLastError();
  }
  if (!d_row_ptr) cudaFreeAsync(rp, stream);
  if (e != cudaSuccess) return cuda_fail(e, "mixed fill");
  return CSR5G_OK;
}

}  // namespace

extern "C" {

int csr5g_rmat_create(int32_t scale, int32_t edge_factor, uint64_t seed, int32_t permute,
                      void* stream_v, csr5g_gen* out, int64_t* m, int64_t* nnz) {
  if (scale < 1 || scale > 30 || edge_factor < 1 || !out || !m || !nnz)
    return fail(CSR5G_EINVAL, "csr5g: R-MAT needs 1 <= scale <= 30 and edge_factor >= 1");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  auto* g = new (std::nothrow) csr5g_gen_s();
  if (!g) return fail(CSR5G_ENOMEM, "csr5g: host allocation failed");
  g->kind = 0;
  g->m = g->n = int64_t(1) << scale;
  g->seed = seed;
  g->scale = scale;
  g->permute = permute;
  g->E = (uint64_t)edge_factor << scale;
  auto bail = [&](int rc) {
    csr5g_gen_release(g);
    return rc;
  };
  int sms = 0;
  if (int rc = sm_count(&sms)) return bail(rc);
  // 1. raw edges per row bin -> row blocks of at most max(block_edges(), one bin) edges
  const int bins_log = std::min(scale, 10);
  const int shift = scale - bins_log;
  const int bins = 1 << bins_log;
  unsigned long long* d_hist = nullptr;
  cudaError_t e = cudaMalloc(&d_hist, sizeof(unsigned long long) * kHistBins);
  if (e != cudaSuccess) return bail(cuda_fail(e, "cudaMalloc(hist)"));
  std::vector<unsigned long long> hist(kHistBins);
  e = cudaMemsetAsync(d_hist, 0, sizeof(unsigned long long) * kHistBins, stream);
  if (e == cudaSuccess) {
    k_rmat_hist<<<grid_for(sms, g->E), 256, 0, stream>>>(g->E, scale, seed, permute, shift, d_hist);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(hist.data(), d_hist, sizeof(unsigned long long) * kHistBins,
                        cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  cudaFree(d_hist);
  if (e != cudaSuccess) return bail(cuda_fail(e, "R-MAT histogram"));
  g->blk_row.push_back(0);
  uint64_t acc = 0;
  for (int b = 0; b < bins; ++b) {
    if (acc > 0 && acc + hist[b] > block_edges()) {
      g->blk_row.push_back((int64_t)b << shift);
      g->blk_cap = std::max<uint64_t>(g->blk_cap, acc);
      acc = 0;
    }
    acc += hist[b];
  }
  g->blk_row.push_back(g->m);
  g->blk_cap = std::max<uint64_t>(g->blk_cap, acc);
  // 2. per block: sorted unique keys -> its rows of the global row_ptr
  if ((e = cudaMalloc(&g->row_ptr, sizeof(int64_t) * (g->m + 1))) != cudaSuccess)
    return bail(cuda_fail(e, "cudaMalloc(row_ptr)"));
  {
    KeyScratch s;
    if (int rc = s.init(g->blk_cap, scale, stream)) return bail(rc);
    int64_t base = 0;
    g->blk_pos.push_back(0);
    for (size_t b = 0; b + 1 < g->blk_row.size(); ++b) {
      int64_t nk = 0;
      if (int rc = rmat_block_keys(g, b, s, sms, stream, &nk)) return bail(rc);
      const int64_t r0 = g->blk_row[b], r1 = g->blk_row[b + 1];
      k_keys_row_ptr<<<(unsigned)((r1 - r0 + 255) / 256), 256, 0, stream>>>(s.k0, nk, r0, r1, base,
                                                                            g->row_ptr);
      if ((e = cudaGetLastError()) != cudaSuccess) return bail(cuda_fail(e, "k_keys_row_ptr"));
      base += nk;
      g->blk_pos.push_back(base);
    }
    g->nnz = base;
    if ((e = cudaMemcpyAsync(g->row_ptr + g->m, &g->nnz, sizeof(int64_t), cudaMemcpyHostToDevice,
                             stream)) != cudaSuccess ||
        (e = cudaStreamSynchronize(stream)) != cudaSuccess)
      return bail(cuda_fail(e, "R-MAT row_ptr"));
  }
  *out = g;
  *m = g->m;
  *nnz = g->nnz;
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

int csr5g_gen_fill_range(csr5g_gen g, int64_t pos_begin, int64_t pos_end, int64_t* d_row_ptr,
                         int32_t* d_col_idx, double* d_val, void* stream_v) {
  if (!g) return fail(CSR5G_EINVAL, "csr5g: NULL generator");
  if (pos_begin < 0 || pos_end < pos_begin || pos_end > g->nnz)
    return fail(CSR5G_EINVAL, "csr5g: entry range outside [0, nnz]");
  if (pos_end > pos_begin && (!d_col_idx || !d_val))
    return fail(CSR5G_EINVAL, "csr5g: col_idx/val is NULL");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  if (g->kind == 0) return rmat_fill(g, pos_begin, pos_end, d_row_ptr, d_col_idx, d_val, stream);
  return mixed_fill(g, pos_begin, pos_end, d_row_ptr, d_col_idx, d_val, stream);
}

int csr5g_gen_fill(csr5g_gen g, int64_t* d_row_ptr, int32_t* d_col_idx, double* d_val,
                   void* stream_v) {
  if (!g) return fail(CSR5G_EINVAL, "csr5g: NULL generator");
  if (!d_row_ptr) return fail(CSR5G_EINVAL, "csr5g: row_ptr is NULL");
  return csr5g_gen_fill_range(g, 0, g->nnz, d_row_ptr, d_col_idx, d_val, stream_v);
}

int csr5g_gen_release(csr5g_gen g) {
  if (!g) return CSR5G_OK;
  cudaFree(g->row_ptr);
  cudaFree(g->len);
  delete g;
  return CSR5G_OK;
}

}  // extern "C"
