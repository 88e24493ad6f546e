// hotx.cu -- hot-column x staging for random-gather plans whose x exceeds L2.
//
// A power-law matrix (R-MAT, Graph500 parameters) sends most of its gathers to
// few columns: at scale 27 the 6% of columns with the most entries take ~90%
// of them.  With vertices permuted those columns are scattered over x, so a
// 32-byte L2 sector holding one hot x value also holds three cold ones and the
// L2 keeps a quarter of what it could; cold gathers (evict-last like the rest)
// push the hot lines out as well.  When x does not fit the L2, the build
//   1. counts entries per column over a sample of the transposed col_idx,
//   2. picks the hot set: the columns whose sampled count reaches the
//      smallest threshold that keeps the set within a byte budget
//      (CSR5G_HOT_MB, 64 MB: half the L2),
//   3. numbers the hot columns by descending sampled count (hottest first, so
//      the most gathered values share the fewest lines) and writes an
//      execution copy of col_idx (the exported CSR5 col_idx is untouched) in
//      which a hot column c becomes ~rank(c) (negative) and a cold one keeps c.
// Every SpMV first stages xh[r] = x[hot[r]] (k_xhot_fill: a coalesced list
// read, one gather per hot column, stores that stay in L2 with evict-last), then the
// tile kernel gathers hot entries from the dense xh (evict-last) and cold
// ones from x with evict-first, so cold lines no longer displace hot ones.
// The products use the same x values in the same order: y is bit-identical
// to the unstaged kernel's.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

namespace csr5g {
namespace {

constexpr int kHotBins = 1024;  // sampled counts >= kHotBins - 1 share the top bin

__global__ void k_hot_count(const int32_t* __restrict__ col, int64_t len, int stride,
                            uint32_t* __restrict__ cnt) {
  const int64_t step = (int64_t)gridDim.x * blockDim.x * stride;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * stride; i < len; i += step)
    atomicAdd(cnt + __ldg(col + i), 1u);
}

__global__ void k_hot_hist(const uint32_t* __restrict__ cnt, int64_t n,
                           unsigned long long* __restrict__ hist) {
  __shared__ unsigned int hs[kHotBins];
  for (int b = threadIdx.x; b < kHotBins; b += blockDim.x) hs[b] = 0;
  __syncthreads();
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n; c += step)
    atomicAdd(hs + min(cnt[c], (uint32_t)(kHotBins - 1)), 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < kHotBins; b += blockDim.x)
    if (hs[b]) atomicAdd(hist + b, (unsigned long long)hs[b]);
}

// one thread per column: the hot bitmap word of each 32 columns and its count
__global__ void k_hot_bits(const uint32_t* __restrict__ cnt, int64_t n, uint32_t thr,
                           uint32_t* __restrict__ bm, int32_t* __restrict__ wc) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t cw = c & ~int64_t(31);
  if (cw >= n) return;
  const bool hot = c < n && cnt[c] >= thr;
  const uint32_t word = __ballot_sync(kFull, hot);
  if ((threadIdx.x & 31) == 0) {
    bm[c >> 5] = word;
    wc[c >> 5] = __popc(word);
  }
}

__global__ void k_hot_list(const uint32_t* __restrict__ bm, const int32_t* __restrict__ wpre,
                           int64_t n, int32_t* __restrict__ hot) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const uint32_t w = bm[c >> 5];
  const int b = (int)(c & 31);
  if ((w >> b) & 1u) hot[wpre[c >> 5] + __popc(w & ((1u << b) - 1u))] = (int32_t)c;
}

// ordering by sampled count: key = count of hot column a (ascending rank),
// value = a; after a stable descending sort, perm[a] = final rank and
// hot_sorted[r] = column
__global__ void k_hot_keys(const int32_t* __restrict__ hot, const uint32_t* __restrict__ cnt,
                           int64_t H, uint32_t* __restrict__ key, int32_t* __restrict__ idx) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= H) return;
  key[a] = cnt[hot[a]];
  idx[a] = (int32_t)a;
}

__global__ void k_hot_perm(const int32_t* __restrict__ order, const int32_t* __restrict__ hot, int64_t H,
                           int32_t* __restrict__ perm, int32_t* __restrict__ hot_sorted) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= H) return;
  const int32_t a = order[r];
  perm[a] = (int32_t)r;
  hot_sorted[r] = hot[a];
}

// (bitmap word, prefix) of each 32 columns in one 8-byte entry: the column
// lookup below is one random L2 read instead of two
__global__ void k_hot_pack(const uint32_t* __restrict__ bm, const int32_t* __restrict__ wpre,
                           int64_t nwords, uint2* __restrict__ pk) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w < nwords) pk[w] = make_uint2(bm[w], (uint32_t)wpre[w]);
}

__device__ __forceinline__ int32_t exec_col(int32_t c, const uint2* __restrict__ pk,
                                            const int32_t* __restrict__ perm) {
  const uint2 e = __ldg(pk + (c >> 5));
  const int b = c & 31;
  if (!((e.x >> b) & 1u)) return c;
  const int32_t a = (int32_t)e.y + __popc(e.x & ((1u << b) - 1u));
  return ~(perm ? __ldg(perm + a) : a);
}

// the execution col_idx of the complete tiles (len is a multiple of 32)
__global__ void k_col_exec(const int4* __restrict__ col, int64_t len4, const uint2* __restrict__ pk,
                           const int32_t* __restrict__ perm, int4* __restrict__ out) {
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len4; i += step) {
    int4 v = col[i];
    v.x = exec_col(v.x, pk, perm);
    v.y = exec_col(v.y, pk, perm);
    v.z = exec_col(v.z, pk, perm);
    v.w = exec_col(v.w, pk, perm);
    out[i] = v;
  }
}

__global__ void k_xhot_fill(const double* __restrict__ x, const int32_t* __restrict__ hot, int64_t H,
                            double* __restrict__ xh) {
  // the tile kernel may launch now: it waits for this grid before it reads xh
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t pol = policy_evict_last();
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < H; i += step)
    st_hint(xh + i, __ldg(x + __ldg(hot + i)), pol);
}

int64_t env_i64(const char* name, int64_t dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoll(e) : dflt;
}

}  // namespace

// Decides and builds the staging (h->vr plans only; CSR5G_HOT = 0 off, 1 on
// whatever x's size, unset: on when 8n exceeds 3/4 of the L2 and the hot set
// takes >= 30% of the sampled gathers).  Out of memory for the execution copy
// is not an error: the handle keeps the plain gathers.
int build_hot_plan(Handle* h, cudaStream_t stream, int64_t* bytes) {
  h->col_x = h->col;
  h->n_hot = 0;
  h->cold_pol = (int)env_i64("CSR5G_HOT_COLD_POL", 0);

  const int64_t mode = env_i64("CSR5G_HOT", -1);
  const int64_t n = h->info.n;
  const int64_t tiled = h->pcs * h->B;
  if (mode == 0 || !h->vr || tiled == 0 || n == 0) return CSR5G_OK;
  int l2 = 0, sms = 0;
  CSR5G_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->device));
  CSR5G_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
  if (mode < 0 && (double)n * 8.0 <= 0.75 * (double)l2) return CSR5G_OK;
  // hottest first and L1-allocated hot gathers (GM 3), for x several times
  // the L2 (R-MAT s27) and around it (R-MAT s24: 1.22 ms against 1.45 for
  // ascending order without L1 at 16 warps, profiles/r02_hot_sweep.txt r02ap)
  h->hot_l1 = (int)env_i64("CSR5G_HOT_L1", 1);
  const int64_t hmax = env_i64("CSR5G_HOT_COLS", env_i64("CSR5G_HOT_MB", 64) * (1 << 20) / 8);
  // sample: about 2^27 entries, every stride-th, stride at most 8 (R-MAT s24:
  // 2, build 5.9 -> 5.1 ms at the same SpMV time; s27: 8 -- 16 left the hot
  // set 21% smaller, profiles/r02_hot_sweep.txt)
  const int stride = (int)std::max<int64_t>(
      1, env_i64("CSR5G_HOT_STRIDE",
                 std::min<int64_t>(8, (tiled + (int64_t(1) << 27) - 1) >> 27)));
  const bool by_count = env_i64("CSR5G_HOT_ORDER", 1) != 0;

  uint32_t* cnt = nullptr;
  unsigned long long* hist = nullptr;
  uint32_t* bm = nullptr;
  int32_t *wc = nullptr, *wpre = nullptr, *hot = nullptr, *colx = nullptr;
  double* xh = nullptr;
  void* cub_tmp = nullptr;
  uint32_t *key = nullptr, *key2 = nullptr;  // count-order sort temporaries
  uint2* pk = nullptr;
  int32_t *idx = nullptr, *order = nullptr, *sorted = nullptr, *perm = nullptr;
  void* st = nullptr;
  const int64_t nwords = (n + 31) / 32;
  // keep = true: the staging survives (hot, colx, xh); every temporary goes
  auto release = [&](bool keep) {
    for (void* p : {(void*)cnt, (void*)hist, (void*)bm, (void*)wc, (void*)wpre, cub_tmp, (void*)pk,
                    (void*)key, (void*)key2, (void*)idx, (void*)order, (void*)perm, st})
      if (p) cudaFreeAsync(p, stream);
    cnt = nullptr, hist = nullptr, bm = nullptr, wc = wpre = nullptr, cub_tmp = nullptr, pk = nullptr;
    key = key2 = nullptr, idx = order = perm = nullptr, st = nullptr;
    if (!keep) {
      for (void* p : {(void*)hot, (void*)colx, (void*)xh, (void*)sorted})
        if (p) cudaFreeAsync(p, stream);
      hot = colx = sorted = nullptr, xh = nullptr;
    }
  };
  // a CUDA failure after the first allocation frees everything before it returns
#define HTRY(call)                                   \
  do {                                               \
    const cudaError_t e_ = (call);                   \
    if (e_ != cudaSuccess) {                         \
      release(false);                                \
      return cuda_fail(e_, #call);                   \
    }                                                \
  } while (0)
  auto alloc = [&](auto** p, size_t nb) {
    const cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(nb, 16), stream);
    if (e != cudaSuccess) cudaGetLastError();
    return e == cudaSuccess;
  };
  // (allocation failures: no staging, not an error)
  if (!alloc(&cnt, sizeof(uint32_t) * n) || !alloc(&hist, sizeof(unsigned long long) * kHotBins)) {
    release(false);
    return CSR5G_OK;
  }
  HTRY(cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * n, stream));
  HTRY(cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * kHotBins, stream));
  k_hot_count<<<sms * 8, 256, 0, stream>>>(h->col, tiled, stride, cnt);
  HTRY(cudaGetLastError());
  k_hot_hist<<<sms * 4, 256, 0, stream>>>(cnt, n, hist);
  HTRY(cudaGetLastError());
  std::vector<unsigned long long> hh(kHotBins);
  HTRY(cudaMemcpyAsync(hh.data(), hist, sizeof(unsigned long long) * kHotBins,
                             cudaMemcpyDeviceToHost, stream));
  HTRY(cudaStreamSynchronize(stream));
  // threshold: the smallest sampled count whose columns fit the budget
  std::vector<double> cols(kHotBins + 1, 0.0), mass(kHotBins + 1, 0.0);
  for (int b = kHotBins - 1; b >= 0; --b) {
    cols[b] = cols[b + 1] + (double)hh[b];
    mass[b] = mass[b + 1] + (double)b * (double)hh[b];
  }
  int thr = 1;
  while (thr < kHotBins - 1 && cols[thr] > (double)hmax) ++thr;
  const int64_t H = (int64_t)cols[thr];
  const double coverage = mass[1] > 0 ? mass[thr] / mass[1] : 0.0;
  if (H == 0 || H > 2 * hmax || (mode < 0 && coverage < 0.3)) {
    release(false);
    return CSR5G_OK;
  }
  size_t cub_bytes = 0;
  HTRY(cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int32_t*)nullptr, (int32_t*)nullptr,
                                           (int)nwords, stream));
  if (!alloc(&bm, sizeof(uint32_t) * nwords) || !alloc(&wc, sizeof(int32_t) * nwords) ||
      !alloc(&wpre, sizeof(int32_t) * nwords) || !alloc(&cub_tmp, cub_bytes) ||
      !alloc(&pk, sizeof(uint2) * nwords) ||
      !alloc(&hot, sizeof(int32_t) * H) || !alloc(&colx, sizeof(int32_t) * h->info.nnz_held) ||
      !alloc(&xh, sizeof(double) * H)) {
    release(false);
    return CSR5G_OK;
  }
  const unsigned cb = (unsigned)((nwords * 32 + 255) / 256);
  k_hot_bits<<<cb, 256, 0, stream>>>(cnt, n, (uint32_t)thr, bm, wc);
  HTRY(cudaGetLastError());
  HTRY(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, wc, wpre, (int)nwords, stream));
  k_hot_list<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(bm, wpre, n, hot);
  HTRY(cudaGetLastError());
  // hottest first (stable: equal counts keep column order), so the most
  // gathered values share the fewest lines
  if (by_count) {
    size_t sb = 0;
    HTRY(cub::DeviceRadixSort::SortPairsDescending(nullptr, sb, key, key2, idx, order, (int)H,
                                                         0, 32, stream));
    if (!alloc(&key, 4 * H) || !alloc(&key2, 4 * H) || !alloc(&idx, 4 * H) ||
        !alloc(&order, 4 * H) || !alloc(&sorted, 4 * H) || !alloc(&perm, 4 * H) || !alloc(&st, sb)) {
      release(false);
      return CSR5G_OK;
    }
    const unsigned hb = (unsigned)((H + 255) / 256);
    k_hot_keys<<<hb, 256, 0, stream>>>(hot, cnt, H, key, idx);
    HTRY(cudaGetLastError());
    HTRY(cub::DeviceRadixSort::SortPairsDescending(st, sb, key, key2, idx, order, (int)H, 0, 32,
                                                         stream));
    k_hot_perm<<<hb, 256, 0, stream>>>(order, hot, H, perm, sorted);
    HTRY(cudaGetLastError());
    int32_t* ascending = hot;
    hot = sorted;
    sorted = nullptr;
    HTRY(cudaFreeAsync(ascending, stream));
  }
  k_hot_pack<<<(unsigned)((nwords + 255) / 256), 256, 0, stream>>>(bm, wpre, nwords, pk);
  HTRY(cudaGetLastError());
  k_col_exec<<<sms * 8, 256, 0, stream>>>(reinterpret_cast<const int4*>(h->col), tiled / 4, pk, perm,
                                          reinterpret_cast<int4*>(colx));
  HTRY(cudaGetLastError());
  const int64_t rest = h->info.nnz_held - tiled;  // the CSR tail keeps its columns
  if (rest > 0)
    HTRY(cudaMemcpyAsync(colx + tiled, h->col + tiled, sizeof(int32_t) * rest,
                               cudaMemcpyDeviceToDevice, stream));
  release(true);
  h->col_x = colx;
  h->hot_cols = hot;
  h->xh = xh;
  h->n_hot = H;
  h->hot_coverage = coverage;
  h->hot_threshold = thr;
  *bytes += (int64_t)(sizeof(int32_t) * (H + h->info.nnz_held) + sizeof(double) * H);
  return CSR5G_OK;
#undef HTRY
}

int launch_xhot_fill(Handle* h, const double* d_x, double* d_xh, cudaStream_t stream) {
  if (h->n_hot == 0) return CSR5G_OK;
  int sms = h->info.num_sms > 0 ? h->info.num_sms : 148;
  const int64_t blocks = std::min<int64_t>((h->n_hot + 255) / 256, (int64_t)sms * 8);
  k_xhot_fill<<<(unsigned)blocks, 256, 0, stream>>>(d_x, h->hot_cols, h->n_hot, d_xh);
  CSR5G_CUDA(cudaGetLastError());
  return CSR5G_OK;
}

}  // namespace csr5g
