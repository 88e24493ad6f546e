// convert.cu -- CSR -> CSR5 on the device (reference: format.cpp:165-252).
//
// Five kernels, all bit-exact with the reference arrays:
//   k_rowscan        one pass over row_ptr: empty-row bitmap + head bitmap over
//                    nonzero positions (the row_ptr walk of format.cpp:93-97)
//   k_tile_ptr       thread per tile boundary: upper_bound + bounded empty-row
//                    check over the bitmap (format.cpp:52-82)
//   k_desc_transpose warp per tile, lane = column: popc / warp scan -> y_offset,
//                    ballot / ffs -> seg_offset, pack (format.cpp:84-121,
//                    descriptor.cpp:38-62); then the tile transpose of col/val
//                    through padded shared memory (format.cpp:226-249)
//   (CUB exclusive scan of per-tile head counts -> empty_offset_ptr)
//   k_eo             warp per flagged tile: row offsets of its heads
//                    (format.cpp:123-136, 213-224)
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <chrono>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <new>

#include "internal.cuh"

namespace csr5g {
namespace {

__global__ void k_rowscan(const int64_t* __restrict__ rp, int64_t m, int64_t pos_begin,
                          int64_t pos_end, uint32_t* __restrict__ empty_bits,
                          uint32_t* __restrict__ head_bits, csr5g_partial* __restrict__ send) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r == 0) *send = csr5g_partial{-1, 0.0};  // no boundary record yet
  const int lane = threadIdx.x & 31;
  const bool inr = r < m;
  int64_t lo = 0, hi = 0;
  if (inr) {
    lo = rp[r];
    hi = rp[r + 1];
  }
  const uint32_t em = __ballot_sync(kFull, inr && lo == hi);
  if (lane == 0 && r < m) empty_bits[r >> 5] = em;
  // Head bit at row_ptr[r]; rows are sorted, so lanes sharing a bitmap word
  // are contiguous: OR them together and issue one atomic per word group.
  const bool valid = inr && lo >= pos_begin && lo < pos_end;
  const int64_t local = lo - pos_begin;
  const int64_t word = valid ? (local >> 5) : (-1 - (int64_t)lane);
  uint32_t bits = valid ? (1u << (local & 31)) : 0u;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t ob = __shfl_down_sync(kFull, bits, d);
    const int64_t ow = __shfl_down_sync(kFull, word, d);
    if (lane + d < 32 && ow == word) bits |= ob;
  }
  const int64_t pw = __shfl_up_sync(kFull, word, 1);
  if (valid && (lane == 0 || pw != word)) atomicOr(&head_bits[word], bits);
}

// tile_ptr entries for global tiles [t_first, t_first + count).
__global__ void k_tile_ptr(const int64_t* __restrict__ rp, int64_t m, int64_t B, int64_t p,
                           int64_t t_first, int64_t count,
                           const uint32_t* __restrict__ empty_bits, uint32_t* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count) return;
  const int64_t t = t_first + idx;
  const int64_t row = row_of_nonzero_dev(rp, m, t * B);
  bool flag = false;
  if (t < p) {
    const int64_t next = row_of_nonzero_dev(rp, m, (t + 1) * B);
    // Rows strictly inside (row, next) that are non-empty each own one of the
    // tile's B nonzeros, so a longer range must contain an empty row.
    if (next - row - 1 >= B) {
      flag = true;
    } else {
      // inclusive right endpoint, rid < m (format.cpp:65-78)
      const int64_t hi = next < m - 1 ? next : m - 1;
      for (int64_t wd = row >> 5; wd <= (hi >> 5) && !flag; ++wd) {
        uint32_t bits = empty_bits[wd];
        const int64_t lo_bit = wd * 32, hi_bit = lo_bit + 31;
        if (row > lo_bit) bits &= ~0u << (row - lo_bit);
        if (hi < hi_bit) bits &= ~0u >> (hi_bit - hi);
        flag = bits != 0;
      }
    }
  }
  out[idx] = (uint32_t)row | (flag ? 0x80000000u : 0u);
}

// sigma head bits of column `lane` of local tile k, bit j = depth j.
__device__ __forceinline__ uint64_t column_bits(const uint32_t* __restrict__ head_bits, int64_t k,
                                                int B, int sigma, int lane) {
  const int64_t pos = k * B + (int64_t)lane * sigma;
  const int64_t w0 = pos >> 5;
  const int o = (int)(pos & 31);
  uint64_t bits = ((uint64_t)head_bits[w0] | ((uint64_t)head_bits[w0 + 1] << 32)) >> o;
  if (o) bits |= (uint64_t)head_bits[w0 + 2] << (64 - o);
  bits &= (1ull << sigma) - 1;  // sigma <= 48
  if (lane == 0) bits |= 1ull;  // bf[0] = 1, format.cpp:98
  return bits;
}

template <typename W>
__global__ void __launch_bounds__(128) k_desc_transpose(
    const uint32_t* __restrict__ head_bits, const uint32_t* __restrict__ tile_ptr,
    const int32_t* __restrict__ col_in, const double* __restrict__ val_in,
    int32_t* __restrict__ col_out, double* __restrict__ val_out, W* __restrict__ desc,
    int64_t* __restrict__ eo_cnt, int64_t pcs, int sigma) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t k = (int64_t)blockIdx.x * 4 + wib;
  if (k >= pcs) return;
  const int B = 32 * sigma;

  // ---- descriptor (format.cpp:102-121 + descriptor.cpp:38-62) ----
  const uint64_t bits = column_bits(head_bits, k, B, sigma, lane);
  const int cnt = __popcll(bits);
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += t;
  }
  const int yoff = incl - cnt;
  const int H = __shfl_sync(kFull, incl, 31);
  const uint32_t hb = __ballot_sync(kFull, cnt > 0);
  const uint64_t above = (uint64_t)hb >> (lane + 1);
  const int seg = cnt ? (above ? __ffsll((long long)above) - 1 : 31 - lane) : 0;
  const uint64_t flags = __brevll(bits) >> (64 - sigma);  // depth j at bit sigma-1-j
  desc[k * 32 + lane] =
      (W)(((uint64_t)yoff << (kSegBits + sigma)) | ((uint64_t)seg << sigma) | flags);
  if (eo_cnt && lane == 0) eo_cnt[k] = (tile_ptr[k] >> 31) ? H : 0;

  // ---- transpose: logical i*sigma+j -> physical j*32+i (format.hpp:76-88) ----
  const uint64_t pol = policy_evict_first();
  double* buf = smem + (size_t)wib * sigma * 33;
  const float inv = 1.0f / (float)sigma;
  const int64_t tb = k * B;
  for (int e = lane; e < B; e += 32) {
    const double v = ld_stream(val_in + tb + e, pol);
    const int i = __float2int_rz(((float)e + 0.5f) * inv);
    buf[(e - i * sigma) * 33 + i] = v;
  }
  __syncwarp();
  for (int j = 0; j < sigma; ++j) val_out[tb + j * 32 + lane] = buf[j * 33 + lane];
  __syncwarp();
  int32_t* ib = reinterpret_cast<int32_t*>(buf);
  for (int e = lane; e < B; e += 32) {
    const int32_t c = ld_stream(col_in + tb + e, pol);
    const int i = __float2int_rz(((float)e + 0.5f) * inv);
    ib[(e - i * sigma) * 33 + i] = c;
  }
  __syncwarp();
  for (int j = 0; j < sigma; ++j) col_out[tb + j * 32 + lane] = ib[j * 33 + lane];
}

// Same output as k_desc_transpose, fed by TMA: persistent warps walk tiles
// gw, gw + W, ...; lane 0 bulk-copies a tile's val (B*8 bytes) and col_idx (B*4)
// into a 2-stage linear ring one tile ahead, so the global reads are deep
// asynchronous streams instead of latency-bound register loads.  The lanes then
// move the tile through a padded buffer (conflict-free both ways) and write
// the transposed rows coalesced.  Needs 16-byte aligned inputs (the launcher
// falls back to k_desc_transpose otherwise).
template <typename W>
__global__ void __launch_bounds__(512) k_desc_transpose_tma(
    const uint32_t* __restrict__ head_bits, const uint32_t* __restrict__ tile_ptr,
    const int32_t* __restrict__ col_in, const double* __restrict__ val_in,
    int32_t* __restrict__ col_out, double* __restrict__ val_out, W* __restrict__ desc,
    int64_t* __restrict__ eo_cnt, int64_t pcs, int sigma, int stage_bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, NW = blockDim.x >> 5;
  const int B = 32 * sigma;
  const int64_t nwt = (int64_t)gridDim.x * NW;
  const int64_t gw = (int64_t)blockIdx.x * NW + wib;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm) + 2 * wib;
  const size_t pad_bytes = ((size_t)sigma * 33 * 8 + 127) / 128 * 128;
  unsigned char* base = sm + 256 + (size_t)wib * (2 * (size_t)stage_bytes + pad_bytes);
  double* buf = reinterpret_cast<double*>(base + 2 * (size_t)stage_bytes);
  const uint64_t pol = policy_evict_first();
  auto issue = [&](int64_t k, int st) {  // lane 0
    unsigned char* dst = base + (size_t)st * stage_bytes;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect(bars + st, (uint32_t)B * 12u);
    bulk_load(dst, val_in + k * B, (uint32_t)B * 8u, bars + st, pol);
    bulk_load(dst + (size_t)B * 8, col_in + k * B, (uint32_t)B * 4u, bars + st, pol);
  };
  if (lane == 0) {
    mbar_init(bars);
    mbar_init(bars + 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (gw < pcs) issue(gw, 0);
    if (gw + nwt < pcs) issue(gw + nwt, 1);
  }
  __syncwarp();
  const float inv = 1.0f / (float)sigma;
  int st = 0;
  uint32_t phase = 0;
  for (int64_t k = gw; k < pcs; k += nwt) {
    // ---- descriptor (format.cpp:102-121 + descriptor.cpp:38-62) ----
    const uint64_t bits = column_bits(head_bits, k, B, sigma, lane);
    const int cnt = __popcll(bits);
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    const int yoff = incl - cnt;
    const int H = __shfl_sync(kFull, incl, 31);
    const uint32_t hb = __ballot_sync(kFull, cnt > 0);
    const uint64_t above = (uint64_t)hb >> (lane + 1);
    const int seg = cnt ? (above ? __ffsll((long long)above) - 1 : 31 - lane) : 0;
    const uint64_t flags = __brevll(bits) >> (64 - sigma);
    desc[k * 32 + lane] =
        (W)(((uint64_t)yoff << (kSegBits + sigma)) | ((uint64_t)seg << sigma) | flags);
    if (eo_cnt && lane == 0) eo_cnt[k] = (tile_ptr[k] >> 31) ? H : 0;

    // ---- transpose: logical i*sigma+j -> physical j*32+i (format.hpp:76-88) ----
    mbar_wait(bars + st, phase);
    const double* sv = reinterpret_cast<const double*>(base + (size_t)st * stage_bytes);
    const int32_t* sc = reinterpret_cast<const int32_t*>(sv + B);
    const int64_t tb = k * B;
    for (int e = lane; e < B; e += 32) {
      const int i = __float2int_rz(((float)e + 0.5f) * inv);
      buf[(e - i * sigma) * 33 + i] = sv[e];
    }
    __syncwarp();
    for (int j = 0; j < sigma; ++j) val_out[tb + j * 32 + lane] = buf[j * 33 + lane];
    __syncwarp();
    int32_t* ib = reinterpret_cast<int32_t*>(buf);
    for (int e = lane; e < B; e += 32) {
      const int i = __float2int_rz(((float)e + 0.5f) * inv);
      ib[(e - i * sigma) * 33 + i] = sc[e];
    }
    __syncwarp();  // the stage has been read: refill it two tiles ahead
    if (lane == 0 && k + 2 * nwt < pcs) issue(k + 2 * nwt, st);
    for (int j = 0; j < sigma; ++j) col_out[tb + j * 32 + lane] = ib[j * 33 + lane];
    __syncwarp();
    st ^= 1;
    phase ^= (st == 0);
  }
}

// empty_offset entries of flagged tiles (format.cpp:123-136): for every head
// in column-major order, row_of_nonzero(g) - tile_row.
// Heads of a flagged tile in order: head 0 is tile_row (eo = 0); the others
// are the non-empty rows r in (tile_row, next_row] whose first nonzero lies
// strictly inside the tile -- row_of_nonzero (format.cpp:42-50) of a head
// position is the rightmost row of its equal row_ptr run, i.e. the non-empty
// row starting there.  Tiles spanning at most kEoScanRows rows: the warp scans
// row_ptr over the span (coalesced; the spans of all tiles overlap only at
// their ends, so the scans read row_ptr about once in total).  Wider spans
// (long empty-row runs): one binary search per head, bounded by the span.
constexpr int64_t kEoScanRows = 2048;
__global__ void k_eo(const uint32_t* __restrict__ head_bits, const uint32_t* __restrict__ tile_ptr,
                     const int64_t* __restrict__ rp, int64_t m, int64_t pcs, int sigma,
                     int64_t pos0, const int64_t* __restrict__ eo_ptr, int32_t* __restrict__ eo) {
  const int lane = threadIdx.x & 31;
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= pcs) return;
  const uint32_t tp = tile_ptr[k];
  if (!(tp >> 31)) return;
  const int B = 32 * sigma;
  const int64_t tile_row = tp & 0x7fffffffu;
  const int64_t next_row = tile_ptr[k + 1] & 0x7fffffffu;
  if (next_row - tile_row <= kEoScanRows) {
    const int64_t start = pos0 + k * B, end = start + B;
    int64_t out = eo_ptr[k];
    if (lane == 0) eo[out] = 0;
    ++out;
    for (int64_t base = tile_row + 1; base <= next_row; base += 32) {
      const int64_t r = base + lane;
      const bool valid = r <= next_row;
      const int64_t a = valid ? rp[r] : 0;
      int64_t b = __shfl_down_sync(kFull, a, 1);
      if (valid && (lane == 31 || r + 1 > next_row)) b = rp[r + 1];
      const bool head = valid && a > start && a < end && b > a;
      const uint32_t hm = __ballot_sync(kFull, head);
      if (head) eo[out + __popc(hm & ((1u << lane) - 1))] = (int32_t)(r - tile_row);
      out += __popc(hm);
    }
    return;
  }
  uint64_t bits = column_bits(head_bits, k, B, sigma, lane);
  const int cnt = __popcll(bits);
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += t;
  }
  int64_t out = eo_ptr[k] + (incl - cnt);
  const int64_t hi = (next_row + 2 < m + 1) ? next_row + 2 : m + 1;
  while (bits) {
    const int j = __ffsll((long long)bits) - 1;
    bits &= bits - 1;
    const int64_t g = pos0 + k * B + (int64_t)lane * sigma + j;
    const int64_t row = upper_bound_dev(rp, tile_row + 1, hi, g) - 1;
    eo[out++] = (int32_t)(row - tile_row);
  }
}

// Per-tile SpMV work in nonzero-equivalents, for the warps' tile ranges (k_tile_scan):
// B (stream + gathers) + w_head * heads + w_row * rows spanned (y stores,
// empty rows zeroed).  Tiles spanning many short and empty rows cost several
// times a tile of long rows; an equal-tile split gives the warps holding them
// (unpermuted power-law matrices: the whole tail) most of the work.  Measured
// on R-MAT s24 unpermuted: equal split 4.42 ms; weights (head, row) = (1,0)
// 3.90, (0,1) 1.91, (1,1) 1.87, (4,2) 1.79 ms.

// Largest per-warp work of the equal-tile split (atomicMax into *out).
__global__ void k_equal_split_max(const int64_t* __restrict__ prefix, int64_t pcs, int nw,
                                  unsigned long long* __restrict__ out) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  const int64_t b = (int64_t)w * pcs / nw, e = (int64_t)(w + 1) * pcs / nw;
  if (e <= b) return;
  const int64_t work = prefix[e - 1] - (b > 0 ? prefix[b - 1] : 0);
  atomicMax(out, (unsigned long long)work);
}

// Warp tile ranges.  The equal-tile split (CSR5 tiles are equal-nnz units)
// unless its busiest warp would carry more than 5/4 of the mean work; then
// warp w starts at the first tile whose inclusive work prefix exceeds w/nw of
// the total.  k_warp_bounds_fix then gives every warp at least one tile.
__global__ void k_warp_bounds(const int64_t* __restrict__ prefix, int64_t pcs, int nw,
                              const unsigned long long* __restrict__ equal_max,
                              int64_t* __restrict__ begin) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w > nw) return;
  if (w == 0 || w == nw) {
    begin[w] = w == 0 ? 0 : pcs;
    return;
  }
  const int64_t total = prefix[pcs - 1];
  if ((double)*equal_max * nw <= 1.25 * (double)total) {
    begin[w] = (int64_t)w * pcs / nw;
    return;
  }
  const int64_t target = (int64_t)((__int128)total * w / nw);
  int64_t lo = 0, hi = pcs;  // first t with prefix[t] > target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (prefix[mid] <= target)
      lo = mid + 1;
    else
      hi = mid;
  }
  begin[w] = lo;
}

// Every warp gets at least one tile: the serial passes
//   for w = 1..nw-1:  b[w] = max(b[w], b[w-1] + 1)
//   for w = nw-1..1:  b[w] = min(b[w], b[w+1] - 1)      (b[0] = 0, b[nw] = pcs)
// are b'[w] = w + max_{j<=w}(b[j] - j) and b''[w] = w + min_{j>=w}(b'[j] - j):
// a prefix max and a suffix min, done by one CTA (nw <= 32 * 1024).
constexpr int kFixThreads = 1024;
// Block-wide exclusive scans for the one-CTA plan kernels (kFixThreads
// threads): warp shuffles, then one pass over the warp totals -- three
// barriers instead of a log-step shared-memory scan's twenty.  fwd: the op
// over threads < t; bwd: the op over threads > t.
template <typename T, typename Op>
__device__ __forceinline__ T block_excl_fwd(T v, T ident, Op op, T* wtot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T o = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v = op(v, o);
  }
  T x = __shfl_up_sync(kFull, v, 1);
  if (lane == 0) x = ident;
  if (lane == 31) wtot[w] = v;
  __syncthreads();
  if (w == 0) {
    T t = lane < nw ? wtot[lane] : ident;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const T o = __shfl_up_sync(kFull, t, d);
      if (lane >= d) t = op(t, o);
    }
    wtot[lane] = t;
  }
  __syncthreads();
  const T before = w > 0 ? wtot[w - 1] : ident;
  __syncthreads();  // wtot is reused by the next scan
  return op(x, before);
}
template <typename T, typename Op>
__device__ __forceinline__ T block_excl_bwd(T v, T ident, Op op, T* wtot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T o = __shfl_down_sync(kFull, v, d);
    if (lane + d < 32) v = op(v, o);
  }
  T x = __shfl_down_sync(kFull, v, 1);
  if (lane == 31) x = ident;
  if (lane == 0) wtot[w] = v;
  __syncthreads();
  if (w == 0) {
    T t = lane < nw ? wtot[lane] : ident;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const T o = __shfl_down_sync(kFull, t, d);
      if (lane + d < 32) t = op(t, o);
    }
    wtot[lane] = t;
  }
  __syncthreads();
  const T after = w + 1 < nw ? wtot[w + 1] : ident;
  __syncthreads();
  return op(x, after);
}
struct MaxOp {
  template <typename T>
  __device__ T operator()(T a, T b) const { return a > b ? a : b; }
};
struct MinOp {
  template <typename T>
  __device__ T operator()(T a, T b) const { return a < b ? a : b; }
};

struct AddOp {
  template <typename T>
  __device__ T operator()(T a, T b) const { return a + b; }
};

// ---- per-tile work and both prefix sums in one pass --------------------------
// k_tile_scan replaces k_tile_work and the two CUB scans (empty_offset_ptr,
// exclusive, format.cpp:213-217; the warp split's work prefix, inclusive):
// a single-pass chained scan with decoupled look-back.  Each CTA takes the
// next chunk of kScanTiles tiles (a dynamic chunk index, so every predecessor
// of a chunk has started), publishes its aggregate, sums its predecessors'
// published values back to the first inclusive prefix, and writes its tiles'
// prefixes -- one launch instead of five on the converter's critical path.
constexpr int kScanThreads = 256, kScanPer = 4, kScanTiles = kScanThreads * kScanPer;
struct ScanStatus {  // flag 0 nothing yet, 1 aggregate published, 2 inclusive prefix published
  unsigned long long flag;
  long long agg_e, agg_w;  // written once, before flag 1 (never changed afterwards)
  long long inc_e, inc_w;  // written once, before flag 2
};

__global__ void __launch_bounds__(kScanThreads) k_tile_scan(
    const uint32_t* __restrict__ head_bits, const uint32_t* __restrict__ tile_ptr, int64_t pcs,
    int sigma, int w_head, int w_row, ScanStatus* status, unsigned int* chunk_ctr,
    int64_t* __restrict__ eo_ptr, int64_t* __restrict__ work_prefix, int* __restrict__ max_heads,
    unsigned long long* __restrict__ single_head) {
  __shared__ int64_t wtot[32];
  __shared__ int64_t pre_e, pre_w;
  __shared__ unsigned int chunk;
  __shared__ int bmax;
  __shared__ unsigned int bone;
  const int t = threadIdx.x;
  if (t == 0) {
    chunk = atomicAdd(chunk_ctr, 1u);
    bmax = 0, bone = 0;
  }
  __syncthreads();
  const int64_t b = chunk;
  const int64_t k0 = b * kScanTiles + (int64_t)t * kScanPer;
  int64_t ec[kScanPer], wk[kScanPer], se = 0, sw = 0;
  int mh = 0;
  unsigned one = 0;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    const int64_t k = k0 + i;
    ec[i] = wk[i] = 0;
    if (k < pcs) {
      const uint32_t* wd = head_bits + k * sigma;  // a tile is sigma 32-bit words
      int h = (wd[0] & 1u) ? 0 : 1;                // bf[0] is forced
      for (int j = 0; j < sigma; ++j) h += __popc(wd[j]);
      const uint32_t tp = tile_ptr[k];
      const int64_t rows = (int64_t)(tile_ptr[k + 1] & 0x7fffffffu) - (tp & 0x7fffffffu) + 1;
      wk[i] = 32ll * sigma + (int64_t)w_head * h + (int64_t)w_row * rows;
      ec[i] = (tp >> 31) ? h : 0;  // empty_offset entries: heads of flagged tiles
      mh = max(mh, h);
      one += h == 1;  // a tile inside one row (long rows need one)
    }
    se += ec[i];
    sw += wk[i];
  }
  if (mh) atomicMax(&bmax, mh);
  if (one) atomicAdd(&bone, one);
  int64_t xe = block_excl_fwd<int64_t>(se, 0, AddOp{}, wtot);
  int64_t xw = block_excl_fwd<int64_t>(sw, 0, AddOp{}, wtot);
  if (t == kScanThreads - 1) {  // the chunk's aggregate: publish, then look back
    const int64_t ae = xe + se, aw = xw + sw;
    volatile ScanStatus* st = status + b;
    int64_t pe = 0, pw = 0;
    if (b == 0) {
      st->inc_e = ae, st->inc_w = aw;
      __threadfence();
      st->flag = 2;
    } else {
      st->agg_e = ae, st->agg_w = aw;
      __threadfence();
      st->flag = 1;
      // a predecessor's flag may move from 1 to 2 at any time: read the field
      // pair that the flag seen names (each is written once, before its flag)
      for (int64_t j = b - 1; j >= 0; --j) {
        volatile ScanStatus* q = status + j;
        unsigned long long f;
        while ((f = q->flag) == 0) {
        }
        __threadfence();
        if (f == 2) {
          pe += q->inc_e;
          pw += q->inc_w;
          break;
        }
        pe += q->agg_e;
        pw += q->agg_w;
      }
      st->inc_e = pe + ae, st->inc_w = pw + aw;
      __threadfence();
      st->flag = 2;
    }
    pre_e = pe, pre_w = pw;
    if (b == (pcs - 1) / kScanTiles) eo_ptr[pcs] = pe + ae;  // the last chunk closes eo_ptr
  }
  __syncthreads();
  xe += pre_e;
  xw += pre_w;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    const int64_t k = k0 + i;
    if (k < pcs) {
      eo_ptr[k] = xe;
      xe += ec[i];
      xw += wk[i];
      work_prefix[k] = xw;
    }
  }
  if (t == 0 && bmax > 0) atomicMax(max_heads, bmax);
  if (t == 0 && bone > 0) atomicAdd(single_head, (unsigned long long)bone);
}

__global__ void __launch_bounds__(kFixThreads) k_warp_bounds_fix(int64_t* __restrict__ begin,
                                                                  int nw) {
  __shared__ int64_t wtot[32];
  const int t = threadIdx.x;
  const int per = (nw + kFixThreads - 1) / kFixThreads;
  // forward over j in [0, nw): inclusive prefix max of begin[j] - j
  int lo = min(nw, t * per), hi = min(nw, lo + per);
  int64_t m = LLONG_MIN;
  for (int j = lo; j < hi; ++j) m = max(m, begin[j] - j);
  int64_t run = block_excl_fwd<int64_t>(m, LLONG_MIN, MaxOp{}, wtot);
  for (int j = lo; j < hi; ++j) {
    run = max(run, begin[j] - j);
    if (j >= 1) begin[j] = j + run;
  }
  __syncthreads();
  // backward over j in [1, nw] (begin[nw] = pcs fixed): suffix min of begin[j] - j
  lo = 1 + min(nw, t * per);
  hi = 1 + min(nw, t * per + per);
  m = LLONG_MAX;
  for (int j = lo; j < hi; ++j) m = min(m, begin[j] - j);
  run = block_excl_bwd<int64_t>(m, LLONG_MAX, MinOp{}, wtot);
  for (int j = hi - 1; j >= lo; --j) {
    run = min(run, begin[j] - j);
    if (j < nw) begin[j] = j + run;
  }
}

// ---- long rows (deterministic mode's fixed summation order) ----------------
// A row whose nonzeros touch three or more parts (complete tiles, the tail)
// is "long": its per-tile partials are stored, one slot per part, and summed
// by the last arriving warp in one fixed order (lane-strided sums, then an
// xor butterfly over 32 lanes), so its value does not depend on which warps,
// SMs or GPUs hold which tiles.  Every other row has one or two partials:
// one is the value, two are added (a + b is b + a) -- also partition-free.
struct LongRowPred {
  const int64_t* rp;
  int64_t B, pc;
  __device__ __forceinline__ bool operator()(int64_t r) const {
    const int64_t lo = rp[r], hi = rp[r + 1];
    if (hi - lo < B + 2) return false;  // three parts: a whole tile plus one entry each side
    const int64_t f = min(lo / B, pc), l = min((hi - 1) / B, pc);
    return l - f >= 2;
  }
};

__device__ __forceinline__ int64_t find_long(const int64_t* __restrict__ lrow, int64_t n,
                                             int64_t row) {
  int64_t lo = 0, hi = n;  // first index with lrow >= row
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (lrow[mid] < row)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < n && lrow[lo] == row ? lo : -1;
}

// per long row L < *count: first tile and number of parts (0 beyond *count)
__global__ void k_long_info(const int64_t* __restrict__ rp, int64_t B, int64_t pc,
                            const int64_t* __restrict__ lrow, const int64_t* __restrict__ count,
                            int64_t cap, int64_t* __restrict__ ltf, int64_t* __restrict__ lnp) {
  const int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (L >= cap) return;
  if (L >= *count) {
    lnp[L] = 0;
    return;
  }
  const int64_t r = lrow[L], f = min(rp[r] / B, pc), l = min((rp[r + 1] - 1) / B, pc);
  ltf[L] = f;
  lnp[L] = l - f + 1;
}

// per held tile, one word: (b << 2) | head0_long | last_long << 1, b = the
// first long id whose row is >= the tile's head-0 row.  The head-0 row's id
// is b; the last head's (a different row) is b + head0_long -- no long row
// fits between the two, since a long row covers a whole tile.
template <typename W>
__global__ void k_long_tags(int64_t pcs, const uint32_t* __restrict__ tile_ptr,
                            const W* __restrict__ desc, const int64_t* __restrict__ eo_ptr,
                            const int32_t* __restrict__ eo, int sigma,
                            const int64_t* __restrict__ lrow, const int64_t* __restrict__ count,
                            int32_t* __restrict__ tag) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= pcs) return;
  const int64_t n = *count;
  const uint32_t tp = tile_ptr[t];
  const int64_t r0 = tp & 0x7fffffffu;
  const uint64_t wd = (uint64_t)desc[t * 32 + 31];
  const int H = (int)(wd >> (kSegBits + sigma)) + __popcll(wd & ((1ull << sigma) - 1));
  const int64_t rl = r0 + ((tp >> 31) ? (int64_t)eo[eo_ptr[t] + H - 1] : H - 1);
  int64_t lo = 0, hi = n;  // first long id with lrow >= r0
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (lrow[mid] < r0)
      lo = mid + 1;
    else
      hi = mid;
  }
  const bool h0 = lo < n && lrow[lo] == r0;
  const int64_t nl = lo + (h0 ? 1 : 0);
  const bool hl = rl != r0 && nl < n && lrow[nl] == rl;
  tag[t] = (int32_t)((lo << 2) | (h0 ? 1 : 0) | (hl ? 2 : 0));
}

__global__ void k_long_tail(int64_t tail_row, int has_tail, const int64_t* __restrict__ lrow,
                            const int64_t* __restrict__ count, int32_t* __restrict__ out) {
  *out = has_tail ? (int32_t)find_long(lrow, *count, tail_row) : -1;
}

// Item rows of the in-kernel calibration (spmv.cu resolve_item): item 2w is
// the row of warp w's first tile start, item 2w+1 the row holding the warp's
// last nonzero -- the last head of its last tile t: H = y_offset + popc(flags)
// of column 31, row = tile_row + (flagged ? eo[eo_ptr[t] + H - 1] : H - 1) --
// and item 2*nwarps (tail) the tail's first row.  O(1) loads per item.
template <typename W>
__global__ void k_item_keys(const int64_t* __restrict__ warp_begin,
                            const uint32_t* __restrict__ tile_ptr, const W* __restrict__ desc,
                            const int64_t* __restrict__ eo_ptr, const int32_t* __restrict__ eo,
                            int sigma, int nwarps, int has_tail_item, int64_t tail_row_begin,
                            const int64_t* __restrict__ lrow, const int64_t* __restrict__ nlong,
                            int64_t* __restrict__ key) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = 2 * nwarps + (has_tail_item ? 1 : 0);
  if (i >= n) return;
  int64_t row;
  if (i == 2 * nwarps) {
    row = tail_row_begin;
  } else if ((i & 1) == 0) {
    row = tile_ptr[warp_begin[i >> 1]] & 0x7fffffffu;
  } else {
    const int64_t t = warp_begin[(i >> 1) + 1] - 1;
    const uint32_t tp = tile_ptr[t];
    const uint64_t wd = (uint64_t)desc[t * 32 + 31];
    const int H = (int)(wd >> (kSegBits + sigma)) + __popcll(wd & ((1ull << sigma) - 1));
    row = (int64_t)(tp & 0x7fffffffu) + ((tp >> 31) ? (int64_t)eo[eo_ptr[t] + H - 1] : H - 1);
  }
  // a long row's partials go through its part slots, not the items: its items
  // get keys of their own (single-item runs the kernel skips)
  key[i] = lrow && find_long(lrow, *nlong, row) >= 0 ? -2 - (int64_t)i : row;
}

// Runs of equal keys (keys are non-decreasing): run_first[i] = prefix max of
// the run starts, run_last[i] = suffix min of the run ends -- one CTA, the
// scans of k_warp_bounds_fix.
__global__ void __launch_bounds__(kFixThreads) k_item_runs(const int64_t* __restrict__ key, int n,
                                                           int32_t* __restrict__ run_first,
                                                           int32_t* __restrict__ run_last,
                                                           int32_t* __restrict__ run_cnt,
                                                           double* __restrict__ item_val) {
  __shared__ int wtot[32];
  const int t = threadIdx.x;
  for (int i = t; i < n; i += kFixThreads) {  // per-launch state: no arrivals, idle pair slots
    run_cnt[i] = 0;
    item_val[i] = __longlong_as_double(-1ll);
  }
  const int per = (n + kFixThreads - 1) / kFixThreads;
  const int lo = min(n, t * per), hi = min(n, lo + per);
  int m = -1;
  for (int i = lo; i < hi; ++i)
    if (i == 0 || key[i] != key[i - 1]) m = i;
  int run = block_excl_fwd<int>(m, -1, MaxOp{}, wtot);
  for (int i = lo; i < hi; ++i) {
    if (i == 0 || key[i] != key[i - 1]) run = i;
    run_first[i] = run;
  }
  m = INT_MAX;
  for (int i = hi - 1; i >= lo; --i)
    if (i == n - 1 || key[i] != key[i + 1]) m = i;
  run = block_excl_bwd<int>(m, INT_MAX, MinOp{}, wtot);
  for (int i = hi - 1; i >= lo; --i) {
    if (i == n - 1 || key[i] != key[i + 1]) run = i;
    run_last[i] = run;
  }
}

// Every scalar the host needs from the build, gathered by one thread into one
// block for a single read-back: row_of_nonzero at two positions (negative
// query = skip), row_ptr at the first and the closing row, the empty_offset
// total, the largest head count, the two tile_ptr words, the locality count.
// format.cpp:42-50 row_of_nonzero by one warp: a 32-ary upper_bound over
// row_ptr[0, m] (4 rounds of coalesced probes for a million rows instead of
// 20 dependent loads)
__device__ int64_t row_of_nonzero_warp(const int64_t* __restrict__ rp, int64_t m, int64_t g) {
  const int lane = threadIdx.x & 31;
  int64_t lo = 0, hi = m + 1;  // first index in [lo, hi) with rp[idx] > g
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = min(lo + (int64_t)(lane + 1) * step - 1, hi - 1);
    const uint32_t b = __ballot_sync(kFull, rp[p] > g);
    if (b == 0) {
      lo = min(lo + 32 * step, hi);
    } else {
      const int f = __ffs(b) - 1;
      const int64_t nlo = lo + (int64_t)f * step, nhi = min(lo + (int64_t)(f + 1) * step, hi);
      lo = nlo;
      hi = nhi;
    }
  }
  const int64_t q = lo + lane;
  const uint32_t b = __ballot_sync(kFull, q < hi && rp[q] > g);
  const int64_t idx = b ? lo + __ffs(b) - 1 : hi;
  int64_t r = idx - 1;
  r = r < 0 ? 0 : r;
  return r > m - 1 ? m - 1 : r;
}

// one CTA of 64 threads: warp 0 and warp 1 find the two rows, thread 0 the rest
__global__ void k_scalars(const int64_t* __restrict__ rp, int64_t m, int64_t g0, int64_t g1,
                          const uint32_t* __restrict__ tile_ptr, int64_t ic,
                          const int64_t* __restrict__ eo_ptr, int64_t pcs,
                          const int* __restrict__ max_heads,
                          const unsigned long long* __restrict__ lines,
                          const unsigned long long* __restrict__ single_head,
                          int64_t* __restrict__ out) {
  const bool rows = m > 0;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w < 2) {
    const int64_t g = w == 0 ? g0 : g1;
    const int64_t r = rows && g >= 0 ? row_of_nonzero_warp(rp, m, g) : -1;
    if (lane == 0) out[w] = r;
  }
  if (threadIdx.x != 0) return;
  out[2] = rows ? rp[tile_ptr[0] & 0x7fffffffu] : -1;
  out[3] = rows ? rp[tile_ptr[ic] & 0x7fffffffu] : -1;
  out[4] = eo_ptr[pcs];
  out[5] = *max_heads;
  out[6] = tile_ptr[0];
  out[7] = tile_ptr[ic];
  out[8] = (int64_t)*lines;
  out[9] = (int64_t)*single_head;
}

// Gather locality of the SpMV: for `samples` evenly spaced tiles, the number
// of distinct 128-byte lines of x that one warp-wide gather (one depth step)
// touches, summed into *acc.  1 = perfectly coalesced, 32 = fully random.
__global__ void k_locality(const int32_t* __restrict__ col, int64_t pcs, int sigma, int64_t samples,
                           unsigned long long* __restrict__ acc) {
  // col is the caller's CSR-order col_idx: tile k's column i, depth j sits at
  // k*B + i*sigma + j (the SpMV reads it transposed, the lines touched by one
  // warp-wide gather are the same), so the sample runs beside the transposition
  const int lane = threadIdx.x & 31;
  const int64_t sidx = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (sidx >= samples) return;
  const int64_t k = sidx * pcs / samples;
  const int B = 32 * sigma;
  unsigned total = 0;
  for (int j = 0; j < sigma; ++j) {
    const int32_t line = col[k * B + (int64_t)lane * sigma + j] >> 4;
    const unsigned peers = __match_any_sync(kFull, line);
    total += (__ffs(peers) - 1) == lane;  // one leader per distinct line
  }
  total = __reduce_add_sync(kFull, total);
  if (lane == 0) atomicAdd(acc, (unsigned long long)total);
}

__global__ void k_untranspose(const int32_t* __restrict__ col_in, const double* __restrict__ val_in,
                              int32_t* __restrict__ col_out, double* __restrict__ val_out,
                              int64_t n_tiled, int sigma) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_tiled) return;
  const int B = 32 * sigma;
  const int64_t k = idx / B;
  const int rem = (int)(idx - k * B);
  const int i = rem / sigma, j = rem - (rem / sigma) * sigma;
  const int64_t src = k * B + (int64_t)j * 32 + i;
  col_out[idx] = col_in[src];
  val_out[idx] = val_in[src];
}

// Handle memory comes from the device's stream-ordered pool with an unbounded
// release threshold: a rebuild after a release reuses the pages instead of
// paying cudaMalloc's page mapping again (allocation is reported separately,
// as the paper separates it from conversion).
thread_local cudaStream_t t_alloc_stream = nullptr;

// Per-device side stream of the converter: the empty_offset / plan chain runs
// on it while the transposition streams the matrix on the caller's stream.
int side_stream(int device, cudaStream_t* out) {
  static std::mutex mu;
  static cudaStream_t side[64] = {};
  if (device < 0 || device >= 64) return fail(CSR5G_EINVAL, "csr5g: device id out of range");
  std::lock_guard<std::mutex> lock(mu);
  if (!side[device]) CSR5G_CUDA(cudaStreamCreateWithFlags(&side[device], cudaStreamNonBlocking));
  *out = side[device];
  return CSR5G_OK;
}

int ensure_pool(int device) {
  static bool done[64] = {};
  if (device < 64 && done[device]) return CSR5G_OK;
  cudaMemPool_t pool;
  CSR5G_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = ~uint64_t(0);
  CSR5G_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  if (device < 64) done[device] = true;
  return CSR5G_OK;
}

template <typename T>
int dev_alloc(T** p, size_t count, double* alloc_ms, int64_t* bytes) {
  const auto t0 = std::chrono::steady_clock::now();
  const size_t nb = std::max<size_t>(count * sizeof(T), 16);
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), nb, t_alloc_stream);
  *alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(CSR5G_ENOMEM, "csr5g: device allocation of " + std::to_string(nb) +
                                  " bytes failed: " + cudaGetErrorString(e));
  }
  *bytes += (int64_t)nb;
  return CSR5G_OK;
}

// CSR5G_TRACE=1: synchronise after each build phase and print the phase times
// to stderr (a profiling aid; off by default, no syncs added when off);
// CSR5G_TRACE=2: the host-side time of each phase, without the syncs.
struct BuildTrace {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point last;
  std::string log;
  bool host_only = false;  // CSR5G_TRACE=2: host (enqueue) time per phase, no syncs
  explicit BuildTrace(cudaStream_t s) : on(std::getenv("CSR5G_TRACE") != nullptr), st(s) {
    host_only = on && std::atoi(std::getenv("CSR5G_TRACE")) == 2;
    last = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    if (!host_only) cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    char buf[96];
    std::snprintf(buf, sizeof buf, " %s=%.3fms", what,
                  std::chrono::duration<double, std::milli>(t - last).count());
    log += buf;
    last = t;
  }
  ~BuildTrace() {
    if (on) std::fprintf(stderr, "[csr5g build]%s\n", log.c_str());
  }
};

int check_params(const csr5g_params* pr, int64_t m, int64_t nnz, bool shard, int64_t* sigma_out,
                 int32_t* yb, int32_t* sb, int32_t* wb) {
  if (!pr) return fail(CSR5G_EINVAL, "csr5g: params is NULL");
  int64_t sigma = pr->sigma;
  if (sigma == 0) {
    if (shard) return fail(CSR5G_EINVAL, "csr5g: a shard build needs the global sigma");
    const int rc = csr5g_select_sigma(m > 0 ? (double)nnz / (double)m : 0.0, pr->r, pr->s, pr->t,
                                      pr->u, &sigma);
    if (rc) return rc;
  }
  // tuning.cpp:8-15
  if (pr->omega < 1 || sigma < 1) return fail(CSR5G_EINVAL, "tuning: omega and sigma must be >= 1");
  if (pr->omega * sigma < 2)
    return fail(CSR5G_EINVAL,
                "tuning: omega * sigma must be >= 2; a tile needs at least two entries for "
                "segmentation");
  if (!(pr->r <= pr->s && pr->s <= pr->t))
    return fail(CSR5G_EINVAL, "tuning: bounds must satisfy r <= s <= t");
  if (pr->u < 1) return fail(CSR5G_EINVAL, "tuning: u must be >= 1");
  if (pr->omega != kOmega)
    return fail(CSR5G_EINVAL,
                "csr5g: omega must be 32 on the GPU path (one warp lane per tile column), got " +
                    std::to_string(pr->omega));
  const int rc = csr5g_layout(pr->omega, sigma, yb, sb, wb);
  if (rc) return rc;
  *sigma_out = sigma;
  return CSR5G_OK;
}

}  // namespace

void free_handle(Handle* h) {
  if (!h) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  free_pipeline(h->pipe);
  free_binding(h->mg);
  for (void* p : {(void*)h->row_ptr, (void*)h->tile_ptr, h->desc, (void*)h->eo_ptr, (void*)h->eo,
                  (void*)h->col, (void*)h->val, (void*)h->item_val, (void*)h->run_first,
                  (void*)h->run_last, (void*)h->run_cnt, (void*)h->send, (void*)h->spill,
                  (void*)h->warp_begin, (void*)h->lrow, (void*)h->ltf, (void*)h->lnp,
                  (void*)h->lbase, (void*)h->nlong_d, (void*)h->ltag,
                  (void*)h->lparts, (void*)h->lcnt, (void*)h->hot_cols, (void*)h->xh,
                  (void*)(h->col_x != h->col ? h->col_x : nullptr)})
    if (p) cudaFreeAsync(p, 0);
  for (const StreamScratch& x : h->scratch) {
    if (x.owned)
      for (void* p : {(void*)x.item_val, (void*)x.run_cnt, (void*)x.spill, (void*)x.lparts,
                      (void*)x.lcnt, (void*)x.xh})
        if (p) cudaFreeAsync(p, 0);
    if (x.done) cudaEventDestroy(x.done);
  }
  cudaDeviceSynchronize();
  cudaSetDevice(prev);
  delete h;
}

int build_handle(int device, int64_t m, int64_t n, int64_t nnz, const int64_t* d_row_ptr,
                 const int32_t* d_col_idx, const double* d_val, const csr5g_params* params,
                 int64_t tile_begin, int64_t tile_end, bool shard, int with_tail,
                 cudaStream_t stream, Handle** out) {
  const auto wall0 = std::chrono::steady_clock::now();
  if (!out) return fail(CSR5G_EINVAL, "csr5g: out is NULL");
  *out = nullptr;
  if (m < 0 || n < 0 || nnz < 0) return fail(CSR5G_EINVAL, "csr: negative dimension");
  if (m >= (int64_t(1) << 31))
    return fail(CSR5G_ERANGE, "csr5g: m >= 2^31 rows needs 64-bit tile pointers (unsupported)");
  if (n >= (int64_t(1) << 31))
    return fail(CSR5G_ERANGE, "csr5g: n >= 2^31 columns does not fit the int32 col_idx");
  if (m > 0 && !d_row_ptr) return fail(CSR5G_EINVAL, "csr5g: row_ptr is NULL");
  int64_t sigma = 0;
  int32_t yb = 0, sb = 0, wb = 0;
  int rc = check_params(params, m, nnz, shard, &sigma, &yb, &sb, &wb);
  if (rc) return rc;
  int ndev = 0;
  CSR5G_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(CSR5G_ECUDA, "csr5g: no such CUDA device");
  CSR5G_CUDA(cudaSetDevice(device));
  int major = 0;
  CSR5G_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major < 10) return fail(CSR5G_ECUDA, "csr5g: built for sm_100a; device is older");

  const int64_t B = kOmega * sigma;
  const int64_t p = (nnz + B - 1) / B, pc = nnz / B, tail = nnz % B;
  if (!shard) {
    tile_begin = 0;
    tile_end = pc;
    with_tail = tail > 0;
  }
  if (tile_begin < 0 || tile_end < tile_begin || tile_end > pc)
    return fail(CSR5G_EINVAL, "csr5g: shard tile range outside [0, p_complete]");
  const bool is_last = tile_end == pc;
  if ((with_tail != 0) != (is_last && tail > 0))
    return fail(CSR5G_EINVAL, "csr5g: the shard ending at p_complete must hold the tail");
  const int64_t pcs = tile_end - tile_begin;
  const int64_t nnz_held = pcs * B + (is_last ? tail : 0);
  if (nnz_held > 0 && (!d_col_idx || !d_val)) return fail(CSR5G_EINVAL, "csr5g: col_idx/val is NULL");
  const int64_t last_ptr = is_last ? p : tile_end;
  const int64_t tile_ptr_len = m > 0 ? last_ptr - tile_begin + 1 : 1;

  BuildTrace trace(stream);
  {
    const int prc = ensure_pool(device);
    if (prc) return prc;
  }
  t_alloc_stream = stream;
  auto* h = new (std::nothrow) Handle();
  if (!h) return fail(CSR5G_ENOMEM, "csr5g: host allocation failed");
  h->device = device;
  h->wide = wb == 64;
  h->pcs = pcs;
  h->t0 = tile_begin;
  h->B = B;
  h->is_last = is_last;
  double alloc_ms = 0.0;
  int64_t bytes = 0;
  uint32_t *head_bits = nullptr, *empty_bits = nullptr;
  int64_t* eo_cnt = nullptr;
  int64_t* scal = nullptr;
  char* zblock = nullptr;  // head_bits | empty_bits | eo_cnt | scal, zeroed by one memset
  int64_t* work_prefix = nullptr;
  int64_t* item_key = nullptr;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  auto cleanup = [&](int code) {
    if (side && code) cudaStreamSynchronize(side);  // error path: side work may be in flight
    for (void* p : {(void*)zblock, (void*)work_prefix,
                    (void*)item_key})
      if (p) cudaFreeAsync(p, stream);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (code) free_handle(h);
    return code;
  };
#define TRY(x)                  \
  do {                          \
    int rc_ = (x);              \
    if (rc_) return cleanup(rc_); \
  } while (0)
#define TRYC(x)                                            \
  do {                                                     \
    cudaError_t e_ = (x);                                  \
    if (e_ != cudaSuccess) return cleanup(cuda_fail(e_, #x)); \
  } while (0)

  const size_t wbytes = h->wide ? 8 : 4;
  TRY(dev_alloc(&h->row_ptr, (size_t)m + 1, &alloc_ms, &bytes));
  TRY(dev_alloc(&h->tile_ptr, (size_t)tile_ptr_len, &alloc_ms, &bytes));
  TRY(dev_alloc(reinterpret_cast<char**>(&h->desc), (size_t)pcs * kOmega * wbytes, &alloc_ms, &bytes));
  TRY(dev_alloc(&h->eo_ptr, (size_t)pcs + 1, &alloc_ms, &bytes));
  TRY(dev_alloc(&h->col, (size_t)nnz_held, &alloc_ms, &bytes));
  TRY(dev_alloc(&h->val, (size_t)nnz_held, &alloc_ms, &bytes));
  TRY(dev_alloc(&h->send, 1, &alloc_ms, &bytes));
  int64_t tmp_bytes = 0;
  const int64_t head_words = (pcs * B + 31) / 32 + 3;
  const int64_t empty_words = (m + 31) / 32 + 1;
  // one zeroed block: the two bitmaps, the per-tile head counts and the
  // scalars (4 lines, 6 emax, 8 max heads, 10-18 the values read back)
  const size_t hb_bytes = ((size_t)head_words * 4 + 7) / 8 * 8;
  const size_t eb_bytes = ((size_t)empty_words * 4 + 7) / 8 * 8;
  // + the chained scan's per-chunk status and chunk counter (k_tile_scan)
  const int64_t scan_chunks = (pcs + kScanTiles - 1) / kScanTiles;
  const size_t zbytes = hb_bytes + eb_bytes + 8 * ((size_t)pcs + 1) + 8 * 22 +
                        sizeof(ScanStatus) * (size_t)scan_chunks + 16;
  TRY(dev_alloc(&zblock, zbytes, &alloc_ms, &tmp_bytes));
  head_bits = reinterpret_cast<uint32_t*>(zblock);
  empty_bits = reinterpret_cast<uint32_t*>(zblock + hb_bytes);
  eo_cnt = reinterpret_cast<int64_t*>(zblock + hb_bytes + eb_bytes);
  scal = eo_cnt + pcs + 1;

  trace.mark("alloc");
  if (m > 0) TRYC(cudaMemcpyAsync(h->row_ptr, d_row_ptr, sizeof(int64_t) * (m + 1),
                                  cudaMemcpyDeviceToDevice, stream));
  TRYC(cudaMemsetAsync(zblock, 0, zbytes, stream));
  if (m == 0) {  // (else k_rowscan writes it)
    TRYC(cudaMemsetAsync(&h->send->row, 0xff, sizeof(int64_t), stream));  // no record: row -1
    TRYC(cudaMemsetAsync(&h->send->value, 0, sizeof(double), stream));
  }

  const int64_t pos0 = tile_begin * B;
  trace.mark("init");
  if (m > 0) {
    k_rowscan<<<(unsigned)((m + 255) / 256), 256, 0, stream>>>(h->row_ptr, m, pos0, pos0 + pcs * B,
                                                               empty_bits, head_bits, h->send);
    TRYC(cudaGetLastError());
    trace.mark("rowscan");
    k_tile_ptr<<<(unsigned)((tile_ptr_len + 255) / 256), 256, 0, stream>>>(
        h->row_ptr, m, B, p, tile_begin, tile_ptr_len, empty_bits, h->tile_ptr);
    TRYC(cudaGetLastError());
  } else {
    TRYC(cudaMemsetAsync(h->tile_ptr, 0, sizeof(uint32_t), stream));  // encode_tile_ptr(0)
  }
  trace.mark("tile_ptr");
  // ---- fork: the transposition streams the matrix on `stream` while the
  // empty_offset chain (head counts, scans, host scalars, k_eo) and the warp
  // plan's work prefix run on the side stream ----
  TRY(side_stream(device, &side));
  TRYC(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
  TRYC(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
  TRYC(cudaEventRecord(ev_fork, stream));
  TRYC(cudaStreamWaitEvent(side, ev_fork, 0));
  if (pcs > 0) {
    // TMA-fed kernel when the input tiles are 16-byte aligned (B*8 and B*4 are
    // multiples of 16 for every sigma); the register-load kernel otherwise
    const bool aligned = ((uintptr_t)d_col_idx & 15) == 0 && ((uintptr_t)d_val & 15) == 0;
    if (aligned) {
      const int stage_bytes = (int)(((size_t)B * 12 + 127) / 128 * 128);
      const size_t pad_bytes = ((size_t)sigma * 33 * 8 + 127) / 128 * 128;
      const size_t per_warp = 2 * (size_t)stage_bytes + pad_bytes;
      const int nw = (int)std::max<size_t>(1, std::min<size_t>(16, (220 * 1024 - 256) / per_warp));
      const size_t smem = 256 + nw * per_warp;
      const int64_t warps_needed = pcs;
      int sms = 0;
      TRYC(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
      const unsigned grid = (unsigned)std::min<int64_t>((warps_needed + nw - 1) / nw, sms);
      if (h->wide) {
        TRY(func_attrs((const void*)k_desc_transpose_tma<uint64_t>, device, (int)smem, -1));
        k_desc_transpose_tma<uint64_t><<<grid, 32 * nw, smem, stream>>>(
            head_bits, h->tile_ptr, d_col_idx, d_val, h->col, h->val, (uint64_t*)h->desc, nullptr,
            pcs, (int)sigma, stage_bytes);
      } else {
        TRY(func_attrs((const void*)k_desc_transpose_tma<uint32_t>, device, (int)smem, -1));
        k_desc_transpose_tma<uint32_t><<<grid, 32 * nw, smem, stream>>>(
            head_bits, h->tile_ptr, d_col_idx, d_val, h->col, h->val, (uint32_t*)h->desc, nullptr,
            pcs, (int)sigma, stage_bytes);
      }
    } else {
      const size_t smem = (size_t)4 * sigma * 33 * sizeof(double);
      const unsigned grid = (unsigned)((pcs + 3) / 4);
      if (h->wide) {
        TRY(func_attrs((const void*)k_desc_transpose<uint64_t>, device, (int)smem, -1));
        k_desc_transpose<uint64_t><<<grid, 128, smem, stream>>>(
            head_bits, h->tile_ptr, d_col_idx, d_val, h->col, h->val, (uint64_t*)h->desc, nullptr,
            pcs, (int)sigma);
      } else {
        TRY(func_attrs((const void*)k_desc_transpose<uint32_t>, device, (int)smem, -1));
        k_desc_transpose<uint32_t><<<grid, 128, smem, stream>>>(
            head_bits, h->tile_ptr, d_col_idx, d_val, h->col, h->val, (uint32_t*)h->desc, nullptr,
            pcs, (int)sigma);
      }
    }
    TRYC(cudaGetLastError());
  }
  if (is_last && tail > 0) {
    TRYC(cudaMemcpyAsync(h->col + pcs * B, d_col_idx + pcs * B, sizeof(int32_t) * tail,
                         cudaMemcpyDeviceToDevice, stream));
    TRYC(cudaMemcpyAsync(h->val + pcs * B, d_val + pcs * B, sizeof(double) * tail,
                         cudaMemcpyDeviceToDevice, stream));
  }
  trace.mark("desc_transpose");

  // ---- side stream: per-tile head counts and work, empty_offset_ptr
  // (exclusive scan, format.cpp:213-217), the work prefix, host scalars ----
  t_alloc_stream = side;
  static const int w_head = [] {
    const char* e = std::getenv("CSR5G_WHEAD");
    return e ? std::atoi(e) : 0;
  }();
  static const int w_row = [] {
    const char* e = std::getenv("CSR5G_WROW");
    return e ? std::atoi(e) : 1;
  }();
  int* max_heads_d = reinterpret_cast<int*>(scal + 8);  // zeroed with the block
  auto* single_head_d = reinterpret_cast<unsigned long long*>(scal + 9);
  if (pcs > 0) {
    TRY(dev_alloc(&work_prefix, (size_t)pcs, &alloc_ms, &tmp_bytes));
    auto* status = reinterpret_cast<ScanStatus*>(scal + 22);  // zeroed with the block
    auto* chunk_ctr = reinterpret_cast<unsigned int*>(status + scan_chunks);
    k_tile_scan<<<(unsigned)scan_chunks, kScanThreads, 0, side>>>(
        head_bits, h->tile_ptr, pcs, (int)sigma, w_head, w_row, status, chunk_ctr, h->eo_ptr,
        work_prefix, max_heads_d, single_head_d);
    TRYC(cudaGetLastError());
  } else {
    TRYC(cudaMemsetAsync(h->eo_ptr, 0, sizeof(int64_t), side));  // eo_ptr = {0}
  }

  // gather locality over up to 4096 sampled tiles (drives the SpMV plan), from
  // the input col_idx, read back with the scalars; its counter sits after them
  h->lines_per_gather = 1.0;
  unsigned long long lines = 0;
  const int64_t samples = std::min<int64_t>(pcs, 4096);
  auto* ctr = reinterpret_cast<unsigned long long*>(scal + 4);  // zeroed with the block
  if (pcs > 0) {
    k_locality<<<(unsigned)((samples * 32 + 255) / 256), 256, 0, side>>>(d_col_idx, pcs,
                                                                       (int)sigma, samples, ctr);
    TRYC(cudaGetLastError());
  }

  // Scalars of the held range, all read back in one copy and one sync of the
  // side stream.  queries: g0 = last position of the held complete tiles,
  // g1 = nnz - 1
  int64_t ptr_first = 0, ptr_close = 0, eo_total = 0;
  const int64_t ic = pcs < tile_ptr_len ? pcs : tile_ptr_len - 1;
  const int64_t g0 = pcs > 0 ? tile_end * B - 1 : -1;
  const int64_t g1 = nnz > 0 ? nnz - 1 : -1;
  int64_t sv[4] = {-1, -1, -1, -1};
  int64_t hs[10];
  k_scalars<<<1, 64, 0, side>>>(h->row_ptr, m, g0, g1, h->tile_ptr, ic, h->eo_ptr, pcs, max_heads_d,
                               reinterpret_cast<const unsigned long long*>(scal + 4), single_head_d,
                               scal + 11);
  TRYC(cudaGetLastError());
  TRYC(cudaMemcpyAsync(hs, scal + 11, sizeof hs, cudaMemcpyDeviceToHost, side));
  TRYC(cudaStreamSynchronize(side));  // the transposition keeps running on `stream`
  trace.mark("scan");
  for (int q = 0; q < 4; ++q) sv[q] = hs[q];
  eo_total = hs[4];
  const int max_heads = (int)hs[5];
  const uint32_t tp0 = (uint32_t)hs[6], tpc = (uint32_t)hs[7];
  lines = (unsigned long long)hs[8];
  const int64_t single_head_tiles = hs[9];
  ptr_first = tp0 & 0x7fffffffu;
  ptr_close = tpc & 0x7fffffffu;
  TRY(dev_alloc(&h->eo, (size_t)eo_total, &alloc_ms, &bytes));
  if (pcs > 0 && eo_total > 0) {
    const int64_t threads = pcs * 32;
    k_eo<<<(unsigned)((threads + 255) / 256), 256, 0, side>>>(
        head_bits, h->tile_ptr, h->row_ptr, m, pcs, (int)sigma, pos0, h->eo_ptr, h->eo);
    TRYC(cudaGetLastError());
  }
  TRYC(cudaEventRecord(ev_join, side));
  t_alloc_stream = stream;
  trace.mark("eo");
  if (pcs > 0) h->lines_per_gather = (double)lines / (double)(samples * sigma);
  TRYC(cudaStreamWaitEvent(stream, ev_join, 0));  // join: eo, eo_ptr, work prefix

  // ---- SpMV plan ----
  const bool is_first = tile_begin == 0;
  h->first_row = ptr_first;
  h->first_owned = is_first || sv[2] >= pos0;
  h->last_row = pcs > 0 ? sv[0] : ptr_first;
  if (is_last) {
    h->tail_row_begin = tail > 0 ? ptr_close : (nnz > 0 ? sv[1] + 1 : 0);
    h->next_row_after = h->tail_row_begin;
  } else {
    h->tail_row_begin = m;
    h->next_row_after = ptr_close;
  }
  h->lead_rows = (is_first && nnz > 0) ? ptr_first : 0;
  h->tail_pos = pc * B;
  h->has_tail_item = is_last && tail > 0;
  int sms = 0;
  TRYC(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  h->max_heads = max_heads;  // with eo_total: may the plan drop the flag paths (NF)?
  h->maybe_long = single_head_tiles > 0;  // (NF plans exclude long rows)
  h->eo_entries = eo_total;
  h->info.sigma = sigma;  // spmv_plan picks the sigma-specialised kernel
  h->info.n = n;          // ... and sizes its shared memory by x
  TRY(spmv_plan(h, sms));
  // hot-column x staging for random plans whose x is several times the L2
  // (hotx.cu); such plans gather in lane order, so the plan is made again
  h->info.nnz_held = nnz_held;
  h->info.num_sms = sms;
  TRY(build_hot_plan(h, stream, &bytes));
  if (h->n_hot > 0) TRY(spmv_plan(h, sms));
  trace.mark("hot");
  const int64_t rows_total = h->lead_rows + (m - h->tail_row_begin);
  h->rows_blocks = rows_total > 0 ? (int)std::min<int64_t>((rows_total + 255) / 256, 2 * sms) : 0;
  const int64_t items = 2 * (int64_t)h->nwarps + 1;
  TRY(dev_alloc(&h->item_val, (size_t)items, &alloc_ms, &bytes));
  TRY(dev_alloc(&h->run_first, (size_t)items, &alloc_ms, &bytes));
  TRY(dev_alloc(&h->run_last, (size_t)items, &alloc_ms, &bytes));
  TRY(dev_alloc(&h->run_cnt, (size_t)items, &alloc_ms, &bytes));
  TRY(dev_alloc(&h->spill, (size_t)std::max(h->nwarps, 1) * (B + 1), &alloc_ms, &bytes));
  if (pcs > 0 && h->nwarps > 0) {
    TRY(dev_alloc(&h->warp_begin, (size_t)h->nwarps + 1, &alloc_ms, &bytes));
    auto* emax = reinterpret_cast<unsigned long long*>(scal + 6);  // zeroed with the block
    k_equal_split_max<<<(unsigned)((h->nwarps + 255) / 256), 256, 0, stream>>>(
        work_prefix, pcs, h->nwarps, emax);
    TRYC(cudaGetLastError());
    k_warp_bounds<<<(unsigned)((h->nwarps + 1 + 255) / 256), 256, 0, stream>>>(
        work_prefix, pcs, h->nwarps, emax, h->warp_begin);
    TRYC(cudaGetLastError());
    k_warp_bounds_fix<<<1, kFixThreads, 0, stream>>>(h->warp_begin, h->nwarps);
    TRYC(cudaGetLastError());
  }
  // long rows (possible only if some tile lies inside one row)
  if (pcs > 0 && single_head_tiles > 0) {
    const int64_t cap = single_head_tiles + 2;  // each long row covers a tile of its own
    h->long_cap = cap;
    TRY(dev_alloc(&h->lrow, (size_t)cap, &alloc_ms, &bytes));
    TRY(dev_alloc(&h->ltf, (size_t)cap, &alloc_ms, &bytes));
    TRY(dev_alloc(&h->lnp, (size_t)cap, &alloc_ms, &bytes));
    TRY(dev_alloc(&h->lbase, (size_t)cap + 1, &alloc_ms, &bytes));
    TRY(dev_alloc(&h->nlong_d, 2, &alloc_ms, &bytes));  // [0] long rows, [1] tail's long id
    TRY(dev_alloc(&h->ltag, (size_t)pcs, &alloc_ms, &bytes));
    const int64_t r_lo = ptr_first;
    const int64_t r_hi = std::max<int64_t>(r_lo, (is_last ? (nnz > 0 ? sv[1] : 0) : sv[0]) + 1);
    LongRowPred pred{h->row_ptr, B, pc};
    cub::CountingInputIterator<int64_t> rows_it(r_lo);
    size_t sel_bytes = 0;
    TRYC(cub::DeviceSelect::If(nullptr, sel_bytes, rows_it, h->lrow, h->nlong_d,
                               r_hi - r_lo, pred, stream));
    void* sel_tmp = nullptr;
    TRY(dev_alloc(reinterpret_cast<char**>(&sel_tmp), sel_bytes, &alloc_ms, &tmp_bytes));
    TRYC(cub::DeviceSelect::If(sel_tmp, sel_bytes, rows_it, h->lrow, h->nlong_d, r_hi - r_lo,
                               pred, stream));
    TRYC(cudaFreeAsync(sel_tmp, stream));
    k_long_info<<<(unsigned)((cap + 255) / 256), 256, 0, stream>>>(h->row_ptr, B, pc, h->lrow,
                                                                   h->nlong_d, cap, h->ltf,
                                                                   h->lnp);
    TRYC(cudaGetLastError());
    size_t scan_bytes = 0;
    TRYC(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, h->lnp, h->lbase, cap, stream));
    void* scan_tmp = nullptr;
    TRY(dev_alloc(reinterpret_cast<char**>(&scan_tmp), scan_bytes, &alloc_ms, &tmp_bytes));
    TRYC(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, h->lnp, h->lbase, cap, stream));
    TRYC(cudaFreeAsync(scan_tmp, stream));
    if (h->wide)
      k_long_tags<uint64_t><<<(unsigned)((pcs + 255) / 256), 256, 0, stream>>>(
          pcs, h->tile_ptr, (const uint64_t*)h->desc, h->eo_ptr, h->eo, (int)sigma, h->lrow,
          h->nlong_d, h->ltag);
    else
      k_long_tags<uint32_t><<<(unsigned)((pcs + 255) / 256), 256, 0, stream>>>(
          pcs, h->tile_ptr, (const uint32_t*)h->desc, h->eo_ptr, h->eo, (int)sigma, h->lrow,
          h->nlong_d, h->ltag);
    k_long_tail<<<1, 1, 0, stream>>>(h->tail_row_begin, h->has_tail_item ? 1 : 0, h->lrow,
                                     h->nlong_d, reinterpret_cast<int32_t*>(h->nlong_d + 1));
    TRYC(cudaGetLastError());
    h->long_slots = pcs + cap + 1;  // parts: one per tile it covers + its first tile + tail
    TRY(dev_alloc(&h->lparts, (size_t)h->long_slots, &alloc_ms, &bytes));
    TRY(dev_alloc(&h->lcnt, (size_t)cap, &alloc_ms, &bytes));
    TRYC(cudaMemsetAsync(h->lcnt, 0, sizeof(int32_t) * cap, stream));
  }
  // runs of the calibration items (the rows warps / the tail share)
  {
    const int n_items = 2 * h->nwarps + (h->has_tail_item ? 1 : 0);
    if (n_items > 0) {
      TRY(dev_alloc(&item_key, (size_t)n_items, &alloc_ms, &tmp_bytes));
      const unsigned kb = (unsigned)((n_items + 255) / 256);
      if (h->wide)
        k_item_keys<uint64_t><<<kb, 256, 0, stream>>>(
            h->warp_begin, h->tile_ptr, (const uint64_t*)h->desc, h->eo_ptr, h->eo, (int)sigma,
            h->nwarps, h->has_tail_item ? 1 : 0, h->tail_row_begin, h->lrow, h->nlong_d, item_key);
      else
        k_item_keys<uint32_t><<<kb, 256, 0, stream>>>(
            h->warp_begin, h->tile_ptr, (const uint32_t*)h->desc, h->eo_ptr, h->eo, (int)sigma,
            h->nwarps, h->has_tail_item ? 1 : 0, h->tail_row_begin, h->lrow, h->nlong_d, item_key);
      TRYC(cudaGetLastError());
      k_item_runs<<<1, kFixThreads, 0, stream>>>(item_key, n_items, h->run_first, h->run_last,
                                                 h->run_cnt, h->item_val);
      TRYC(cudaGetLastError());
    }
  }
  trace.mark("plan");

  // ---- info ----
  csr5g_info& in = h->info;
  in.m = m;
  in.n = n;
  in.nnz = nnz;
  in.omega = kOmega;
  in.sigma = sigma;
  in.p = p;
  in.p_complete = pc;
  in.tail_len = tail;
  in.tile_begin = tile_begin;
  in.tile_end = tile_end;
  in.has_tail = is_last && tail > 0;
  in.tile_ptr_bits = 32;
  in.word_bits = wb;
  in.y_offset_bits = yb;
  in.seg_offset_bits = sb;
  in.num_sms = sms;
  in.spmv_warps = h->nwarps;
  in.tile_ptr_len = tile_ptr_len;
  in.empty_offset_len = eo_total;
  in.nnz_held = nnz_held;
  in.metadata_bytes = tile_ptr_len * 4 + pcs * kOmega * (int64_t)wbytes;
  in.device_bytes = bytes;
  // nnz*(8+4) + 4(p+1) + W*32*pc + 4|eo| + 8n + 8m (per held range)
  in.spmv_bytes = nnz_held * 12 + tile_ptr_len * 4 + pcs * kOmega * (int64_t)wbytes +
                  eo_total * 4 + 8 * n + 8 * m;
  in.first_row = h->first_row;
  in.last_row = h->last_row;
  in.own_row_begin = is_first ? 0 : (h->first_owned ? h->first_row : h->first_row + 1);
  if (is_last) {
    in.own_row_end = m;
  } else {
    const bool close_starts_here = sv[3] >= tile_end * B;  // next shard owns its first row
    in.own_row_end = close_starts_here ? ptr_close : ptr_close + 1;
  }
  in.alloc_ms = alloc_ms;
  in.lines_per_gather = h->lines_per_gather;
  in.warps_per_cta = h->warps_per_block;
  in.stages = h->stages;
  in.smem_bytes = h->smem_bytes;
  in.x_mode = h->x_mode;
  in.x_window = h->x_window ? 1 : 0;
  in.kernel_variant = h->vr ? 1 : (h->nf ? 2 : 0);
  in.hot_cols = h->n_hot;
  in.hot_coverage = h->hot_coverage;
  // the build is synchronous (format.hpp:182 returns a finished value): the
  // handle is usable from any stream once it returns
  TRYC(cudaStreamSynchronize(stream));
  in.long_rows = 0;
  if (h->nlong_d)
    TRYC(cudaMemcpy(&in.long_rows, h->nlong_d, sizeof(int64_t), cudaMemcpyDeviceToHost));
  trace.mark("final");
  in.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
  *out = h;
  return cleanup(CSR5G_OK);
#undef TRY
#undef TRYC
}

int launch_to_csr(Handle* h, int32_t* d_col, double* d_val, cudaStream_t stream) {
  CSR5G_CUDA(cudaSetDevice(h->device));
  const int64_t tiled = h->pcs * h->B;
  if (tiled > 0) {
    k_untranspose<<<(unsigned)((tiled + 255) / 256), 256, 0, stream>>>(h->col, h->val, d_col, d_val,
                                                                        tiled, (int)h->info.sigma);
    CSR5G_CUDA(cudaGetLastError());
  }
  const int64_t rest = h->info.nnz_held - tiled;
  if (rest > 0) {
    CSR5G_CUDA(cudaMemcpyAsync(d_col + tiled, h->col + tiled, sizeof(int32_t) * rest,
                               cudaMemcpyDeviceToDevice, stream));
    CSR5G_CUDA(cudaMemcpyAsync(d_val + tiled, h->val + tiled, sizeof(double) * rest,
                               cudaMemcpyDeviceToDevice, stream));
  }
  return CSR5G_OK;
}

}  // namespace csr5g
