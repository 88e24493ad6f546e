// internal.cuh -- shared types and device helpers of libcsr5g.so.
//
// Layout in HBM (one handle; sizes for the held complete tiles k in [0, pcs)):
//   row_ptr   int64 [m+1]          copy of the global CSR row pointer
//   tile_ptr  u32   [tile_ptr_len] bit 31 = empty-row flag, low 31 = first row
//   tile_desc W     [pcs*32]       W = u32 (sigma <= 17) or u64; lane-major per tile
//   eo_ptr    int64 [pcs+1]        empty_offset list bounds (flagged tiles only)
//   eo        int32 [E]            row offsets per segment head of flagged tiles
//   col_idx   int32 [nnz_held]     tile-transposed: (col i, depth j) at k*B + j*32 + i
//   val       f64   [nnz_held]     same order; tail (last shard) stays in CSR order
// The transposed order makes every depth step of a tile one fully coalesced
// 128 B (col) + 256 B (val) warp access.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/csr5g.h"

namespace csr5g {

constexpr int kOmega = 32;
constexpr int kSegBits = 5;  // ceil_log2(32), descriptor.cpp:22-36
constexpr int kSpmvThreads = 256;
constexpr int kSpmvWarpsPerBlock = kSpmvThreads / 32;
constexpr uint32_t kFull = 0xffffffffu;

// Peer copies of y (p2p.cu, fused iterative y -> x): every final y value is
// also stored into each peer's next-x buffer over NVLink.  skip_row: a row
// whose value here is still partial (an owner's boundary row before the
// fix-up, which mirrors the total itself).
constexpr int kMaxMirror = 7;  // one NVSwitch box: 8 GPUs
// mc: the NVLS multicast mapping of every rank's next-x buffer (p2p.cu): one
// multimem store reaches all of them through the switch, instead of n peer
// stores over NVLink.
struct Mirrors {
  double* p[kMaxMirror];
  int32_t n;
  int64_t skip_row;
  double* mc;
};

__host__ __device__ __forceinline__ bool mir_on(const Mirrors& m) { return m.n != 0 || m.mc != nullptr; }

__device__ __forceinline__ void mirror_store(const Mirrors& m, int64_t r, double v) {
  if (m.mc) {
    asm volatile("multimem.st.global.f64 [%0], %1;" ::"l"(m.mc + r), "d"(v) : "memory");
    return;
  }
#pragma unroll
  for (int g = 0; g < kMaxMirror; ++g)
    if (g < m.n) m.p[g][r] = v;
}

// Everything the SpMV kernels read, passed by value.
struct SpmvArgs {
  const int64_t* row_ptr;
  const uint32_t* tile_ptr;
  const void* desc;
  const int64_t* eo_ptr;
  const int32_t* eo;
  const int32_t* col;
  const double* val;
  const double* x;
  double* y;
  double* item_val;        // run partials (deterministic mode), per stream
  const int32_t* run_first;  // item i's run of equal rows is items [run_first[i], run_last[i]]
  const int32_t* run_last;
  int32_t* run_cnt;        // arrivals per run (indexed by its first item), per stream
  csr5g_partial* send;
  uint32_t* send_flag;     // p2p.cu: owner's ready flag for the send record (or null)
  uint32_t send_epoch;
  double* spill;           // per-warp overflow slots for closed segment sums
  const int64_t* warp_begin;  // warp w holds tiles [warp_begin[w], warp_begin[w+1])
  int64_t pcs;             // complete tiles held
  int64_t pos0;            // global nonzero position of local index 0
  int64_t next_row_after;  // first row after the last held complete tile's range
  int64_t lead_rows;       // rows [0, lead_rows) are empty and zeroed here
  int64_t tail_row_begin;  // rows [tail_row_begin, m) computed from the tail here
  int64_t tail_pos;        // global position where the tail starts (pc*B)
  int64_t m;
  int64_t tile_ptr_len;
  int64_t first_row;       // row of head 0 of the first held tile
  int32_t first_owned;     // that row starts inside this handle
  int32_t has_tail_item;   // tail exists: its first row is item 2*nwarps
  int32_t sigma;
  int32_t B;
  int32_t nwarps;          // tile warps (each a contiguous tile range)
  int32_t stages;          // TMA ring depth per warp
  int32_t stage_bytes;     // one tile: val | col_idx | descriptor words
  int32_t bar_bytes;       // mbarrier area at the start of shared memory
  int32_t atomic;          // SpmvMode::atomic
  int32_t x_mode;          // x gather path: 0 L1+evict_last, 1 L1 no-allocate+evict_last,
                           // 2 LSU, 3 .cg, 4 plain .nc, 5 = 1 with a 64 B L2 prefetch,
                           // 6 = 4 with 64 B, 7 / 8 = 1 / 5 in CSR order (VR only)
  int32_t stream_only;     // profiling: run the TMA ring without gathers/math
  int32_t early_gather;    // random gathers: issue tile k+1's gathers before tile k's depth loop
  float x_frac;            // share of x lines given evict_last (the rest evict_first)
  int32_t y_hint;          // y stores: 1 = L2 evict_first, no L1 allocation
  Mirrors mir;             // fused iterative mode: peer next-x buffers (n = 0: none)
  // long rows (three or more parts; convert.cu "long rows"), deterministic mode
  int32_t has_long;        // the handle may hold long rows
  int64_t t0;              // global index of the first held tile
  const int32_t* ltag;     // per tile: (b << 2) | head-0 row long | last row long << 1
  const int64_t* lrow;     // per long id: row, first tile, parts, first slot
  const int64_t* ltf;
  const int64_t* lnp;
  const int64_t* lbase;
  const int32_t* tail_long;  // long id of the tail's first row, or -1
  double* lparts;          // part slots (per stream)
  int32_t* lcnt;           // arrivals per long row (per stream; reset by the last)
  int64_t trace_tile;      // trace launch (csr5g_spmv_tile): the tile and its outputs
  int64_t* trace_row;
  double* trace_val;
  int32_t* trace_count;
  // hot-column x staging (hotx.cu): a.col holds the execution col_idx, whose
  // negative entries c address xh[~c] (the hot columns' x values, refreshed
  // per SpMV); the others address x[c] with the cold policy
  const double* xh;
  int32_t cold_pol;        // cold gathers: 0 evict_first, 1 evict_normal, 2 evict_last
  int32_t hot_l1;          // hot gathers allocate in L1
  int32_t pdl;             // launched as a programmatic dependent of k_xhot_fill
  int32_t nf2_slots;       // k_spmv_nf2: closed-segment slots per tile
};

struct Pipeline;  // pipeline.cu: host-vector copy/compute pipeline

// Per-stream SpMV scratch (the reference's per-worker workspaces,
// spmv.hpp:27-38): concurrent spmv calls on one handle from distinct streams
// each get their own run items and closed-segment spill area.
struct StreamScratch {
  cudaStream_t stream;
  double* item_val;
  int32_t* run_cnt;
  double* spill;
  double* lparts = nullptr;  // long-row part slots and arrival counters
  int32_t* lcnt = nullptr;
  double* xh = nullptr;        // hot-column x values (hotx.cu), per stream
  cudaEvent_t done = nullptr;  // recorded after the last SpMV that used it
  uint64_t last_use = 0;       // LRU stamp
  bool owned = true;           // false: the handle's own arrays (freed with it)
};
constexpr size_t kMaxStreamScratch = 8;  // scratch sets per handle (LRU beyond)
struct Binding;   // p2p.cu: a shard's NVLink boundary exchange

struct Handle {
  int device = 0;
  csr5g_info info{};
  bool wide = false;  // 64-bit descriptor words
  int64_t pcs = 0, t0 = 0, B = 0;
  int64_t* row_ptr = nullptr;
  uint32_t* tile_ptr = nullptr;
  void* desc = nullptr;
  int64_t* eo_ptr = nullptr;
  int32_t* eo = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
  double* item_val = nullptr;
  int32_t* run_first = nullptr;  // static run structure of the items (built once)
  int32_t* run_last = nullptr;
  int32_t* run_cnt = nullptr;    // zeroed; every launch leaves it zeroed
  csr5g_partial* send = nullptr;
  csr5g_partial* send_ext = nullptr;  // caller-provided record slot
  uint32_t* send_flag = nullptr;      // p2p.cu: owner's ready flag for this shard's record
  uint32_t send_epoch = 0;            // value stored into send_flag by the current call
  Mirrors mir{};                      // p2p.cu: peer copies of y for the current call
  Binding* mg = nullptr;              // p2p.cu: NVLink boundary exchange of this shard
  double* spill = nullptr;            // nwarps * (B + 1) doubles
  int64_t* warp_begin = nullptr;      // nwarps + 1 tile-range bounds, split by tile work
  int64_t next_row_after = 0, lead_rows = 0, tail_row_begin = 0, tail_pos = 0;
  int64_t first_row = 0, last_row = 0;
  bool first_owned = true, is_last = true, has_tail_item = false;
  int nwarps = 0, tile_blocks = 0, rows_blocks = 0;
  double lines_per_gather = 1.0;  // sampled x-gather locality (1 = coalesced, 32 = random)
  int x_mode = 0;                 // gather path chosen by the plan
  bool x_window = false;          // L2 persisting window on x
  bool vr = false;                // values outside the TMA ring (k_spmv<SIG, true>)
  bool nf = false;                // no flagged tile, heads fit the slots (k_spmv<SIG, false, true>)
  int max_heads = 0;              // most segment heads in one tile
  // long rows (convert.cu "long rows"): ids, per-tile tags, per-row info
  bool maybe_long = false;
  int64_t long_cap = 0, long_slots = 0;
  int64_t *lrow = nullptr, *ltf = nullptr, *lnp = nullptr, *lbase = nullptr, *nlong_d = nullptr;
  int32_t* ltag = nullptr;
  double* lparts = nullptr;  // the first stream's part slots / counters
  int32_t* lcnt = nullptr;
  int64_t eo_entries = 0;         // empty_offset entries
  // hot-column x staging (hotx.cu): the execution copy of col_idx (hot
  // columns renumbered to ~rank), the hot columns in ascending order, and the
  // first stream's staged x values; n_hot = 0: no staging (col_x = col)
  int32_t* col_x = nullptr;
  int32_t* hot_cols = nullptr;
  double* xh = nullptr;
  int64_t n_hot = 0;
  double hot_coverage = 0.0;      // sampled share of gathers that hit a hot column
  int hot_threshold = 0;          // sampled count a hot column reaches
  int cold_pol = 0;               // cold gathers' L2 policy (SpmvArgs::cold_pol)
  int hot_l1 = 0;                 // hot gathers allocate in L1 (SpmvArgs::hot_l1)
  int gm = 0;                     // compile-time gather mode of the plan's kernel (k_spmv GM)
  bool nf2 = false;               // NF plan on the two-tiles-per-iteration kernel (spmv_nf2.cuh)
  int nf2_slots = 0;
  int warps_per_block = 0, stages = 0, stage_bytes = 0, bar_bytes = 0, smem_bytes = 0;
  int carveout_pct = -1;  // preferred shared-memory carveout of the SpMV kernel
  // per-stream SpMV scratch (the handle's own arrays are the first set);
  // guarded by scratch_mu
  std::vector<StreamScratch> scratch;
  uint64_t scratch_clock = 0;
  std::mutex scratch_mu;
  Pipeline* pipe = nullptr;  // created by the first host-vector SpMV
  std::mutex pipe_mu;        // host-vector calls from several threads enqueue one at a time
};

// ---- errors --------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
int resolve_device(int* device);  // device < 0: the current device

#define CSR5G_CUDA(call)                                   \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return ::csr5g::cuda_fail(e_, #call); \
  } while (0)

// ---- launchers implemented in convert.cu / spmv.cu -------------------------
int build_handle(int device, int64_t m, int64_t n, int64_t nnz, const int64_t* d_row_ptr,
                 const int32_t* d_col_idx, const double* d_val, const csr5g_params* params,
                 int64_t tile_begin, int64_t tile_end, bool shard, int with_tail,
                 cudaStream_t stream, Handle** out);
void free_handle(Handle* h);
int launch_spmv(Handle* h, const double* d_x, double* d_y, int mode, cudaStream_t stream,
                cudaEvent_t ev0, cudaEvent_t ev1);
int launch_fixup(Handle* h, const csr5g_partial* d_all, int world, int rank, double* d_y,
                 cudaStream_t stream);
int launch_to_csr(Handle* h, int32_t* d_col, double* d_val, cudaStream_t stream);
int launch_tile_trace(Handle* h, int64_t k, const double* d_x, int64_t* d_rows, double* d_vals,
                      int32_t* d_count, cudaStream_t stream);
int spmv_plan(Handle* h, int sms);
int build_hot_plan(Handle* h, cudaStream_t stream, int64_t* bytes);
int launch_xhot_fill(Handle* h, const double* d_x, double* d_xh, cudaStream_t stream);
int func_attrs(const void* fn, int device, int smem, int carve);
int scratch_done(Handle* h, cudaStream_t stream);
int scratch_for(Handle* h, cudaStream_t stream, double** iv, int32_t** rc, double** sp,
                double** lp, int32_t** lc, double** xh);
int spmv_host_batch(Handle* h, const double* const* xs, double* const* ys, int64_t count,
                    int mode, cudaStream_t stream);
void free_pipeline(Pipeline* p);
void free_binding(Binding* b);
int csr_spmv(int device, int kernel, int64_t m, int64_t n, int64_t nnz, const int64_t* rp,
             const int32_t* col, const double* val, const double* x, double* y,
             cudaStream_t stream);

// ---- device helpers ----------------------------------------------------------
// TMA bulk copies with mbarrier completion (tile kernel, transposition)
__device__ __forceinline__ uint32_t saddr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(saddr(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}

// One TMA bulk copy global -> shared, completion counted on `bar`.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar)), "l"(pol)
      : "memory");
}

// arm `bar` for `bytes` of bulk copies (one arrival)
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// evict_last for a fraction of the lines (chosen by address), evict_first for
// the rest: a working set larger than L2 keeps a resident part instead of
// thrashing all of it
__device__ __forceinline__ uint64_t policy_evict_last_frac(float f) {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(p) : "f"(f));
  return p;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol)
               : "memory");
}
// Streaming read-once loads: no L1 allocation, evict-first in L2.
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t ld_stream(const uint64_t* p, uint64_t pol) {
  uint64_t v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
// x gathers: L1-cached, evict-last in L2 so the streamed matrix does not push x out.
__device__ __forceinline__ double ld_keep(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// x gathers that skip L1 allocation (random gathers with no reuse in L1).
__device__ __forceinline__ double ld_keep_na(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// x gathers through the coherent LSU path (not the read-only/texture path).
__device__ __forceinline__ double ld_x_lsu(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
// plain read-only gather: no L2 policy operand (saves the uniform-register
// moves a cache_hint needs per load)
__device__ __forceinline__ double ld_x_plain(const double* p) {
  double v;
  asm("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
// Random gathers with a 64-byte L2 prefetch size: without the qualifier a
// random 8-byte load moves ~2.4 sectors from DRAM, with it ~1.5
// (tools/sector_probe.cu, profiles/r02_sector_probe.txt).
__device__ __forceinline__ double ld_keep_na64(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::64B.f64 %0, [%1], %2;"
      : "=d"(v)
      : "l"(p), "l"(pol));
  return v;
}
// Hot-column split gathers (hotx.cu): c < 0 reads the staged hot value
// xh[~c] (kept in L2 with ph), c >= 0 the original x[c] (policy pc).
__device__ __forceinline__ double ld_x_split(const double* x, const double* xh, int32_t c,
                                             uint64_t ph, uint64_t pc) {
  const bool hot = c < 0;
  const double* p = hot ? xh + ~c : x + c;
  const uint64_t pol = hot ? ph : pc;
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_x_split64(const double* x, const double* xh, int32_t c,
                                               uint64_t ph, uint64_t pc) {
  const bool hot = c < 0;
  const double* p = hot ? xh + ~c : x + c;
  const uint64_t pol = hot ? ph : pc;
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::64B.f64 %0, [%1], %2;"
      : "=d"(v)
      : "l"(p), "l"(pol));
  return v;
}
// the same, hot values allocated in L1 (the hottest columns come first in xh
// and are re-read by every warp of the SM; an extra rank test to allocate
// only the hottest measured slower, 13.9 vs 13.0 ms on R-MAT s27)
template <bool PF64>
__device__ __forceinline__ double ld_x_split_l1(const double* x, const double* xh, int32_t c,
                                                uint64_t ph, uint64_t pc) {
  double v;
  if (c < 0) {
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(xh + ~c), "l"(ph));
  } else if (PF64) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::64B.f64 %0, [%1], %2;"
        : "=d"(v)
        : "l"(x + c), "l"(pc));
  } else {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(x + c), "l"(pc));
  }
  return v;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_x_plain64(const double* p) {
  double v;
  asm("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_x_cg(const double* p) {
  double v;
  asm("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// upper_bound over row_ptr[lo, hi): first index with row_ptr[idx] > g (hi if none).
__device__ __forceinline__ int64_t upper_bound_dev(const int64_t* __restrict__ rp, int64_t lo,
                                                   int64_t hi, int64_t g) {
  while (lo < hi) {
    const int64_t mid = lo + ((hi - lo) >> 1);
    if (rp[mid] <= g)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// format.cpp:42-50 row_of_nonzero over the full row_ptr (m+1 entries).
__device__ __forceinline__ int64_t row_of_nonzero_dev(const int64_t* __restrict__ rp, int64_t m,
                                                      int64_t g) {
  if (m <= 0) return 0;
  int64_t r = upper_bound_dev(rp, 0, m + 1, g) - 1;
  r = r < 0 ? 0 : r;
  return r > m - 1 ? m - 1 : r;
}

}  // namespace csr5g
