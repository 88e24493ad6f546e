// spmv_kernel.cuh -- the CSR5 SpMV tile kernel template k_spmv<SIGMA, VR, NF,
// TR> (reference: spmv.cpp:42-124, 224-298), included by the instantiation
// units spmv_inst_*.cu (one per variant, compiled in parallel) and
// dispatched by spmv.cu.
//
// k_spmv<SIGMA>: persistent grid (one CTA per SM), one warp = one contiguous
//   range of tiles (CSR5 tiles are equal-work units, so a static split
//   balances).  Specialised per sigma so the depth loop is fully unrolled.
//   * TMA ring: each warp streams its tiles through an S-stage shared-memory
//     ring with bulk copies (cp.async.bulk, completion on one mbarrier per
//     stage).  A tile's val (B*8 bytes), col_idx (B*4) and descriptor words
//     (32*W) are contiguous in HBM thanks to the CSR5 transposition, so a tile
//     is three bulk copies issued by lane 0, S-1 tiles ahead of the one being
//     computed: the matrix stream never waits on the dependent x gathers.
//   * Depth loop (Algorithm 8, spmv.cpp:61-95, lane i = column i): all x
//     gathers of the tile are issued first (L1/L2, evict-last), then sigma
//     FMAs; a warp-uniform test on the OR of the lanes' bit flags guards the
//     rare segment-close path, which only writes the closed sum to a per-warp
//     shared-memory slot indexed by its segment head.
//   * Splice (fast segmented sum, spmv.cpp:97-105): 5-step shuffle segmented
//     suffix scan over a ballot of head-bearing lanes -- no scan-and-subtract.
//   * Write-back: lanes walk the tile's heads in order (coalesced
//     empty_offset reads, near-coalesced y stores) and zero the empty rows
//     between heads.  Rows wholly inside the warp's range are final; only the
//     first and last row runs of a warp can be shared, so each warp emits two
//     (row, partial) items.
//   * Before its tiles every thread takes a grid-stride share of the "rows
//     part": CSR tail rows (spmv.cpp:110-124), leading/trailing empty rows.
// Calibration (spmv.cpp:224-298) happens inside the same kernel: the items of
//   a row shared between warps (or with the tail) form a run known at build
//   time (k_item_runs); the last writer of a run sums its partials in item
//   order and writes the row (resolve_item).  Atomic mode instead adds items
//   with fp64 atomics into a zeroed y (spmv.cpp:273-295).
#pragma once

#include <type_traits>

#include "internal.cuh"

namespace csr5g {
namespace {

__device__ __forceinline__ void sts_if(int32_t* p, int32_t v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t@p st.shared.b32 [%0], %1;\n\t}" ::"r"(
          saddr(p)),
      "r"(v), "r"((int)pred)
      : "memory");
}

template <bool LONG = true>
__device__ void resolve_item(const SpmvArgs& a, int64_t idx, int64_t row, double v);
__device__ __forceinline__ void long_arrive_thread(const SpmvArgs& a, int64_t L, int cnt);

// Tail rows and leading/trailing empty rows, grid-stride over all threads.
template <bool LONG>
__device__ void rows_part(const SpmvArgs& a) {
  const int64_t tail_rows = a.m - a.tail_row_begin;
  const int64_t total = a.lead_rows + tail_rows;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    if (idx < a.lead_rows) {
      a.y[idx] = 0.0;
      if (mir_on(a.mir)) mirror_store(a.mir, idx, 0.0);
      continue;
    }
    const int64_t r = a.tail_row_begin + (idx - a.lead_rows);
    int64_t lo = a.row_ptr[r];
    const int64_t hi = a.row_ptr[r + 1];
    if (lo < a.tail_pos) lo = a.tail_pos;
    double s = 0.0;
    for (int64_t q = lo; q < hi; ++q) s = fma(a.val[q - a.pos0], a.x[a.col[q - a.pos0]], s);
    if (a.has_tail_item && r == a.tail_row_begin) {
      const int64_t L = LONG && a.has_long ? (int64_t)*a.tail_long : -1;
      if (L >= 0) {  // the last part of a long row
        a.lparts[a.lbase[L] + a.lnp[L] - 1] = s;
        long_arrive_thread(a, L, 1);
      } else {
        resolve_item<LONG>(a, 2 * (int64_t)a.nwarps, r, s);
      }
    } else {
      a.y[r] = s;
      if (mir_on(a.mir)) mirror_store(a.mir, r, s);
    }
  }
}

__device__ __forceinline__ uint64_t warp_or64(uint64_t v) {
  const uint32_t lo = __reduce_or_sync(kFull, (uint32_t)v);
  const uint32_t hi = __reduce_or_sync(kFull, (uint32_t)(v >> 32));
  return ((uint64_t)hi << 32) | lo;
}

// The send record goes to local memory (collective exchange) or straight into
// the owner rank's mailbox over NVLink (p2p.cu), followed there by its ready
// flag: value stores, system-scope fence, then the flag store with release.
__device__ __forceinline__ void write_run(int64_t row, double v, double* y, int64_t first_row,
                                          int first_owned, csr5g_partial* send, uint32_t* flag,
                                          uint32_t epoch, const Mirrors& mir) {
  if (!first_owned && row == first_row) {
    send->row = row;
    send->value = v;
    if (flag) {
      __threadfence_system();
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag), "r"(epoch) : "memory");
    }
  } else {
    y[row] = v;
    if (mir_on(mir) && row != mir.skip_row) mirror_store(mir, row, v);
  }
}

// In-kernel calibration (deterministic mode).  Rows wholly inside a warp's
// tile range are final in the warp; only its first and last row runs can be
// shared, so it emits two items (2w, 2w+1; the tail's first row is item
// 2*nwarps).  Their rows are fixed by the structure, so the build records for
// every item the run of equal rows it belongs to (k_item_runs).  The writer of
// an item stores its partial, fences and counts an arrival on the run; the
// last arrival sums the run's partials in item order (deterministic whatever
// the arrival order), resets the counter for the next launch and writes the
// row (y, or the shard's send record, spmv.cpp:267-272).  No second kernel.
// A run of two partials (the common case: a row shared by two neighbouring
// warps) needs no fence or counter: both writers exchange their value through
// one 64-bit atomic on the run's slot, and the second adds the two (a + b is
// b + a bit for bit).  The slot's idle value is all ones, a NaN that no
// arithmetic produces (results are the canonical NaN); the second writer
// restores it for the next launch.
constexpr unsigned long long kSlotIdle = ~0ull;

// A NaN partial is exchanged as the canonical NaN, whose bits differ from the
// idle pattern whatever payload the NaN carried.
__device__ __forceinline__ double exchangeable(double v) {
  return v != v ? __longlong_as_double(0x7ff8000000000000ll) : v;
}

__device__ __forceinline__ bool pair_exchange(const SpmvArgs& a, int s, double v, double* total) {
  v = exchangeable(v);
  auto* slot = reinterpret_cast<unsigned long long*>(a.item_val + s);
  const unsigned long long old = atomicExch(slot, (unsigned long long)__double_as_longlong(v));
  if (old == kSlotIdle) return false;
  *slot = kSlotIdle;
  *total = __longlong_as_double((long long)old) + v;
  return true;
}

// The sum of a long run's partials, items s..e, in one fixed order whichever
// thread finishes the run: lane l of a warp sums items s+l, s+l+32, ... in
// turn, then an xor butterfly (resolve_item_warp); a single thread
// (resolve_item, e.g. the tail's) replays exactly that order.
__device__ __noinline__ double sum_fixed_order(const double* p, int64_t n) {
  double t[32];
#pragma unroll
  for (int l = 0; l < 32; ++l) {
    t[l] = 0.0;
    for (int64_t j = l; j < n; j += 32) t[l] += __ldcg(p + j);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    double n[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) n[l] = t[l] + t[l ^ d];
#pragma unroll
    for (int l = 0; l < 32; ++l) t[l] = n[l];
  }
  return t[0];
}

// Long rows (convert.cu "long rows"): every part of the row sits in its slot;
// `cnt` more parts have been stored by the caller (a warp, lane 0; or one
// thread for the tail's part).  The arrival that completes the row sums its
// parts in sum_fixed_order's order -- the warp version below does the same
// additions -- and writes it.
__device__ __forceinline__ void long_arrive_thread(const SpmvArgs& a, int64_t L, int cnt) {
  __threadfence();
  if (atomicAdd(a.lcnt + L, cnt) + cnt != (int)a.lnp[L]) return;
  __threadfence();
  const double t = sum_fixed_order(a.lparts + a.lbase[L], a.lnp[L]);
  a.lcnt[L] = 0;
  write_run(a.lrow[L], t, a.y, a.first_row, a.first_owned, a.send, a.send_flag, a.send_epoch,
            a.mir);
}

__device__ __forceinline__ void long_arrive_warp(const SpmvArgs& a, int64_t L, int cnt, int lane) {
  const int64_t n = a.lnp[L];
  if (cnt == n) {
    __syncwarp();  // every part is this warp's (lane 0's stores): no count needed
  } else {
    int last = 0;
    if (lane == 0) {
      __threadfence();  // this warp's part stores (lane 0) before the count
      last = atomicAdd(a.lcnt + L, cnt) + cnt == (int)n;
    }
    if (!__shfl_sync(kFull, last, 0)) return;
    __threadfence();
  }
  const double* p = a.lparts + a.lbase[L];
  double t = 0.0;
  for (int64_t j = lane; j < n; j += 32) t += __ldcg(p + j);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(kFull, t, d);
  if (lane == 0) {
    if (cnt != n) a.lcnt[L] = 0;
    write_run(a.lrow[L], t, a.y, a.first_row, a.first_owned, a.send, a.send_flag, a.send_epoch,
              a.mir);
  }
}

// LONG = false (NF plans: no row covers a whole tile, so no run has more
// than two items) leaves the three-or-more path, and its call, out.
template <bool LONG>
__device__ void resolve_item(const SpmvArgs& a, int64_t idx, int64_t row, double v) {
  if (a.atomic) {  // spmv.cpp:273-295: fp64 atomics into the zeroed y
    if (v != 0.0) atomicAdd(a.y + row, v);
    return;
  }
  const int s = a.run_first[idx], e = a.run_last[idx];
  double t = v;
  if (e == s + 1) {
    if (!pair_exchange(a, s, v, &t)) return;
  } else if (e > s) {
    __stcg(a.item_val + idx, v);
    __threadfence();
    if (atomicAdd(a.run_cnt + s, 1) != e - s) return;
    __threadfence();
    if (LONG) {
      t = sum_fixed_order(a.item_val + s, e - s + 1);
    } else {
      t = 0.0;
      for (int j = s; j <= e; ++j) t += __ldcg(a.item_val + j);
    }
    a.run_cnt[s] = 0;
  }
  write_run(row, t, a.y, a.first_row, a.first_owned, a.send, a.send_flag, a.send_epoch, a.mir);
}

// The same, called by a whole warp (idx, row, v uniform): the last arrival's
// warp sums a long run 32 items at a time (fixed tree, deterministic).
__device__ __forceinline__ void resolve_item_warp(const SpmvArgs& a, int64_t idx, int64_t row,
                                                  double v, int lane) {
  const int s = a.atomic ? 0 : a.run_first[idx], e = a.atomic ? 0 : a.run_last[idx];
  if (a.atomic || e <= s + 1) {  // single partial, pair exchange, or atomic mode
    if (lane == 0) resolve_item(a, idx, row, v);
    return;
  }
  int last = 0;
  if (lane == 0) {
    __stcg(a.item_val + idx, v);
    __threadfence();
    last = atomicAdd(a.run_cnt + s, 1) == e - s;
  }
  if (!__shfl_sync(kFull, last, 0)) return;
  __threadfence();
  double t = 0.0;
  for (int j = s + lane; j <= e; j += 32) t += __ldcg(a.item_val + j);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(kFull, t, d);
  if (lane == 0) {
    a.run_cnt[s] = 0;
    write_run(row, t, a.y, a.first_row, a.first_owned, a.send, a.send_flag, a.send_epoch, a.mir);
  }
}

}  // namespace

// Warps per CTA: short tiles need fewer registers and less shared memory per
// warp, and random gathers want as many warps in flight as fit.  sigma <= 5:
// 20 warps (96 registers, no spills) beat 24 (80 registers, spills and
// rematerialised addresses): Laplacian 1000^2 35.2 -> 33.5 us.
__host__ __device__ constexpr int spmv_threads(int sigma) {
  return sigma <= 5 ? 640 : sigma <= 13 ? 512 : sigma <= 32 ? 384 : 256;
}
__host__ __device__ constexpr int spmv_threads_nf(int sigma) {
  return sigma <= 5 ? 768 : spmv_threads(sigma);  // 80 registers suffice without the flag paths
}
#ifndef CSR5G_VR_GM_THREADS16
#define CSR5G_VR_GM_THREADS16 512
#endif
// VR kernels with a compile-time gather mode (fewer registers than the
// runtime switch)
__host__ __device__ constexpr int spmv_threads_vr_gm(int sigma) {
  return sigma <= 16 && sigma > 13 ? CSR5G_VR_GM_THREADS16 : spmv_threads(sigma);
}
__host__ __device__ constexpr int spmv_threads_of(int sigma, bool vr, bool nf, int gm) {
  return nf ? spmv_threads_nf(sigma) : (vr && gm != 0) ? spmv_threads_vr_gm(sigma) : spmv_threads(sigma);
}
// closed-segment slots per warp in shared memory (tiles rarely have more heads)
constexpr int kClosedSlots = 128;
constexpr int kEoSlots = 128;  // >= kClosedSlots - 1 heads of a shared-slot tile
constexpr int kVrMaxSigma = 24;  // VR variants are instantiated up to this sigma

// Outside the anonymous namespace: the sigma instantiations are reached
// through a function-pointer switch, and the runtime must register each one.
// VR ("values in registers", random-gather plans, sigma <= kVrMaxSigma): the
// ring carries only col_idx and the descriptor words; a tile's values are
// loaded coalesced straight into registers together with its x gathers, so a
// warp's ring is a third of the size and more of the SM's L1 stays free for
// outstanding gather misses.
// NF ("no flags"): the plan proved that no tile is flagged and every tile's
// heads fit the shared-memory slots (Laplacian-like matrices), so the
// empty_offset staging, the spill path and the empty-row zeroing compile out.
// TR ("trace", test hook csr5g_spmv_tile): one warp runs the general kernel on
// the single tile a.trace_tile and records every head's final value (its
// contribution, spmv.cpp:211-222) instead of writing y.
// GM (gather mode) fixes the plan's x load path at compile time, so the tile
// loop carries no per-tile mode branches: 1 = VR lane order, no L1 allocation
// (x_mode 1); 2 = VR CSR order with the 64-byte prefetch (x_mode 8); 3 = VR
// hot-column staging, hot values L1-allocated, cold ones 64-byte prefetched
// (x_mode 5 + hot_l1); 4 = plain read-only loads (x_mode 4, local plans);
// 5 = VR hot-column staging, lane order, no L1 allocation, no prefetch
// (x_mode 1 without hot_l1).
// GM = 0 keeps the runtime switch over every x_mode (experiments, trace).
template <int SIG, bool VR, bool NF = false, bool TR = false, int GM = 0>
__global__ void __launch_bounds__(spmv_threads_of(SIG, VR, NF, GM), 1)
    k_spmv(SpmvArgs a) {
  using W = typename std::conditional<(SIG <= 17), uint32_t, uint64_t>::type;
  constexpr int B = 32 * SIG;
  constexpr int CH = SIG <= 32 ? SIG : (SIG + 1) / 2;  // x gathers in flight per lane
  static_assert(!VR || CH == SIG, "VR needs the whole tile's gathers in one batch");
  constexpr int CAPC = B < kClosedSlots ? B : kClosedSlots;
  constexpr uint64_t FMASK = (1ull << SIG) - 1;
  // GM 4 (local plans) compiles the profiling knobs (stream_only, y_hint)
  // out, and early gathers, which only random non-VR plans use: Laplacian
  // 24.8 -> 22.7 us, st27 0.442 -> 0.435 ms.  The VR kernels keep them --
  // without them R-MAT s24 measured slower (1.42 vs 1.27 ms, GM 5), an
  // effect of the compiler's schedule, not of the knobs' work.
  constexpr bool KNOBS = GM != 4;
  constexpr bool EARLY_OK = !VR && SIG <= 18 && GM != 4;  // a second x array fits in registers
  constexpr uint32_t COL_OFF = VR ? 0 : B * 8, DESC_OFF = COL_OFF + B * 4;
  constexpr uint32_t TILE_BYTES = DESC_OFF + 32 * sizeof(W);

  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (!TR && a.first_owned && !a.atomic && blockIdx.x == 0 && threadIdx.x == 0) {
    a.send->row = -1;  // this handle has no partial to send
    a.send->value = 0.0;
  }
  const int NW = blockDim.x >> 5;
  const int S = a.stages;
  const int w = blockIdx.x * NW + wib;
  const bool has_tiles = w < a.nwarps;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + wib * S;
  // closed-segment slots (slot h + 1 = head h): in shared memory when a tile's
  // H + 1 slots fit in CAPC, else (tiles of very short rows) all of them in a
  // per-warp global spill area
  double* closed = reinterpret_cast<double*>(smem + a.bar_bytes) + (size_t)wib * CAPC;
  // empty_offset entries of a flagged shared-slot tile, staged before the
  // next tile's gathers go out so the write-back issues no global loads
  int32_t* eos = reinterpret_cast<int32_t*>(smem + a.bar_bytes + (size_t)NW * CAPC * 8) +
                 (size_t)wib * kEoSlots;
  unsigned char* ring = smem + a.bar_bytes + (size_t)NW * (CAPC * 8 + kEoSlots * 4) +
                        (size_t)wib * S * a.stage_bytes;
  double* __restrict__ spill = a.spill + (size_t)w * (B + 1);  // slots 0..B
  // x_mode 7 (VR): the tile's x values, gathered in CSR order, pass through
  // this per-warp buffer into the lane-per-column order of the depth loop
  double* xex = reinterpret_cast<double*>(smem + a.bar_bytes + (size_t)NW * (CAPC * 8 + kEoSlots * 4) +
                                          (size_t)NW * S * a.stage_bytes) + (size_t)wib * SIG * 33;
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_x = a.x_frac >= 1.0f ? policy_evict_last() : policy_evict_last_frac(a.x_frac);
  const uint64_t pol_cold = a.cold_pol == 2   ? policy_evict_last()
                            : a.cold_pol == 1 ? policy_evict_normal()
                                              : policy_evict_first();
  const W* __restrict__ desc = static_cast<const W*>(a.desc);

  int64_t kb = 0, ke = 0;
  if (has_tiles) {
    kb = TR ? a.trace_tile : a.warp_begin[w];
    ke = TR ? kb + 1 : a.warp_begin[w + 1];
  }
  auto issue = [&](int64_t k, int s) {  // lane 0 only
    unsigned char* st = ring + (size_t)s * a.stage_bytes;
    uint64_t* bar = bars + s;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)),
                 "r"(TILE_BYTES)
                 : "memory");
    if (!VR) bulk_load(st, a.val + k * B, B * 8, bar, pol_s);
    bulk_load(st + COL_OFF, a.col + k * B, B * 4, bar, pol_s);
    bulk_load(st + DESC_OFF, desc + k * 32, 32 * sizeof(W), bar, pol_s);
  };
  if (has_tiles && lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(bars + s);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < S && kb + s < ke; ++s) issue(kb + s, s);
  }
  __syncwarp();

  if (!TR) rows_part<!NF>(a);
  if (has_tiles) {
    double* __restrict__ y = a.y;
    const bool yh = KNOBS && a.y_hint != 0;
    const bool mirrored = mir_on(a.mir);
    auto put_y = [&](int64_t r, double v) {
      if (TR) return;
      if (yh)
        st_hint(y + r, v, pol_s);
      else
        y[r] = v;
      if (mirrored) mirror_store(a.mir, r, v);
    };
    int64_t pend_row = -1;
    double pend_val = 0.0;
    bool pend_first = true;
    // the pending run is a long row: its parts go to their slots (pend_cnt of
    // them stored so far by this warp); first_long: the warp's first run was
    bool pend_long = false, first_long = false;
    int32_t pend_L = -1, pend_cnt = 0;
    int32_t ltv = 0;  // long tags of 32 tiles (batched like tile_ptr)
    // the warp's first run is resolved after its loop, together with the last
    // one (both pair exchanges in flight at once, none stalls the tile loop)
    int64_t first_row = -1;
    double first_val = 0.0;
    uint32_t tpv = 0, tpv_next = 0;
    int64_t eov = 0;
    int s = 0;
    uint32_t phase = 0;
    // x gathers run one tile ahead: while tile k is spliced and written back,
    // the first CH gathers of tile k+1 (whose col_idx already sit in the next
    // ring stage) are in flight.
    // VR: the tile's values come in with its gathers (coalesced, streaming)
    double va[VR ? CH : 1];
    auto gather = [&](int st_idx, int64_t kt, double(&xv)[CH]) {
      const int32_t* sc = reinterpret_cast<const int32_t*>(ring + (size_t)st_idx * a.stage_bytes + COL_OFF);
      if (VR) {
  #pragma unroll
        for (int u = 0; u < (VR ? CH : 0); ++u)
          va[u] = ld_stream(a.val + kt * B + u * 32 + lane, pol_s);
      }
      if constexpr (GM == 1) {
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = ld_keep_na(a.x + sc[u * 32 + lane], pol_x);
      } else if constexpr (GM == 2) {
  #pragma unroll
        for (int u = 0; u < CH; ++u) {
          const int e = u * 32 + lane, i = e / SIG, j = e - (e / SIG) * SIG;
          xv[u] = ld_keep_na64(a.x + sc[j * 32 + i], pol_x);
        }
      } else if constexpr (GM == 3) {
  #pragma unroll
        for (int u = 0; u < CH; ++u)
          xv[u] = ld_x_split_l1<true>(a.x, a.xh, sc[u * 32 + lane], pol_x, pol_cold);
      } else if constexpr (GM == 5) {
  #pragma unroll
        for (int u = 0; u < CH; ++u)
          xv[u] = ld_x_split(a.x, a.xh, sc[u * 32 + lane], pol_x, pol_cold);
      } else if constexpr (GM == 4) {
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = ld_x_plain(a.x + sc[u * 32 + lane]);
      } else if (a.x_mode == 9) {  // profiling: no gathers (x taken as the column's parity)
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = (double)(sc[u * 32 + lane] & 1);
      } else if (a.x_mode == 10) {  // profiling: every gather reads x[0] (an L1 hit)
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = ld_keep(a.x + (sc[u * 32 + lane] & 0), pol_x);
      } else if (VR && a.xh) {  // hot-column staging (hotx.cu): c < 0 reads xh[~c]
        const bool csr_order = a.x_mode == 7 || a.x_mode == 8, pf64 = a.x_mode == 8 || a.x_mode == 5;
  #pragma unroll
        for (int u = 0; u < CH; ++u) {
          const int e = u * 32 + lane, i = e / SIG, j = e - (e / SIG) * SIG;
          const int32_t c = sc[csr_order ? j * 32 + i : u * 32 + lane];
          if (a.hot_l1)
            xv[u] = pf64 ? ld_x_split_l1<true>(a.x, a.xh, c, pol_x, pol_cold)
                         : ld_x_split_l1<false>(a.x, a.xh, c, pol_x, pol_cold);
          else
            xv[u] = pf64 ? ld_x_split64(a.x, a.xh, c, pol_x, pol_cold)
                         : ld_x_split(a.x, a.xh, c, pol_x, pol_cold);
        }
      } else if (VR && (a.x_mode == 7 || a.x_mode == 8)) {  // CSR order: lane L fetches entry u*32 + L
  #pragma unroll
        for (int u = 0; u < CH; ++u) {
          const int e = u * 32 + lane, i = e / SIG, j = e - (e / SIG) * SIG;
          if (a.x_mode == 8)
            xv[u] = ld_keep_na64(a.x + sc[j * 32 + i], pol_x);
          else
            xv[u] = ld_keep_na(a.x + sc[j * 32 + i], pol_x);
        }
      } else if (a.x_mode == 1) {
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = ld_keep_na(a.x + sc[u * 32 + lane], pol_x);
      } else if (a.x_mode == 2) {
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = ld_x_lsu(a.x + sc[u * 32 + lane], pol_x);
      } else if (a.x_mode == 3) {
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = ld_x_cg(a.x + sc[u * 32 + lane]);
      } else if (a.x_mode == 4) {
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = ld_x_plain(a.x + sc[u * 32 + lane]);
      } else if (a.x_mode == 5) {
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = ld_keep_na64(a.x + sc[u * 32 + lane], pol_x);
      } else if (a.x_mode == 6) {
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = ld_x_plain64(a.x + sc[u * 32 + lane]);
      } else {
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = ld_keep(a.x + sc[u * 32 + lane], pol_x);
      }
    };
    double xa[CH];
    // staged plans: the staged values are complete from here on (k_xhot_fill)
    if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    mbar_wait(bars, 0);
    gather(0, kb, xa);

    for (int64_t k = kb; k < ke; ++k) {
      const int slot = (int)((k - kb) & 31);
      if (slot == 0) {  // per-tile scalars, 32 tiles per batch
        const int64_t last = a.tile_ptr_len - 1;
        tpv = a.tile_ptr[k + lane < last ? k + lane : last];
        tpv_next = a.tile_ptr[k + 32 < last ? k + 32 : last];
        if (!NF) eov = a.eo_ptr[k + lane < a.pcs ? k + lane : a.pcs];
        if (!NF && !TR && a.has_long) ltv = a.ltag[k + lane < a.pcs ? k + lane : a.pcs - 1];
      }
      const uint32_t tp = __shfl_sync(kFull, tpv, slot);
      const uint32_t tpn_s = __shfl_sync(kFull, tpv, (slot + 1) & 31);
      const uint32_t tpn = slot == 31 ? tpv_next : tpn_s;
      const int64_t eo_base = __shfl_sync(kFull, eov, slot);
      const int64_t tile_row = tp & 0x7fffffffu;
      const bool flagged = !NF && (tp >> 31) != 0;
      const int64_t next_row = (k + 1 == a.pcs) ? a.next_row_after : (int64_t)(tpn & 0x7fffffffu);
      const int32_t* __restrict__ eo = a.eo + eo_base;

      // profiling knob 2: compute only -- every tile re-reads the resident
      // stage 0, no TMA traffic after the prologue (y is garbage)
      const bool compute_only = KNOBS && a.stream_only == 2;
      const int sn = compute_only ? 0 : (s + 1 == S ? 0 : s + 1);
      const uint32_t pn = compute_only ? 0u : (s + 1 == S ? phase ^ 1u : phase);
      if (KNOBS && a.stream_only == 1) {  // profiling knob 1: the TMA ring alone (y is garbage)
        mbar_wait(bars + s, phase);
        __syncwarp();
        if (lane == 0 && k + S < ke) issue(k + S, s);
        s = s + 1 == S ? 0 : s + 1;
        phase = s == 0 ? phase ^ 1u : phase;
        continue;
      }
      // random gathers (long misses): tile k+1's gathers also overlap tile k's
      // depth loop, at the cost of a second register array and a copy
      double xn[CH];
      if (EARLY_OK && a.early_gather && k + 1 < ke) {
        if (!compute_only) mbar_wait(bars + sn, pn);
        gather(sn, k + 1, xn);
      }
      const unsigned char* st = ring + (size_t)s * a.stage_bytes;
      const double* sv = reinterpret_cast<const double*>(st);
      const int32_t* sc = reinterpret_cast<const int32_t*>(st + COL_OFF);
      const uint64_t wd = (uint64_t)reinterpret_cast<const W*>(st + DESC_OFF)[lane];
      const uint64_t fr = __brevll(wd & FMASK) >> (64 - SIG);  // bit j = depth j
      const int yoff = (int)(wd >> (kSegBits + SIG));
      const int cnt = __popcll(fr);
      const int H = __shfl_sync(kFull, yoff + cnt, 31);
      const bool fast = NF || H < CAPC;
      // a flagged shared-slot tile's empty_offset entries (H < 128: at most 4
      // per lane) are in flight during the depth loop
      int32_t eov4[4] = {0, 0, 0, 0};
      if (flagged && fast) {
  #pragma unroll
        for (int q = 0; q < 4; ++q)
          if (lane + 32 * q < H) eov4[q] = eo[lane + 32 * q];
      }

      // ---- depth loop (spmv.cpp:61-95): gathers first, then FMAs ----
      // Every close at a bit flag goes to a slot: lane i's k-th flag ends the
      // segment of head yoff_i + k - 1 (k = 0: the piece continuing the column to
      // the left, "red"), stored at slot yoff_i + k (slot h + 1 = head h).  A
      // tile whose slots fit in shared memory (the common case) stores them
      // there; tiles of very short rows (more heads than slots) use the
      // per-warp global spill area.  Both use the gathered x registers.
      double sum = 0.0, red = 0.0;
      // one unrolled loop for both slot areas: shared memory (to_smem) or the
      // per-warp global spill area, which also keeps this lane's first close
      // ("red") in a register
      auto depth_loop = [&](auto to_smem) {
        constexpr bool SM = decltype(to_smem)::value;
        double* cp = SM ? closed + yoff : spill + yoff;
        bool any = false;
  #pragma unroll
        for (int j0 = 0; j0 < SIG; j0 += CH) {
          double xv[CH];
          if (j0 == 0 && VR && (GM == 2 || (GM == 0 && (a.x_mode == 7 || a.x_mode == 8)))) {
            constexpr int rs = 33;  // row stride 33: no bank conflicts
  #pragma unroll
            for (int u = 0; u < CH; ++u) {
              const int e = u * 32 + lane, i = e / SIG, j = e - (e / SIG) * SIG;
              xex[j * rs + i] = xa[u];
            }
            __syncwarp();
  #pragma unroll
            for (int u = 0; u < CH; ++u) xv[u] = xex[u * rs + lane];
            __syncwarp();
          } else if (j0 == 0) {
  #pragma unroll
            for (int u = 0; u < CH; ++u) xv[u] = xa[u];
          } else {
  #pragma unroll
            for (int u = 0; u < CH; ++u)
              if (j0 + u < SIG) xv[u] = ld_keep(a.x + sc[(j0 + u) * 32 + lane], pol_x);
          }
  #pragma unroll
          for (int u = 0; u < CH; ++u) {
            const int j = j0 + u;
            if (j < SIG) {
              if ((fr >> j) & 1ull) {  // predicated: store, advance, restart
                if (!SM) {
                  red = any ? red : sum;
                  any = true;
                }
                *cp++ = sum;
                sum = 0.0;
              }
              sum = fma(VR ? va[VR ? u : 0] : sv[j * 32 + lane], xv[u], sum);
            }
          }
        }
      };
      if (fast)
        depth_loop(std::true_type{});
      else
        depth_loop(std::false_type{});
      // predicated stores on every path: the loads above are consumed here, before
      // the gathers go out, on flagged and unflagged tiles alike (a branch would
      // leave a possibly-outstanding load whose scoreboard the gathers reuse)
  #pragma unroll
      for (int q = 0; q < 4; ++q)
        if (!NF) sts_if(eos + lane + 32 * q, eov4[q], flagged && fast && lane + 32 * q < H);
      __syncwarp();
      if (lane == 0 && k + S < ke && !compute_only) issue(k + S, s);  // refill this stage
      // gathers for tile k+1 land in the registers the depth loop just drained;
      // their latency overlaps this tile's splice, write-back and run merge
      if (EARLY_OK && a.early_gather) {
  #pragma unroll
        for (int u = 0; u < CH; ++u) xa[u] = xn[u];
      } else if (k + 1 < ke) {
        if (!compute_only) mbar_wait(bars + sn, pn);
        gather(sn, k + 1, xa);
      }
      s = sn;
      phase = pn;

      // ---- splice across columns: tmp[i] = piece handed left by column i+1 ----
      const bool seen = cnt > 0;
      // this lane's own first close: read back from shared memory (the spill
      // loop keeps it in a register, so no global load here has to wait for
      // the next tile's gathers)
      if (fast && seen) red = closed[yoff];
      const double give = seen ? red : sum;
      double tmp = __shfl_down_sync(kFull, give, 1);
      if (lane == 31) tmp = 0.0;
      const uint32_t hb = __ballot_sync(kFull, seen);
      double acc = tmp;
      // every column holds a head (rows no longer than sigma: stencils,
      // Laplacians): end == lane on every lane, the scan adds nothing
      if (hb != kFull) {
        const uint64_t above = (uint64_t)hb >> (lane + 1);
        const int end = above ? lane + __ffsll((long long)above) - 1 : 31;
  #pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const double o = __shfl_down_sync(kFull, acc, d);
          if (lane + d <= end) acc += o;
        }
      }
      if (seen) {  // the column's bottom piece
        if (fast)
          closed[yoff + cnt] = sum + acc;
        else
          spill[yoff + cnt] = sum + acc;
      }
      __syncwarp();

      // ---- write-back of the tile's heads in order ----
      // Two copies of one loop: shared-slot tiles read slots and empty_offset
      // from shared memory only, spill tiles from global memory.
      if constexpr (NF) {
        // NF plans: no tile is flagged (head h is row tile_row + h, no empty
        // row to zero) and no tile lies inside one row (maybe_long is false),
        // so every tile has H >= 2 heads: its head-0 run closes here, heads
        // 1..H-2 are final, and only the last head carries over -- the same
        // stores and additions as the general path below, in fewer
        // instructions (Laplacian 1000^2: the tile loop is issue-bound).
        const double c0 = closed[1], cL = closed[H];
        for (int h = lane + 1; h < H - 1; h += 32) put_y(tile_row + h, closed[h + 1]);
        __syncwarp();  // closed[] is rewritten by the next tile
        if (k == kb) {
          first_row = tile_row;
          first_val = c0;
        } else if (lane == 0) {
          if (tile_row == pend_row) {
            put_y(pend_row, pend_val + c0);
          } else {
            put_y(pend_row, pend_val);
            put_y(tile_row, c0);
          }
        }
        pend_row = tile_row + H - 1;
        pend_val = cL;
        pend_first = false;
        continue;
      }
      double c0 = 0.0, cL = 0.0;
      int64_t rL = 0;
      int64_t defer_lo = 0, defer_hi = 0;
      auto write_back = [&](auto eo_at, auto slot_at) {
        c0 = slot_at(1);
        cL = slot_at(H);
        // an unflagged tile has no empty row in [tile_row, next_row]: its last
        // head is row tile_row + H - 1 and nothing after it needs zeroing, so
        // the loop stops before it (H = 33, common at sigma * 32 = rows * nnz/row
        // plus one partial row, then takes one trip instead of two)
        const int hend = flagged ? H : H - 1;
        const int nch = (hend + 31) >> 5;
  #pragma unroll 1
        for (int c = 0; c < nch; ++c) {  // warp-uniform trip count
          const int h = lane + 32 * c;
          if (h >= hend) break;
          const int64_t r = tile_row + (flagged ? (int64_t)eo_at(h) : (int64_t)h);
          if (h == H - 1) rL = r;
          if (h != 0 && h != H - 1) put_y(r, slot_at(h + 1));
          if (flagged || h == H - 1) {  // empty rows up to the next head (or next tile)
            const int64_t nr = h + 1 < H ? tile_row + (int64_t)eo_at(h + 1) : next_row;
            if (nr - r - 1 <= 8) {
              for (int64_t q = r + 1; q < nr; ++q) put_y(q, 0.0);
            } else if (defer_hi == defer_lo) {
              defer_lo = r + 1;
              defer_hi = nr;
            } else {
              for (int64_t q = r + 1; q < nr; ++q) put_y(q, 0.0);
            }
          }
        }
      };
      if (fast)
        write_back([&](int i) { return eos[i]; }, [&](int i) { return closed[i]; });
      else
        write_back([&](int i) { return eo[i]; }, [&](int i) { return spill[i]; });
      rL = flagged ? __shfl_sync(kFull, rL, (H - 1) & 31) : tile_row + H - 1;
      uint32_t dm = flagged ? __ballot_sync(kFull, defer_hi > defer_lo) : 0u;
      while (dm) {  // long empty-row runs: zero cooperatively
        const int src = __ffs(dm) - 1;
        dm &= dm - 1;
        const int64_t lo = __shfl_sync(kFull, defer_lo, src);
        const int64_t hi = __shfl_sync(kFull, defer_hi, src);
        for (int64_t q = lo + lane; q < hi; q += 32) put_y(q, 0.0);
      }
      if (TR) {  // the tile's contributions: every head's row and final value
        for (int h = lane; h < H; h += 32) {
          a.trace_row[h] = tile_row + (flagged ? (int64_t)(fast ? eos[h] : eo[h]) : (int64_t)h);
          a.trace_val[h] = fast ? closed[h + 1] : spill[h + 1];
        }
        if (lane == 0) *a.trace_count = H;
        return;
      }
      __syncwarp();  // closed[] is rewritten by the next tile

      // ---- row runs across the warp's consecutive tiles ----
      auto flush = [&]() {  // warp-uniform
        if (!NF && pend_long) {
          long_arrive_warp(a, pend_L, pend_cnt, lane);
        } else if (pend_first) {
          first_row = pend_row;
          first_val = pend_val;
        } else if (lane == 0) {
          put_y(pend_row, pend_val);
        }
      };
      if (NF || !a.has_long) {  // no long rows: fold every run here
        if (k == kb) {
          pend_row = tile_row;
          pend_val = c0;
          pend_first = true;
        } else if (tile_row == pend_row) {
          pend_val += c0;
        } else {
          flush();
          pend_row = tile_row;
          pend_val = c0;
          pend_first = false;
        }
        if (H >= 2) {
          flush();
          pend_row = rL;
          pend_val = cL;
          pend_first = false;
        }
      } else {
        // long rows (three or more parts) store each part in its slot instead
        // of folding it here (the fixed-order sum happens at the row's last
        // arrival, long_arrive_warp)
        const int ltg = __shfl_sync(kFull, ltv, slot);
        const int l0 = (ltg & 1) ? ltg >> 2 : -1;
        const int lL = (ltg & 2) ? (ltg >> 2) + (ltg & 1) : -1;
        auto store_part = [&](int L, double v) {
          if (lane == 0) a.lparts[a.lbase[L] + (k + a.t0 - a.ltf[L])] = v;
        };
        auto start = [&](int64_t row, double v, int L) {
          pend_row = row;
          if (L >= 0) {
            store_part(L, v);
            pend_long = true;
            pend_L = L;
            pend_cnt = 1;
          } else {
            pend_val = v;
            pend_long = false;
          }
        };
        if (k == kb) {
          start(tile_row, c0, l0);
          pend_first = !pend_long;
          first_long = pend_long;
        } else if (tile_row == pend_row) {
          if (pend_long) {
            store_part(pend_L, c0);
            ++pend_cnt;
          } else {
            pend_val += c0;
          }
        } else {
          flush();
          pend_first = false;
          start(tile_row, c0, l0);
        }
        if (H >= 2) {
          flush();
          pend_first = false;
          start(rL, cL, lL);
        }
      }
    }
    if (KNOBS && a.stream_only) return;  // profiling knobs: no rows were produced
    const bool last_long = !NF && pend_long;
    if (last_long) long_arrive_warp(a, pend_L, pend_cnt, lane);
    // a long row's items are single-item runs of their own (k_item_keys):
    // nothing to resolve for them
    const bool do0 = NF || !first_long, do1 = NF || !last_long;
    const int64_t i0 = 2 * (int64_t)w, i1 = i0 + 1;
    const int64_t r0 = pend_first ? pend_row : first_row;
    const double v0 = pend_first ? pend_val : first_val;
    const double v1 = pend_first ? 0.0 : pend_val;
    // (NF plans never have a run of more than two items: no row covers a tile)
    const bool short_runs = NF || (a.run_last[i0] - a.run_first[i0] <= 1 &&
                                   a.run_last[i1] - a.run_first[i1] <= 1);
    if (a.atomic) {  // spmv.cpp:273-295: fp64 atomics into the zeroed y
      if (lane == 0) {
        if (do0 && v0 != 0.0) atomicAdd(a.y + r0, v0);
        if (do1 && v1 != 0.0) atomicAdd(a.y + pend_row, v1);
      }
    } else if (short_runs) {
      // both runs hold one or two partials: lane 0 issues both exchanges, then
      // finishes whichever it completed
      if (lane == 0) {
        const int s0 = a.run_first[i0], e0 = a.run_last[i0];
        const int s1 = a.run_first[i1], e1 = a.run_last[i1];
        unsigned long long o0 = 0, o1 = 0;
        if (e0 > s0 && do0)
          o0 = atomicExch(reinterpret_cast<unsigned long long*>(a.item_val + s0),
                          (unsigned long long)__double_as_longlong(exchangeable(v0)));
        if (e1 > s1 && do1)
          o1 = atomicExch(reinterpret_cast<unsigned long long*>(a.item_val + s1),
                          (unsigned long long)__double_as_longlong(exchangeable(v1)));
        if (!do0) {
        } else if (e0 == s0) {
          write_run(r0, v0, a.y, a.first_row, a.first_owned, a.send, a.send_flag, a.send_epoch,
                    a.mir);
        } else if (o0 != kSlotIdle && !(s1 == s0 && e1 > s1)) {
          a.item_val[s0] = __longlong_as_double((long long)kSlotIdle);
          write_run(r0, __longlong_as_double((long long)o0) + v0, a.y, a.first_row,
                    a.first_owned, a.send, a.send_flag, a.send_epoch, a.mir);
        }
        if (!do1) {
        } else if (e1 == s1) {
          write_run(pend_row, v1, a.y, a.first_row, a.first_owned, a.send, a.send_flag,
                    a.send_epoch, a.mir);
        } else if (o1 != kSlotIdle) {
          a.item_val[s1] = __longlong_as_double((long long)kSlotIdle);
          write_run(pend_row, __longlong_as_double((long long)o1) + v1, a.y, a.first_row,
                    a.first_owned, a.send, a.send_flag, a.send_epoch, a.mir);
        }
      }
    } else {
      if (do0) resolve_item_warp(a, i0, r0, v0, lane);
      if (do1) resolve_item_warp(a, i1, pend_row, v1, lane);
    }
  }
}

using SpmvFn = void (*)(SpmvArgs);
constexpr int kNfMaxSigma = 8;  // NF variants are instantiated up to this sigma

// the sigma switch of each instantiation unit (nullptr: not instantiated)
SpmvFn spmv_fn_general(int sigma);
SpmvFn spmv_fn_vr(int sigma);
SpmvFn spmv_fn_nf(int sigma);
SpmvFn spmv_fn_trace(int sigma);
SpmvFn spmv_fn_vr_gm(int sigma, int gm);  // GM 1..3, 5 (spmv_inst_vr_gm*.cu)
SpmvFn spmv_fn_local_gm4(int sigma, bool nf);  // GM 4, general / NF (spmv_inst_gm4.cu)

// k_spmv<S..MAX, ...> as a sigma switch, instantiated where it is called
template <int S, int MAX, bool VR, bool NF, bool TR, int GM>
SpmvFn pick_sigma(int sigma) {
  if constexpr (S > MAX) {
    return nullptr;
  } else {
    return sigma == S ? k_spmv<S, VR, NF, TR, GM> : pick_sigma<S + 1, MAX, VR, NF, TR, GM>(sigma);
  }
}

}  // namespace csr5g
