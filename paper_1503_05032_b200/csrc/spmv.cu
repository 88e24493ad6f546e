// spmv.cu -- CSR5 SpMV (reference: spmv.cpp:42-124, 224-298).
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
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
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

__device__ void resolve_item(const SpmvArgs& a, int64_t idx, int64_t row, double v);

// Tail rows and leading/trailing empty rows, grid-stride over all threads.
__device__ void rows_part(const SpmvArgs& a) {
  const int64_t tail_rows = a.m - a.tail_row_begin;
  const int64_t total = a.lead_rows + tail_rows;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    if (idx < a.lead_rows) {
      a.y[idx] = 0.0;
      if (a.mir.n) mirror_store(a.mir, idx, 0.0);
      continue;
    }
    const int64_t r = a.tail_row_begin + (idx - a.lead_rows);
    int64_t lo = a.row_ptr[r];
    const int64_t hi = a.row_ptr[r + 1];
    if (lo < a.tail_pos) lo = a.tail_pos;
    double s = 0.0;
    for (int64_t q = lo; q < hi; ++q) s = fma(a.val[q - a.pos0], a.x[a.col[q - a.pos0]], s);
    if (a.has_tail_item && r == a.tail_row_begin) {
      resolve_item(a, 2 * (int64_t)a.nwarps, r, s);
    } else {
      a.y[r] = s;
      if (a.mir.n) mirror_store(a.mir, r, s);
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
    if (mir.n && row != mir.skip_row) mirror_store(mir, row, v);
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

__device__ __forceinline__ bool pair_exchange(const SpmvArgs& a, int s, double v, double* total) {
  auto* slot = reinterpret_cast<unsigned long long*>(a.item_val + s);
  const unsigned long long old = atomicExch(slot, (unsigned long long)__double_as_longlong(v));
  if (old == kSlotIdle) return false;
  *slot = kSlotIdle;
  *total = __longlong_as_double((long long)old) + v;
  return true;
}

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
    t = 0.0;
#pragma unroll 4
    for (int j = s; j <= e; ++j) t += __ldcg(a.item_val + j);
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
template <int SIG, bool VR, bool NF = false>
__global__ void __launch_bounds__(NF ? spmv_threads_nf(SIG) : spmv_threads(SIG), 1)
    k_spmv(SpmvArgs a) {
  using W = typename std::conditional<(SIG <= 17), uint32_t, uint64_t>::type;
  constexpr int B = 32 * SIG;
  constexpr int CH = SIG <= 32 ? SIG : (SIG + 1) / 2;  // x gathers in flight per lane
  static_assert(!VR || CH == SIG, "VR needs the whole tile's gathers in one batch");
  constexpr int CAPC = B < kClosedSlots ? B : kClosedSlots;
  constexpr uint64_t FMASK = (1ull << SIG) - 1;
  constexpr bool EARLY_OK = !VR && SIG <= 18;  // a second x array fits in registers
  constexpr uint32_t COL_OFF = VR ? 0 : B * 8, DESC_OFF = COL_OFF + B * 4;
  constexpr uint32_t TILE_BYTES = DESC_OFF + 32 * sizeof(W);

  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (a.first_owned && !a.atomic && blockIdx.x == 0 && threadIdx.x == 0) {
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
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_x = a.x_frac >= 1.0f ? policy_evict_last() : policy_evict_last_frac(a.x_frac);
  const W* __restrict__ desc = static_cast<const W*>(a.desc);

  int64_t kb = 0, ke = 0;
  if (has_tiles) {
    kb = a.warp_begin[w];
    ke = a.warp_begin[w + 1];
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

  rows_part(a);
  if (has_tiles) {
    double* __restrict__ y = a.y;
    const bool yh = a.y_hint != 0;
    const bool mirrored = a.mir.n != 0;
    auto put_y = [&](int64_t r, double v) {
      if (yh)
        st_hint(y + r, v, pol_s);
      else
        y[r] = v;
      if (mirrored) mirror_store(a.mir, r, v);
    };
    int64_t pend_row = -1;
    double pend_val = 0.0;
    bool pend_first = true;
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
      if (a.x_mode == 1) {
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
      } else {
  #pragma unroll
        for (int u = 0; u < CH; ++u) xv[u] = ld_keep(a.x + sc[u * 32 + lane], pol_x);
      }
    };
    double xa[CH];
    mbar_wait(bars, 0);
    gather(0, kb, xa);

    for (int64_t k = kb; k < ke; ++k) {
      const int slot = (int)((k - kb) & 31);
      if (slot == 0) {  // per-tile scalars, 32 tiles per batch
        const int64_t last = a.tile_ptr_len - 1;
        tpv = a.tile_ptr[k + lane < last ? k + lane : last];
        tpv_next = a.tile_ptr[k + 32 < last ? k + 32 : last];
        if (!NF) eov = a.eo_ptr[k + lane < a.pcs ? k + lane : a.pcs];
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
      const bool compute_only = a.stream_only == 2;
      const int sn = compute_only ? 0 : (s + 1 == S ? 0 : s + 1);
      const uint32_t pn = compute_only ? 0u : (s + 1 == S ? phase ^ 1u : phase);
      if (a.stream_only == 1) {  // profiling knob 1: the TMA ring alone (y is garbage)
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
          if (j0 == 0) {
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
      __syncwarp();  // closed[] is rewritten by the next tile

      // ---- row runs across the warp's consecutive tiles ----
      auto flush = [&]() {  // warp-uniform
        if (pend_first) {
          first_row = pend_row;
          first_val = pend_val;
        } else if (lane == 0) {
          put_y(pend_row, pend_val);
        }
      };
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
    }
    if (a.stream_only) return;  // profiling knobs: no rows were produced
    const int64_t i0 = 2 * (int64_t)w, i1 = i0 + 1;
    const int64_t r0 = pend_first ? pend_row : first_row;
    const double v0 = pend_first ? pend_val : first_val;
    const double v1 = pend_first ? 0.0 : pend_val;
    const bool short_runs = !a.atomic && a.run_last[i0] - a.run_first[i0] <= 1 &&
                            a.run_last[i1] - a.run_first[i1] <= 1;
    if (short_runs) {
      // both runs hold one or two partials: lane 0 issues both exchanges, then
      // finishes whichever it completed
      if (lane == 0) {
        const int s0 = a.run_first[i0], e0 = a.run_last[i0];
        const int s1 = a.run_first[i1], e1 = a.run_last[i1];
        unsigned long long o0 = 0, o1 = 0;
        if (e0 > s0)
          o0 = atomicExch(reinterpret_cast<unsigned long long*>(a.item_val + s0),
                          (unsigned long long)__double_as_longlong(v0));
        if (e1 > s1)
          o1 = atomicExch(reinterpret_cast<unsigned long long*>(a.item_val + s1),
                          (unsigned long long)__double_as_longlong(v1));
        if (e0 == s0) {
          write_run(r0, v0, a.y, a.first_row, a.first_owned, a.send, a.send_flag, a.send_epoch,
                    a.mir);
        } else if (o0 != kSlotIdle && !(s1 == s0 && e1 > s1)) {
          a.item_val[s0] = __longlong_as_double((long long)kSlotIdle);
          write_run(r0, __longlong_as_double((long long)o0) + v0, a.y, a.first_row,
                    a.first_owned, a.send, a.send_flag, a.send_epoch, a.mir);
        }
        if (e1 == s1) {
          write_run(pend_row, v1, a.y, a.first_row, a.first_owned, a.send, a.send_flag,
                    a.send_epoch, a.mir);
        } else if (o1 != kSlotIdle) {
          a.item_val[s1] = __longlong_as_double((long long)kSlotIdle);
          write_run(pend_row, __longlong_as_double((long long)o1) + v1, a.y, a.first_row,
                    a.first_owned, a.send, a.send_flag, a.send_epoch, a.mir);
        }
      }
    } else {
      resolve_item_warp(a, i0, r0, v0, lane);
      resolve_item_warp(a, i1, pend_row, v1, lane);
    }
  }
}

namespace {

__global__ void k_fixup(const csr5g_partial* __restrict__ all, int world, int rank, int64_t row,
                        double* __restrict__ y) {
  double acc = y[row];
  for (int s = rank + 1; s < world; ++s) {
    if (all[s].row != row) break;
    acc += all[s].value;
  }
  y[row] = acc;
}

using SpmvFn = void (*)(SpmvArgs);

// sigma is 1..48 at omega = 32 (the 64-bit descriptor limit, descriptor.cpp:22-36)
constexpr int kNfMaxSigma = 8;  // NF variants are instantiated up to this sigma

SpmvFn spmv_fn(int sigma, bool vr, bool nf = false) {
  if (nf && !vr && sigma <= kNfMaxSigma) {
    switch (sigma) {
#define CSR5G_KN(S) \
  case S:           \
    return k_spmv<S, false, true>;
      CSR5G_KN(1) CSR5G_KN(2) CSR5G_KN(3) CSR5G_KN(4) CSR5G_KN(5) CSR5G_KN(6) CSR5G_KN(7)
      CSR5G_KN(8)
#undef CSR5G_KN
      default:
        return nullptr;
    }
  }
  if (vr) {
    switch (sigma) {
#define CSR5G_KV(S) \
  case S:           \
    return k_spmv<S, true>;
      CSR5G_KV(1) CSR5G_KV(2) CSR5G_KV(3) CSR5G_KV(4) CSR5G_KV(5) CSR5G_KV(6) CSR5G_KV(7)
      CSR5G_KV(8) CSR5G_KV(9) CSR5G_KV(10) CSR5G_KV(11) CSR5G_KV(12) CSR5G_KV(13) CSR5G_KV(14)
      CSR5G_KV(15) CSR5G_KV(16) CSR5G_KV(17) CSR5G_KV(18) CSR5G_KV(19) CSR5G_KV(20)
      CSR5G_KV(21) CSR5G_KV(22) CSR5G_KV(23) CSR5G_KV(24)
#undef CSR5G_KV
      default:
        return nullptr;
    }
  }
  switch (sigma) {
#define CSR5G_K(S) \
  case S:          \
    return k_spmv<S, false>;
    CSR5G_K(1) CSR5G_K(2) CSR5G_K(3) CSR5G_K(4) CSR5G_K(5) CSR5G_K(6) CSR5G_K(7) CSR5G_K(8)
    CSR5G_K(9) CSR5G_K(10) CSR5G_K(11) CSR5G_K(12) CSR5G_K(13) CSR5G_K(14) CSR5G_K(15)
    CSR5G_K(16) CSR5G_K(17) CSR5G_K(18) CSR5G_K(19) CSR5G_K(20) CSR5G_K(21) CSR5G_K(22)
    CSR5G_K(23) CSR5G_K(24) CSR5G_K(25) CSR5G_K(26) CSR5G_K(27) CSR5G_K(28) CSR5G_K(29)
    CSR5G_K(30) CSR5G_K(31) CSR5G_K(32) CSR5G_K(33) CSR5G_K(34) CSR5G_K(35) CSR5G_K(36)
    CSR5G_K(37) CSR5G_K(38) CSR5G_K(39) CSR5G_K(40) CSR5G_K(41) CSR5G_K(42) CSR5G_K(43)
    CSR5G_K(44) CSR5G_K(45) CSR5G_K(46) CSR5G_K(47) CSR5G_K(48)
#undef CSR5G_K
    default:
      return nullptr;
  }
}

}  // namespace

int spmv_plan(Handle* h, int sms) {
  // Shared memory per warp: closed-segment slots (B doubles) + S ring stages.
  // One CTA per SM.  The shared-memory budget depends on the sampled gather
  // locality (lines_per_gather, from the converter):
  //  * local gathers (stencils): up to 226 KB -- the largest ring and warp
  //    count; x gathers mostly hit L1/L2 with few misses in flight;
  //  * random gathers: whatever shared memory is not carved out stays L1,
  //    which is where outstanding gather misses land.  About 100 KB of ring
  //    with 2 stages measured best on both R-MAT s24 (x 134 MB > L2; 2 stages
  //    x 4/6/7/9/10 warps = 64/85/99/127/141 KB -> 2.10/1.74/1.67/1.76/2.02
  //    ms) and mixed s23 (x 67 MB < L2; 6/9/11/12 warps = 57/85/103/113 KB ->
  //    0.67/0.56/0.52/0.53 ms).  tools/gather_probe.cu: uniform random
  //    8-byte gathers top out near 275 G/s (x in L2) and 115 G/s (x 134 MB)
  //    with <= 50% carveout, and fall to 65 / 44 G/s at a 100% carveout.
  const int sigma = (int)h->info.sigma;
  const int wbytes = h->wide ? 8 : 4;
  const bool random = h->lines_per_gather >= 8.0;
  // random plans with short tiles keep the values out of the ring (VR)
  static const int vr_env = [] {
    const char* e = std::getenv("CSR5G_VR");
    return e ? std::atoi(e) : -1;
  }();
  h->vr = random && sigma <= kVrMaxSigma && vr_env != 0;
  if (vr_env == 1 && sigma <= kVrMaxSigma) h->vr = true;
  static const int nf_env = [] {  // CSR5G_NF=0: keep the general kernel (A/B)
    const char* e = std::getenv("CSR5G_NF");
    return e ? std::atoi(e) : -1;
  }();
  h->nf = nf_env != 0 && !h->vr && sigma <= kNfMaxSigma && h->pcs > 0 && h->eo_entries == 0 &&
          h->max_heads < std::min<int64_t>(h->B, kClosedSlots);
  const int64_t tile_bytes = h->B * (h->vr ? 4 : 12) + 32 * wbytes;
  const int stage_bytes = (int)((tile_bytes + 127) / 128 * 128);
  const int closed_bytes = (int)(std::min<int64_t>(h->B, kClosedSlots) * 8);
  int budget = !random ? 226 * 1024 : 104 * 1024;
  if (h->vr) {
    // VR plans: a 2-stage col_idx ring is ~2-4 KB per warp, so warps are
    // bounded by the thread cap or by how many misses the memory system
    // absorbs: with x larger than L2 fewer warps win (R-MAT s24, x 134 MB:
    // 6/8/10/12 warps -> 1.62/1.50/1.45/1.55 ms), with x inside L2 the most
    // (mixed 2^23, x 67 MB: 11/12/16 warps -> 0.514/0.505/0.469 ms)
    int l2 = 0;
    CSR5G_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->device));
    budget = (double)h->info.n * 8.0 > 0.75 * (double)l2 ? 60 * 1024 : 72 * 1024;
  }
  if (const char* e = std::getenv("CSR5G_BUDGET_KB")) budget = std::atoi(e) * 1024;  // experiments
  h->x_mode = random ? 1 : 4;  // random: no L1 allocation; local: plain ld.global.nc
  // No L2 persisting window on x by default: with the 2-stage random plan it
  // gains < 1% (R-MAT s24 1.658 vs 1.669 ms) while its persisting lines outlive
  // the launch and slowed the next unrelated SpMV by 13% (st27 0.504 vs 0.446
  // ms).  CSR5G_XWINDOW=1 turns it on for experiments.
  h->x_window = false;
  // experiment overrides, read when the plan is made
  if (const char* e = std::getenv("CSR5G_XMODE")) h->x_mode = std::atoi(e);
  if (const char* e = std::getenv("CSR5G_XWINDOW")) h->x_window = std::atoi(e) != 0;
  // stages: the tile being reduced + the next tile (its gathers go out as
  // soon as the current depth loop ends) + TMA lead; 2 minimum
  const int min_stages = 2;
  // random gathers: two stages -- the shared memory a third would take is
  // worth more as L1 for outstanding gather misses (measured: R-MAT s24 at
  // 150 KB, 7 warps: 2 stages 1.67 ms, 3 stages 2.11 ms)
  // NF plans (short tiles, sigma <= 8): two stages too -- the 2 KB tile
  // arrives well within one tile's work, and the smaller ring leaves more L1
  // (Laplacian 1000^2 at 24 warps: 2 / 3 stages 25.1 / 26.0 us mean)
  int nw = (h->nf ? spmv_threads_nf(sigma) : spmv_threads(sigma)) / 32,
      stages = random || h->nf ? 2 : 4;
  // one mbarrier per warp and stage at the start, 128-byte aligned
  auto bars = [](int w, int st) { return (w * st * 8 + 127) / 128 * 128; };
  auto need = [&](int w, int st) {
    return bars(w, st) + w * (closed_bytes + kEoSlots * 4 + st * stage_bytes);
  };
  // local gathers: warps per SM matter most (keep them, give up depth first);
  // random gathers: keep the TMA lead (depth), give up warps
  if (!random)
    while (stages > min_stages && need(nw, stages) > budget) --stages;
  while (nw > 1 && need(nw, stages) > budget) --nw;
  while (stages > min_stages && need(nw, stages) > budget) --stages;
  if (const char* e = std::getenv("CSR5G_NW")) nw = std::max(1, std::min(nw, std::atoi(e)));
  if (const char* e = std::getenv("CSR5G_STAGES")) {
    stages = std::max(min_stages, std::min(4, std::atoi(e)));
    while (nw > 1 && need(nw, stages) > budget) --nw;
  }
  h->warps_per_block = nw;
  h->stages = stages;
  h->stage_bytes = stage_bytes;
  h->bar_bytes = bars(nw, stages);
  h->smem_bytes = need(nw, stages);
  // Ask for the smallest shared-memory carveout that holds the ring: the rest
  // of the SM's 256 KB stays L1, which is where outstanding gather misses land
  // (measured: a 233 KB carveout halves R-MAT throughput through mio/lg
  // throttling).  The attributes are set per launch (func_attrs): handles of
  // one sigma can carry different plans.
  {
    int max_smem = 0;
    CSR5G_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor,
                                      h->device));
    const int need_bytes = h->smem_bytes + 1024;  // + the per-CTA reserved 1 KB
    int pct = (int)((100LL * need_bytes + max_smem - 1) / max_smem);
    h->carveout_pct = std::min(100, std::max(0, pct));
  }
  const int64_t max_warps = (int64_t)sms * nw;
  h->nwarps = (int)std::min<int64_t>(max_warps, h->pcs);
  h->tile_blocks = (h->nwarps + nw - 1) / nw;
  return CSR5G_OK;
}

// Kernel attributes (dynamic shared memory, carveout) as the handle's plan
// needs them, set only when they differ from the last values set on that
// device (a host-side map lookup per launch).
int func_attrs(const void* fn, int device, int smem, int carve) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, std::pair<int, int>> cur;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cur.find({fn, device});
  if (it != cur.end() && it->second == std::make_pair(smem, carve)) return CSR5G_OK;
  CSR5G_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (carve >= 0)
    CSR5G_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
  cur[{fn, device}] = {smem, carve};
  return CSR5G_OK;
}

// The scratch of `stream`: the handle's own arrays for the first stream that
// runs an SpMV on it, arrays allocated (stream-ordered) for every other one.
int scratch_for(Handle* h, cudaStream_t stream, double** iv, int32_t** rc, double** sp) {
  std::lock_guard<std::mutex> lock(h->scratch_mu);
  if (!h->scratch_claimed) {
    h->scratch_claimed = true;
    h->scratch_stream = stream;
  }
  if (stream == h->scratch_stream) {
    *iv = h->item_val;
    *rc = h->run_cnt;
    *sp = h->spill;
    return CSR5G_OK;
  }
  for (const StreamScratch& x : h->extra_scratch)
    if (x.stream == stream) {
      *iv = x.item_val;
      *rc = x.run_cnt;
      *sp = x.spill;
      return CSR5G_OK;
    }
  const size_t items = 2 * (size_t)h->nwarps + 1;
  const size_t spill = (size_t)std::max(h->nwarps, 1) * (size_t)(h->B + 1);
  StreamScratch x{stream, nullptr, nullptr, nullptr};
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&x.item_val), items * 8, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(x.item_val, 0xff, items * 8, stream);  // idle slots
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&x.run_cnt), items * 4, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(x.run_cnt, 0, items * 4, stream);
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&x.spill), spill * 8, stream);
  if (e != cudaSuccess) {
    for (void* p : {(void*)x.item_val, (void*)x.run_cnt, (void*)x.spill})
      if (p) cudaFreeAsync(p, stream);
    return cuda_fail(e, "per-stream SpMV scratch");
  }
  h->extra_scratch.push_back(x);
  *iv = x.item_val;
  *rc = x.run_cnt;
  *sp = x.spill;
  return CSR5G_OK;
}

int launch_spmv(Handle* h, const double* d_x, double* d_y, int mode, cudaStream_t stream,
                cudaEvent_t ev0, cudaEvent_t ev1) {
  CSR5G_CUDA(cudaSetDevice(h->device));
  const csr5g_info& in = h->info;
  if (in.m == 0) {
    if (ev0) CSR5G_CUDA(cudaEventRecord(ev0, stream));
    if (ev1) CSR5G_CUDA(cudaEventRecord(ev1, stream));
    return CSR5G_OK;
  }
  const bool atomic = mode == CSR5G_MODE_ATOMIC;
  if (atomic) {
    if (h->t0 != 0 || !h->is_last)
      return fail(CSR5G_EINVAL, "csr5g: atomic mode is single-device only");
    CSR5G_CUDA(cudaMemsetAsync(d_y, 0, sizeof(double) * in.m, stream));
  }
  SpmvArgs a{};
  a.row_ptr = h->row_ptr;
  a.tile_ptr = h->tile_ptr;
  a.desc = h->desc;
  a.eo_ptr = h->eo_ptr;
  a.eo = h->eo;
  a.col = h->col;
  a.val = h->val;
  a.x = d_x;
  a.y = d_y;
  if (int rc = scratch_for(h, stream, &a.item_val, &a.run_cnt, &a.spill)) return rc;
  a.run_first = h->run_first;
  a.run_last = h->run_last;
  a.send = h->send_ext ? h->send_ext : h->send;
  a.send_flag = h->send_flag;
  a.send_epoch = h->send_epoch;
  a.warp_begin = h->warp_begin;
  a.pcs = h->pcs;
  a.pos0 = h->t0 * h->B;
  a.next_row_after = h->next_row_after;
  a.lead_rows = h->lead_rows;
  a.tail_row_begin = h->tail_row_begin;
  a.tail_pos = h->tail_pos;
  a.m = in.m;
  a.tile_ptr_len = in.tile_ptr_len;
  a.first_row = h->first_row;
  a.first_owned = h->first_owned;
  a.has_tail_item = h->has_tail_item;
  a.sigma = (int)in.sigma;
  a.B = (int)h->B;
  a.nwarps = h->nwarps;
  a.stages = h->stages;
  a.stage_bytes = h->stage_bytes;
  a.bar_bytes = h->bar_bytes;
  a.atomic = atomic;
  a.mir = h->mir;
  const int grid = std::max(h->tile_blocks, h->rows_blocks);
  const int threads = 32 * h->warps_per_block;
  const int x_mode = h->x_mode;
  const bool x_window = h->x_window;
  a.x_mode = x_mode;
  a.early_gather = h->lines_per_gather >= 8.0 ? 1 : 0;
  static const float x_frac_env = [] {
    const char* e = std::getenv("CSR5G_XFRAC");
    return e ? (float)std::atof(e) : -1.0f;
  }();
  static const int y_hint_env = [] {
    const char* e = std::getenv("CSR5G_YHINT");
    return e ? std::atoi(e) : -1;
  }();
  a.x_frac = x_frac_env > 0.0f ? std::min(1.0f, x_frac_env) : 1.0f;
  a.y_hint = y_hint_env >= 0 ? y_hint_env : 0;
  if (const char* e = std::getenv("CSR5G_EARLY")) a.early_gather = std::atoi(e) != 0;
  static const int stream_only = [] {  // 1: TMA ring only, 2: compute only (profiling)
    const char* e = std::getenv("CSR5G_STREAM_ONLY");
    return e ? std::atoi(e) : 0;
  }();
  a.stream_only = stream_only;
  const int64_t items = 2 * (int64_t)h->nwarps + (h->has_tail_item ? 1 : 0);
  if (ev0) CSR5G_CUDA(cudaEventRecord(ev0, stream));
  if (grid > 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = h->smem_bytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    if (x_window) {
      // keep x resident in an L2 persisting window (set-aside sized at build)
      int max_win = 0, max_persist = 0;
      cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, h->device);
      cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, h->device);
      static bool limit_set = false;
      if (!limit_set) {
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist);
        limit_set = true;
      }
      const size_t xb = std::min<size_t>((size_t)in.n * 8, (size_t)max_win);
      attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
      attr[0].val.accessPolicyWindow.base_ptr = const_cast<double*>(d_x);
      attr[0].val.accessPolicyWindow.num_bytes = xb;
      attr[0].val.accessPolicyWindow.hitRatio =
          xb ? std::min(1.0f, (float)max_persist / (float)xb) : 1.0f;
      attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
    }
    const SpmvFn fn = spmv_fn(a.sigma, h->vr, h->nf);
    if (int rc = func_attrs((const void*)fn, h->device, h->smem_bytes, h->carveout_pct)) return rc;
    CSR5G_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
  }
  if (ev1) CSR5G_CUDA(cudaEventRecord(ev1, stream));
  // the rows shared between warps were merged inside the kernel
  // (resolve_item); a handle with nothing to multiply has no record
  if (!atomic && items == 0 && grid == 0) {  // no record: row -1 (all ones), value 0.0
    CSR5G_CUDA(cudaMemsetAsync(&a.send->row, 0xff, sizeof(int64_t), stream));
    CSR5G_CUDA(cudaMemsetAsync(&a.send->value, 0, sizeof(double), stream));
  }
  return CSR5G_OK;
}

int launch_fixup(Handle* h, const csr5g_partial* d_all, int world, int rank, double* d_y,
                 cudaStream_t stream) {
  CSR5G_CUDA(cudaSetDevice(h->device));
  if (h->is_last || h->pcs == 0) return CSR5G_OK;        // nothing continues past the tail
  if (!h->first_owned && h->last_row == h->first_row) return CSR5G_OK;  // row owned upstream
  k_fixup<<<1, 1, 0, stream>>>(d_all, world, rank, h->last_row, d_y);
  CSR5G_CUDA(cudaGetLastError());
  return CSR5G_OK;
}

}  // namespace csr5g

