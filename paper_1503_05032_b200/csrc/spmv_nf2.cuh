// spmv_nf2.cuh -- k_spmv_nf2<SIGMA>: the NF plans' tile kernel with two tiles
// per iteration (reference: spmv.cpp:42-124, 224-298; the NF conditions of
// spmv_kernel.cuh: no flagged tile, no tile inside one row, every tile's heads
// fit the slots, sigma <= 8).
//
// Small-sigma tiles (a 2D Laplacian's sigma = 5: 160 entries, ~33 heads) give
// each warp little independent work per iteration: the depth loop is a chain
// of sigma dependent DFMAs, the splice a chain of shuffles, and one warp of
// the general kernel waits on them tile after tile (issue-bound at 55% issue
// activity).  Here a warp takes its tiles in pairs: one ring stage holds two
// consecutive tiles (one bulk copy per array: they are contiguous in HBM),
// both tiles' gathers go out together, and their depth loops, splices and
// write-backs interleave -- two independent dependency chains per warp.  The
// arithmetic, the closes, the splice and the run merge of each tile are the
// NF kernel's, in the same order: y is bit-identical to it.
// The next pair's gathers go out before this pair's splices, like the NF
// kernel's next tile.  Measured on the Laplacian 1000^2: 21.5 us against the
// NF kernel's 20.7 (both bottom out near 20.4 us, so the per-warp work is
// not what bounds it).  Opt-in (CSR5G_NF2=1), tested bit-identical.
#pragma once

#include "spmv_kernel.cuh"

namespace csr5g {

constexpr int kNf2Threads = 640;  // 20 warps (two tiles of state per warp)

template <int SIG>
__global__ void __launch_bounds__(kNf2Threads, 1) k_spmv_nf2(SpmvArgs a) {
  constexpr int B = 32 * SIG;
  constexpr uint64_t FMASK = (1ull << SIG) - 1;
  constexpr uint32_t COL_OFF = 2 * B * 8, DESC_OFF = COL_OFF + 2 * B * 4;
  constexpr uint32_t STAGE = (DESC_OFF + 64 * 4 + 127) / 128 * 128;
  static_assert(SIG <= 17, "NF2 reads 32-bit descriptor words");

  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, NW = blockDim.x >> 5;
  if (a.first_owned && !a.atomic && blockIdx.x == 0 && threadIdx.x == 0) {
    a.send->row = -1;  // this handle has no partial to send
    a.send->value = 0.0;
  }
  const int w = blockIdx.x * NW + wib;
  const bool has_tiles = w < a.nwarps;
  const int CAP = a.nf2_slots;  // per tile: slot h + 1 = head h, H + 1 <= CAP
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + wib * 2;
  double* slotA = reinterpret_cast<double*>(smem + a.bar_bytes) + (size_t)wib * 2 * CAP;
  double* slotB = slotA + CAP;
  unsigned char* ring = smem + a.bar_bytes + (size_t)NW * 2 * CAP * 8 + (size_t)wib * 2 * STAGE;
  const uint64_t pol_s = policy_evict_first();
  const uint32_t* __restrict__ desc = static_cast<const uint32_t*>(a.desc);

  int64_t kb = 0, ke = 0;
  if (has_tiles) {
    kb = a.warp_begin[w];
    ke = a.warp_begin[w + 1];
  }
  // one stage = tiles k and k + 1 (when k + 1 < ke): val, col_idx, descriptors
  auto issue = [&](int64_t k, int s) {  // lane 0 only
    const uint32_t nt = k + 1 < ke ? 2u : 1u;
    unsigned char* st = ring + (size_t)s * STAGE;
    uint64_t* bar = bars + s;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect(bar, nt * (B * 12 + 128));
    bulk_load(st, a.val + k * B, nt * B * 8, bar, pol_s);
    bulk_load(st + COL_OFF, a.col + k * B, nt * B * 4, bar, pol_s);
    bulk_load(st + DESC_OFF, desc + k * 32, nt * 128, bar, pol_s);
  };
  if (has_tiles && lane == 0) {
    for (int s = 0; s < 2; ++s) mbar_init(bars + s);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    issue(kb, 0);
    if (kb + 2 < ke) issue(kb + 2, 1);
  }
  __syncwarp();

  rows_part<false>(a);
  if (!has_tiles) return;

  double* __restrict__ y = a.y;
  const bool mirrored = mir_on(a.mir);
  auto put_y = [&](int64_t r, double v) {
    y[r] = v;
    if (mirrored) mirror_store(a.mir, r, v);
  };
  int64_t pend_row = -1, first_row = -1;
  double pend_val = 0.0, first_val = 0.0;
  uint32_t tpv = 0;
  int s = 0;
  uint32_t phase = 0;
  // one tile's closes (Algorithm 8) into its slots and its column sum
  auto unpack = [&](uint32_t wd, uint64_t* fr, int* yoff, int* cnt) {
    *fr = __brevll((uint64_t)wd & FMASK) >> (64 - SIG);  // bit j = depth j
    *yoff = (int)(wd >> (kSegBits + SIG));
    *cnt = __popcll(*fr);
  };
  // the fast segmented sum (spmv.cpp:97-105): a shuffle segmented suffix scan
  auto splice = [&](double* slot, uint64_t fr, int yoff, int cnt, double sum) {
    const bool seen = cnt > 0;
    const double red = seen ? slot[yoff] : 0.0;
    const double give = seen ? red : sum;
    double tmp = __shfl_down_sync(kFull, give, 1);
    if (lane == 31) tmp = 0.0;
    const uint32_t hb = __ballot_sync(kFull, seen);
    double acc = tmp;
    if (hb != kFull) {
      const uint64_t above = (uint64_t)hb >> (lane + 1);
      const int end = above ? lane + __ffsll((long long)above) - 1 : 31;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double o = __shfl_down_sync(kFull, acc, d);
        if (lane + d <= end) acc += o;
      }
    }
    if (seen) slot[yoff + cnt] = sum + acc;
  };
  // heads 1..H-2 are final rows; head 0 closes the run carried in, head H-1
  // starts the next (every NF tile has H >= 2)
  auto finish = [&](double* slot, int64_t k, int64_t row, int H) {
    const double c0 = slot[1], cL = slot[H];
    for (int h = lane + 1; h < H - 1; h += 32) put_y(row + h, slot[h + 1]);
    if (k == kb) {
      first_row = row;
      first_val = c0;
    } else if (lane == 0) {
      if (row == pend_row) {
        put_y(pend_row, pend_val + c0);
      } else {
        put_y(pend_row, pend_val);
        put_y(row, c0);
      }
    }
    pend_row = row + H - 1;
    pend_val = cL;
  };

  // the gathers of a pair (the stage holding it has landed)
  double xA[SIG], xB[SIG];
  auto gather = [&](int st_idx, bool two) {
    const int32_t* sc = reinterpret_cast<const int32_t*>(ring + (size_t)st_idx * STAGE + COL_OFF);
#pragma unroll
    for (int u = 0; u < SIG; ++u) xA[u] = ld_x_plain(a.x + sc[u * 32 + lane]);
    if (two) {
#pragma unroll
      for (int u = 0; u < SIG; ++u) xB[u] = ld_x_plain(a.x + sc[B + u * 32 + lane]);
    }
  };
  mbar_wait(bars, 0);
  gather(0, kb + 1 < ke);

  for (int64_t k = kb; k < ke; k += 2) {
    const bool two = k + 1 < ke;
    const int slot = (int)((k - kb) & 31);  // even: tiles slot, slot + 1 of the batch
    if (slot == 0) {
      const int64_t last = a.tile_ptr_len - 1;
      tpv = a.tile_ptr[k + lane < last ? k + lane : last];
    }
    const int64_t rowA = __shfl_sync(kFull, tpv, slot) & 0x7fffffffu;
    const int64_t rowB = __shfl_sync(kFull, tpv, slot + 1) & 0x7fffffffu;
    const unsigned char* st = ring + (size_t)s * STAGE;
    const double* sv = reinterpret_cast<const double*>(st);
    const uint32_t* sd = reinterpret_cast<const uint32_t*>(st + DESC_OFF);
    uint64_t frA, frB = 0;
    int yoffA, cntA, yoffB = 0, cntB = 0;
    unpack(sd[lane], &frA, &yoffA, &cntA);
    if (two) unpack(sd[32 + lane], &frB, &yoffB, &cntB);
    const int HA = __shfl_sync(kFull, yoffA + cntA, 31);
    const int HB = __shfl_sync(kFull, yoffB + cntB, 31);
    // depth loops of both tiles, interleaved (two independent chains)
    double sumA = 0.0, sumB = 0.0;
    double* cpA = slotA + yoffA;
    double* cpB = slotB + yoffB;
#pragma unroll
    for (int j = 0; j < SIG; ++j) {
      if ((frA >> j) & 1ull) {
        *cpA++ = sumA;
        sumA = 0.0;
      }
      sumA = fma(sv[j * 32 + lane], xA[j], sumA);
      if (two) {
        if ((frB >> j) & 1ull) {
          *cpB++ = sumB;
          sumB = 0.0;
        }
        sumB = fma(sv[B + j * 32 + lane], xB[j], sumB);
      }
    }
    __syncwarp();
    // the next pair's gathers go out now: their latency overlaps this pair's
    // splices and write-backs (they land in the registers just drained)
    const int sn = s ^ 1;
    const uint32_t pn = sn == 0 ? phase ^ 1u : phase;
    if (k + 2 < ke) {
      mbar_wait(bars + sn, pn);
      gather(sn, k + 3 < ke);
    }
    // this stage is consumed: refill it with the pair after next
    if (lane == 0 && k + 4 < ke) issue(k + 4, s);
    s = sn;
    phase = pn;
    splice(slotA, frA, yoffA, cntA, sumA);
    if (two) splice(slotB, frB, yoffB, cntB, sumB);
    __syncwarp();
    finish(slotA, k, rowA, HA);
    if (two) finish(slotB, k + 1, rowB, HB);
    __syncwarp();  // the slots are rewritten by the next pair
  }

  // the warp's first and last runs (spmv_kernel.cuh: NF plans have no run of
  // more than two items)
  const int64_t i0 = 2 * (int64_t)w, i1 = i0 + 1;
  if (a.atomic) {  // spmv.cpp:273-295: fp64 atomics into the zeroed y
    if (lane == 0) {
      if (first_val != 0.0) atomicAdd(a.y + first_row, first_val);
      if (pend_val != 0.0) atomicAdd(a.y + pend_row, pend_val);
    }
  } else if (lane == 0) {
    const int s0 = a.run_first[i0], e0 = a.run_last[i0];
    const int s1 = a.run_first[i1], e1 = a.run_last[i1];
    unsigned long long o0 = 0, o1 = 0;
    if (e0 > s0)
      o0 = atomicExch(reinterpret_cast<unsigned long long*>(a.item_val + s0),
                      (unsigned long long)__double_as_longlong(exchangeable(first_val)));
    if (e1 > s1)
      o1 = atomicExch(reinterpret_cast<unsigned long long*>(a.item_val + s1),
                      (unsigned long long)__double_as_longlong(exchangeable(pend_val)));
    if (e0 == s0) {
      write_run(first_row, first_val, a.y, a.first_row, a.first_owned, a.send, a.send_flag,
                a.send_epoch, a.mir);
    } else if (o0 != kSlotIdle && !(s1 == s0 && e1 > s1)) {
      a.item_val[s0] = __longlong_as_double((long long)kSlotIdle);
      write_run(first_row, __longlong_as_double((long long)o0) + first_val, a.y, a.first_row,
                a.first_owned, a.send, a.send_flag, a.send_epoch, a.mir);
    }
    if (e1 == s1) {
      write_run(pend_row, pend_val, a.y, a.first_row, a.first_owned, a.send, a.send_flag,
                a.send_epoch, a.mir);
    } else if (o1 != kSlotIdle) {
      a.item_val[s1] = __longlong_as_double((long long)kSlotIdle);
      write_run(pend_row, __longlong_as_double((long long)o1) + pend_val, a.y, a.first_row,
                a.first_owned, a.send, a.send_flag, a.send_epoch, a.mir);
    }
  }
}

SpmvFn spmv_fn_nf2(int sigma);  // spmv_inst_nf2.cu (sigma 1..kNfMaxSigma)

}  // namespace csr5g
