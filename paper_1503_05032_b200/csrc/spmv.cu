// spmv.cu -- CSR5 SpMV (reference: spmv.cpp:42-124, 224-298).
//
// k_spmv: persistent grid, one warp = one contiguous range of tiles (CSR5
//   tiles are equal-work units, so a static split balances).  Per tile the
//   warp runs Algorithm 8 with lane i = column i (spmv.cpp:61-95): sigma
//   coalesced depth steps of col/val, x gathered through L1/L2, segment
//   closes at each bit flag.  The cross-column splice (fast segmented sum,
//   spmv.cpp:97-105) is a 5-step shuffle segmented suffix scan driven by a
//   ballot of head-bearing lanes -- no shared memory, no scan-and-subtract.
//   Rows wholly inside the warp's range are stored straight to y; only the
//   first and the last row run of each warp can be shared with a neighbour,
//   so each warp emits exactly two (row, partial) items.  Empty rows are
//   zeroed here from the empty_offset gaps (no memset of y).
//   Leading blocks ("rows part") compute the CSR tail rows (spmv.cpp:110-124)
//   and zero leading/trailing empty rows.
// k_calibrate: deterministic merge of the 2*warps+1 items (keys are
//   non-decreasing rows): segmented reduction per warp window, forward walk
//   for runs crossing windows; y[row] = run total.  Atomic mode instead adds
//   items with fp64 atomics into a zeroed y (spmv.cpp:273-295).
#include <climits>

#include "internal.cuh"

namespace csr5g {
namespace {

__device__ __forceinline__ void put_item(const SpmvArgs& a, int64_t idx, int64_t row, double v) {
  if (a.atomic) {
    if (v != 0.0) atomicAdd(a.y + row, v);
  } else {
    a.item_row[idx] = row;
    a.item_val[idx] = v;
  }
}

__device__ void rows_part(const SpmvArgs& a) {
  const int64_t tail_rows = a.m - a.tail_row_begin;
  const int64_t total = a.lead_rows + tail_rows;
  const int64_t stride = (int64_t)a.rows_blocks * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    if (idx < a.lead_rows) {
      a.y[idx] = 0.0;
      continue;
    }
    const int64_t r = a.tail_row_begin + (idx - a.lead_rows);
    int64_t lo = a.row_ptr[r];
    const int64_t hi = a.row_ptr[r + 1];
    if (lo < a.tail_pos) lo = a.tail_pos;
    double s = 0.0;
    for (int64_t q = lo; q < hi; ++q) s = fma(a.val[q - a.pos0], a.x[a.col[q - a.pos0]], s);
    if (a.has_tail_item && r == a.tail_row_begin)
      put_item(a, 2 * (int64_t)a.nwarps, r, s);
    else
      a.y[r] = s;
  }
}

template <typename W>
__global__ void __launch_bounds__(kSpmvThreads) k_spmv(SpmvArgs a) {
  if ((int)blockIdx.x < a.rows_blocks) {
    rows_part(a);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int w = ((int)blockIdx.x - a.rows_blocks) * kSpmvWarpsPerBlock + (threadIdx.x >> 5);
  if (w >= a.nwarps) return;
  const int64_t kb = (int64_t)w * a.pcs / a.nwarps;
  const int64_t ke = (int64_t)(w + 1) * a.pcs / a.nwarps;
  const uint64_t pol_s = policy_evict_first();
  const uint64_t pol_x = policy_evict_last();
  const int sigma = a.sigma;
  const int64_t B = a.B;
  const uint64_t fmask = (1ull << sigma) - 1;
  const W* __restrict__ desc = static_cast<const W*>(a.desc);
  double* __restrict__ y = a.y;

  int64_t pend_row = -1;
  double pend_val = 0.0;
  bool pend_first = true;

  for (int64_t k = kb; k < ke; ++k) {
    const uint32_t tp = a.tile_ptr[k];
    const int64_t tile_row = tp & 0x7fffffffu;
    const bool flagged = (tp >> 31) != 0;
    const int64_t next_row =
        (k + 1 == a.pcs) ? a.next_row_after : (int64_t)(a.tile_ptr[k + 1] & 0x7fffffffu);
    const uint64_t wd = (uint64_t)ld_stream(desc + k * 32 + lane, pol_s);
    const uint64_t fr = __brevll(wd & fmask) >> (64 - sigma);  // bit j = depth j
    const int yoff = (int)(wd >> (kSegBits + sigma));
    const int cnt = __popcll(fr);
    const int H = __shfl_sync(kFull, yoff + cnt, 31);
    const int32_t* __restrict__ eo = flagged ? a.eo + a.eo_ptr[k] : nullptr;

    // rows of heads h and h+1 (h+1 == H means "the next tile's first row")
    auto head_row = [&](int h) -> int64_t { return tile_row + (eo ? (int64_t)eo[h] : (int64_t)h); };
    int64_t defer_lo = 0, defer_hi = 0;
    // zero the empty rows strictly between row(h) and the next head's row
    auto gap = [&](int h, int64_t r) {
      if (!eo && h + 1 < H) return;  // unflagged tile: consecutive heads are adjacent rows
      const int64_t nr = (h + 1 < H) ? head_row(h + 1) : next_row;
      const int64_t lo = r + 1;
      if (nr - lo <= 8) {
        for (int64_t q = lo; q < nr; ++q) y[q] = 0.0;
      } else if (defer_hi == defer_lo) {
        defer_lo = lo;
        defer_hi = nr;
      } else {
        for (int64_t q = lo; q < nr; ++q) y[q] = 0.0;
      }
    };

    const int64_t base = k * B + lane;
    double sum = 0.0, red = 0.0, c0 = 0.0;
    bool seen = false;
    int head = yoff;
    for (int j0 = 0; j0 < sigma; j0 += 8) {
      int32_t c[8];
      double v[8], xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (j0 + u < sigma) {
          c[u] = ld_stream(a.col + base + (int64_t)(j0 + u) * 32, pol_s);
          v[u] = ld_stream(a.val + base + (int64_t)(j0 + u) * 32, pol_s);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j0 + u < sigma) xv[u] = ld_keep(a.x + c[u], pol_x);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u;
        if (j < sigma) {
          if ((fr >> j) & 1ull) {
            if (!seen) {
              red = sum;  // piece continuing the column to the left (spmv.cpp:75-77)
              seen = true;
            } else {      // segment sealed inside this column
              const int64_t r = head_row(head);
              if (head == 0)
                c0 = sum;
              else
                y[r] = sum;
              gap(head, r);
              ++head;
            }
            sum = 0.0;
          }
          sum = fma(v[u], xv[u], sum);
        }
      }
    }
    // ---- splice across columns: tmp[i] = piece handed left by column i+1 ----
    const double give = seen ? red : sum;
    double tmp = __shfl_down_sync(kFull, give, 1);
    if (lane == 31) tmp = 0.0;
    const uint32_t hb = __ballot_sync(kFull, seen);
    const uint64_t above = (uint64_t)hb >> (lane + 1);
    const int end = above ? lane + __ffsll((long long)above) - 1 : 31;
    double acc = tmp;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double o = __shfl_down_sync(kFull, acc, d);
      if (lane + d <= end) acc += o;
    }
    double cL = 0.0;
    int64_t rL = 0;
    if (seen) {
      const int hbh = yoff + cnt - 1;  // head owning this column's bottom piece
      const double blue = sum + acc;
      const int64_t r = head_row(hbh);
      if (hbh == 0) c0 = blue;
      if (hbh == H - 1) {
        cL = blue;
        rL = r;
      }
      if (hbh != 0 && hbh != H - 1) y[r] = blue;
      gap(hbh, r);
    }
    // long empty-row runs: zero cooperatively
    uint32_t dm = __ballot_sync(kFull, defer_hi > defer_lo);
    while (dm) {
      const int src = __ffs(dm) - 1;
      dm &= dm - 1;
      const int64_t lo = __shfl_sync(kFull, defer_lo, src);
      const int64_t hi = __shfl_sync(kFull, defer_hi, src);
      for (int64_t q = lo + lane; q < hi; q += 32) y[q] = 0.0;
    }
    const int L = 31 - __clz(hb);
    c0 = __shfl_sync(kFull, c0, 0);
    cL = __shfl_sync(kFull, cL, L);
    rL = __shfl_sync(kFull, rL, L);

    // ---- row runs across the warp's consecutive tiles ----
    auto flush = [&]() {
      if (lane == 0) {
        if (pend_first)
          put_item(a, 2 * (int64_t)w, pend_row, pend_val);
        else
          y[pend_row] = pend_val;
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
  if (lane == 0) {
    if (pend_first) {
      put_item(a, 2 * (int64_t)w, pend_row, pend_val);
      put_item(a, 2 * (int64_t)w + 1, pend_row, 0.0);
    } else {
      put_item(a, 2 * (int64_t)w + 1, pend_row, pend_val);
    }
  }
}

__device__ __forceinline__ void write_run(int64_t row, double v, double* y, int64_t first_row,
                                          int first_owned, csr5g_partial* send) {
  if (!first_owned && row == first_row) {
    send->row = row;
    send->value = v;
  } else {
    y[row] = v;
  }
}

__global__ void k_calibrate(const int64_t* __restrict__ item_row,
                            const double* __restrict__ item_val, int64_t N, double* __restrict__ y,
                            int64_t first_row, int first_owned, csr5g_partial* send) {
  const int lane = threadIdx.x & 31;
  const int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x - lane;
  if (base >= N) return;
  if (base == 0 && lane == 0) {
    send->row = -1;
    send->value = 0.0;
  }
  __syncwarp();
  const int64_t i = base + lane;
  const bool valid = i < N;
  const int64_t key = valid ? item_row[i] : (LLONG_MAX - lane);
  int64_t prev = __shfl_up_sync(kFull, key, 1);
  if (lane == 0) prev = base > 0 ? item_row[base - 1] : LLONG_MIN;
  const bool start = valid && key != prev;
  const uint32_t sm = __ballot_sync(kFull, start);
  const uint32_t vm = __ballot_sync(kFull, valid);
  const uint64_t above = (uint64_t)sm >> (lane + 1);
  const int end = above ? lane + __ffsll((long long)above) - 1 : 31 - __clz(vm);
  double v = valid ? item_val[i] : 0.0;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double o = __shfl_down_sync(kFull, v, d);
    if (lane + d <= end) v += o;
  }
  const int ls = sm ? 31 - __clz(sm) : -1;
  bool cont = false;
  int64_t rk = 0;
  if (ls >= 0) {
    rk = __shfl_sync(kFull, key, ls);
    cont = (base + 32 < N) && item_row[base + 32] == rk;
  }
  if (start && !(cont && lane == ls)) write_run(key, v, y, first_row, first_owned, send);
  if (cont) {
    double total = __shfl_sync(kFull, v, ls);
    for (int64_t pos = base + 32;; pos += 32) {
      const int64_t q = pos + lane;
      const bool mt = q < N && item_row[q] == rk;
      const uint32_t mm = __ballot_sync(kFull, mt);
      double s = mt ? item_val[q] : 0.0;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(kFull, s, d);
      total += s;
      if (mm != kFull) break;
    }
    if (lane == 0) write_run(rk, total, y, first_row, first_owned, send);
  }
}

__global__ void k_fixup(const csr5g_partial* __restrict__ all, int world, int rank, int64_t row,
                        double* __restrict__ y) {
  double acc = y[row];
  for (int s = rank + 1; s < world; ++s) {
    if (all[s].row != row) break;
    acc += all[s].value;
  }
  y[row] = acc;
}

template <typename W>
int occ(int* bps) {
  CSR5G_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k_spmv<W>, kSpmvThreads, 0));
  if (*bps < 1) *bps = 1;
  return CSR5G_OK;
}

}  // namespace

int spmv_occupancy(bool wide, int* bps) { return wide ? occ<uint64_t>(bps) : occ<uint32_t>(bps); }

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
  a.item_row = h->item_row;
  a.item_val = h->item_val;
  a.send = h->send_ext ? h->send_ext : h->send;
  a.pcs = h->pcs;
  a.pos0 = h->t0 * h->B;
  a.next_row_after = h->next_row_after;
  a.lead_rows = h->lead_rows;
  a.tail_row_begin = h->tail_row_begin;
  a.tail_pos = h->tail_pos;
  a.m = in.m;
  a.first_row = h->first_row;
  a.first_owned = h->first_owned;
  a.has_tail_item = h->has_tail_item;
  a.sigma = (int)in.sigma;
  a.B = (int)h->B;
  a.nwarps = h->nwarps;
  a.rows_blocks = h->rows_blocks;
  a.atomic = atomic;
  const int grid = h->rows_blocks + h->tile_blocks;
  if (ev0) CSR5G_CUDA(cudaEventRecord(ev0, stream));
  if (grid > 0) {
    if (h->wide)
      k_spmv<uint64_t><<<grid, kSpmvThreads, 0, stream>>>(a);
    else
      k_spmv<uint32_t><<<grid, kSpmvThreads, 0, stream>>>(a);
    CSR5G_CUDA(cudaGetLastError());
  }
  if (ev1) CSR5G_CUDA(cudaEventRecord(ev1, stream));
  const int64_t items = 2 * (int64_t)h->nwarps + (h->has_tail_item ? 1 : 0);
  if (!atomic && items > 0) {
    k_calibrate<<<(unsigned)((items + 255) / 256), 256, 0, stream>>>(
        h->item_row, h->item_val, items, d_y, h->first_row, h->first_owned, a.send);
    CSR5G_CUDA(cudaGetLastError());
  } else if (!atomic) {
    const csr5g_partial none{-1, 0.0};
    CSR5G_CUDA(cudaMemcpyAsync(a.send, &none, sizeof none, cudaMemcpyHostToDevice, stream));
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
