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

#include "spmv_kernel.cuh"
#include "spmv_nf2.cuh"

namespace csr5g {
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

// The plan's kernel: the compile-time gather mode when the plan's x path has
// one (spmv_kernel.cuh, GM), else the runtime-switch variant.  CSR5G_GM=0
// forces the runtime variant (A/B).
int gather_mode(const Handle* h) {
  const char* e = std::getenv("CSR5G_GM");
  if (e && std::atoi(e) == 0) return 0;
  // the profiling / experiment knobs GM 4 compiles out
  for (const char* k : {"CSR5G_STREAM_ONLY", "CSR5G_YHINT", "CSR5G_EARLY"})
    if (std::getenv(k) && !h->vr) return 0;
  if (h->vr) {
    if (h->n_hot > 0) return h->x_mode == 5 && h->hot_l1 ? 3 : h->x_mode == 1 && !h->hot_l1 ? 5 : 0;
    return h->x_mode == 1 ? 1 : h->x_mode == 8 ? 2 : 0;
  }
  return h->x_mode == 4 ? 4 : 0;
}

SpmvFn spmv_fn(int sigma, bool vr, bool nf, int gm) {
  SpmvFn f = nullptr;
  if ((gm >= 1 && gm <= 3 || gm == 5) && vr) f = spmv_fn_vr_gm(sigma, gm);
  if (gm == 4 && !vr) f = spmv_fn_local_gm4(sigma, nf && sigma <= kNfMaxSigma);
  if (f) return f;
  if (nf && !vr && sigma <= kNfMaxSigma) return spmv_fn_nf(sigma);
  if (vr) return spmv_fn_vr(sigma);
  return spmv_fn_general(sigma);
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
  h->nf = nf_env != 0 && !h->vr && !h->maybe_long && sigma <= kNfMaxSigma && h->pcs > 0 &&
          h->eo_entries == 0 &&
          h->max_heads < std::min<int64_t>(h->B, kClosedSlots);
  const int64_t tile_bytes = h->B * (h->vr ? 4 : 12) + 32 * wbytes;
  const int stage_bytes = (int)((tile_bytes + 127) / 128 * 128);
  const int closed_bytes = (int)(std::min<int64_t>(h->B, kClosedSlots) * 8);
  int budget = !random ? 226 * 1024 : 104 * 1024;
  h->x_mode = random ? 1 : 4;  // random: no L1 allocation; local: plain ld.global.nc
  if (h->vr) {
    // VR plans: a 2-stage col_idx ring is ~2-4 KB per warp, so warps are
    // bounded by the thread cap or by how many misses the memory system
    // absorbs: with x larger than L2 fewer warps win (R-MAT s24, x 134 MB:
    // 6/8/10/12 warps -> 1.62/1.50/1.45/1.55 ms), with x inside L2 the most
    // (mixed 2^23, x 67 MB: 11/12/16 warps -> 0.514/0.505/0.469 ms)
    int l2 = 0;
    CSR5G_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->device));
    const double xb = (double)h->info.n * 8.0;
    budget = xb > 0.75 * (double)l2 ? 60 * 1024 : 72 * 1024;
    // with hot-column staging most gathers hit the dense staged values in L2
    // and more warps win again: R-MAT s24 10 / 13 / 16 warps (budget 60 / 80 /
    // 100 KB) -> 1.45 / 1.37 / 1.28 ms
    if (h->n_hot > 0) {
      budget = 100 * 1024;
      h->x_mode = 5;  // staged hot values L1-allocated, cold ones 64-byte prefetched (GM 3)
    }
    // x several times the L2 (R-MAT s26/s27: 537 MB / 1.07 GB): the gathers
    // are DRAM-random-access bound.  Issued in CSR order (lane L fetches the
    // tile's logical entry u*32 + L, exchanged into the lane-per-column order
    // through shared memory) with a 64-byte L2 prefetch size, and 12 warps:
    // R-MAT s27 38.8 -> 28.3 ms, s26 15.3 -> 11.6 ms; at s25 (268 MB) and
    // below the plain order wins (4.19 vs 4.48 ms), so the switch sits at
    // 3x the L2 (profiles/r02_csr_order_gathers.txt)
    // With hot-column staging (hotx.cu) most gathers read the dense staged
    // values instead, and lane order with the 64-byte prefetch on the cold
    // rest wins: R-MAT s27 (hot set 64 MB) x_mode 8 / 1 / 5 = 16.4 / 15.6 /
    // 14.7 ms, 13.0 with the hot values allocated in L1
    // (profiles/r02_hot_sweep.txt)
    if (xb > 3.0 * (double)l2) {
      h->x_mode = h->n_hot > 0 ? 5 : 8;
      budget = 120 * 1024;
    }
  }
  if (const char* e = std::getenv("CSR5G_BUDGET_KB")) budget = std::atoi(e) * 1024;  // experiments
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
  h->gm = gather_mode(h);
  int nw = spmv_threads_of(sigma, h->vr, h->nf, h->gm) / 32,
      stages = random || h->nf ? 2 : 4;
  // one mbarrier per warp and stage at the start, 128-byte aligned
  auto bars = [](int w, int st) { return (w * st * 8 + 127) / 128 * 128; };
  // x_mode 7/8 (CSR-order gathers, VR only) need a sigma x 33 exchange buffer per warp
  if ((h->x_mode == 7 || h->x_mode == 8) && !h->vr) h->x_mode = 1;
  const int xex_bytes = (h->x_mode == 7 || h->x_mode == 8) ? sigma * 33 * 8 : 0;
  auto need = [&](int w, int st) {
    return bars(w, st) + w * (closed_bytes + kEoSlots * 4 + st * stage_bytes + xex_bytes);
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
  // NF plans at sigma <= 8 may run the two-tiles-per-iteration kernel
  // (spmv_nf2.cuh, opt-in CSR5G_NF2=1): measured no faster on the Laplacian
  // 1000^2 (21.5 vs 20.7 us; both bottom out near 20.4 us), kept as a tested
  // alternative
  h->nf2 = false;
  if (h->nf && sigma <= kNfMaxSigma && !h->wide) {
    const char* e = std::getenv("CSR5G_NF2");
    if (e && std::atoi(e) == 1) {
      const int cap = (h->max_heads + 3) / 2 * 2;  // H + 1 slots, even (16-byte ring alignment)
      const int stage = (int)((2 * h->B * 12 + 64 * 4 + 127) / 128 * 128);
      const int per_warp = 2 * cap * 8 + 2 * stage;
      int nw2 = kNf2Threads / 32;
      if (const char* q = std::getenv("CSR5G_NW")) nw2 = std::max(1, std::min(nw2, std::atoi(q)));
      while (nw2 > 1 && bars(nw2, 2) + nw2 * per_warp > 226 * 1024) --nw2;
      if (bars(nw2, 2) + nw2 * per_warp <= 226 * 1024) {
        h->nf2 = true;
        h->nf2_slots = cap;
        nw = nw2;
        stages = 2;
        h->warps_per_block = nw;
        h->stages = 2;
        h->stage_bytes = stage;
        h->bar_bytes = bars(nw, 2);
        h->smem_bytes = bars(nw, 2) + nw * per_warp;
        int max_smem = 0;
        CSR5G_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor,
                                          h->device));
        h->carveout_pct = std::min(100, (int)((100LL * (h->smem_bytes + 1024) + max_smem - 1) / max_smem));
      }
    }
  }
  const int64_t max_warps = (int64_t)sms * nw;
  h->nwarps = (int)std::min<int64_t>(max_warps, h->pcs);
  h->tile_blocks = (h->nwarps + nw - 1) / nw;
  return CSR5G_OK;
}

// Kernel attributes as the handle's plan needs them.  The dynamic
// shared-memory limit only ever rises (a concurrent launch of the same kernel
// for a plan with more shared memory cannot lower it under another thread's
// launch); the carveout is a preference and follows the latest plan.
int func_attrs(const void* fn, int device, int smem, int carve) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, std::pair<int, int>> cur;
  std::lock_guard<std::mutex> lock(mu);
  auto& c = cur.try_emplace({fn, device}, std::make_pair(-1, -1)).first->second;
  if (smem > c.first) {
    CSR5G_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    c.first = smem;
  }
  if (carve >= 0 && carve != c.second) {
    CSR5G_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    c.second = carve;
  }
  return CSR5G_OK;
}

// The scratch set of `stream` (the reference's per-worker workspaces,
// spmv.hpp:27-38): the handle's own arrays for the first stream, sets
// allocated stream-ordered for others, at most kMaxStreamScratch of them --
// beyond that the least recently used set moves to the new stream, which
// first waits for the set's last SpMV (an event recorded after every launch),
// so a set is never shared by two kernels in flight.  (A stream destroyed and
// re-created at the same address with its last SpMV still running would
// share its set: the caller's stream lifetime is assumed, as for any
// per-stream workspace.)
int scratch_for(Handle* h, cudaStream_t stream, double** iv, int32_t** rc, double** sp,
                double** lp, int32_t** lc, double** xh) {
  std::lock_guard<std::mutex> lock(h->scratch_mu);
  StreamScratch* x = nullptr;
  for (StreamScratch& s : h->scratch)
    if (s.stream == stream) x = &s;
  if (!x && h->scratch.empty()) {
    h->scratch.push_back(StreamScratch{stream, h->item_val, h->run_cnt, h->spill, h->lparts,
                                       h->lcnt, h->xh});
    h->scratch.back().owned = false;
    x = &h->scratch.back();
  }
  bool moved = false;  // the set changes hands: wait for its previous user
  if (!x && h->scratch.size() >= kMaxStreamScratch) {
    x = &h->scratch[0];
    for (StreamScratch& s : h->scratch)
      if (s.last_use < x->last_use) x = &s;
    x->stream = stream;
    moved = true;
  }
  if (!x) {
    const size_t items = 2 * (size_t)h->nwarps + 1;
    const size_t spill = (size_t)std::max(h->nwarps, 1) * (size_t)(h->B + 1);
    StreamScratch n{stream, nullptr, nullptr, nullptr};
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&n.item_val), items * 8, stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(n.item_val, 0xff, items * 8, stream);  // idle slots
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&n.run_cnt), items * 4, stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(n.run_cnt, 0, items * 4, stream);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&n.spill), spill * 8, stream);
    if (e == cudaSuccess && h->long_cap > 0) {
      e = cudaMallocAsync(reinterpret_cast<void**>(&n.lparts), h->long_slots * 8, stream);
      if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&n.lcnt), h->long_cap * 4, stream);
      if (e == cudaSuccess) e = cudaMemsetAsync(n.lcnt, 0, h->long_cap * 4, stream);
    }
    if (e == cudaSuccess && h->n_hot > 0)
      e = cudaMallocAsync(reinterpret_cast<void**>(&n.xh), h->n_hot * 8, stream);
    if (e != cudaSuccess) {
      for (void* p : {(void*)n.item_val, (void*)n.run_cnt, (void*)n.spill, (void*)n.lparts,
                      (void*)n.lcnt, (void*)n.xh})
        if (p) cudaFreeAsync(p, stream);
      return cuda_fail(e, "per-stream SpMV scratch");
    }
    h->scratch.push_back(n);
    x = &h->scratch.back();
  }
  if (!x->done) CSR5G_CUDA(cudaEventCreateWithFlags(&x->done, cudaEventDisableTiming));
  // (inside a stream capture the graph's own ordering serialises the kernels;
  // an event recorded outside it may not be waited on there)
  if (moved) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CSR5G_CUDA(cudaStreamIsCapturing(stream, &cap));
    if (cap == cudaStreamCaptureStatusNone) CSR5G_CUDA(cudaStreamWaitEvent(stream, x->done, 0));
  }
  x->last_use = ++h->scratch_clock;
  *iv = x->item_val;
  *rc = x->run_cnt;
  *sp = x->spill;
  *lp = x->lparts;
  *lc = x->lcnt;
  *xh = x->xh;
  return CSR5G_OK;
}

// after the SpMV kernel of `stream`: its scratch set is free again from here
int scratch_done(Handle* h, cudaStream_t stream) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CSR5G_CUDA(cudaStreamIsCapturing(stream, &cap));
  if (cap != cudaStreamCaptureStatusNone) return CSR5G_OK;
  std::lock_guard<std::mutex> lock(h->scratch_mu);
  for (StreamScratch& s : h->scratch)
    if (s.stream == stream && s.done) CSR5G_CUDA(cudaEventRecord(s.done, stream));
  return CSR5G_OK;
}

bool pdl_env() {  // CSR5G_PDL=0: launch the tile kernel after the fill completes (A/B)
  static const bool on = [] {
    const char* e = std::getenv("CSR5G_PDL");
    return !e || std::atoi(e) != 0;
  }();
  return on;
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
  a.col = h->col_x ? h->col_x : h->col;  // execution col_idx (hot columns renumbered)
  a.val = h->val;
  a.x = d_x;
  a.y = d_y;
  double* xh = nullptr;
  if (int rc = scratch_for(h, stream, &a.item_val, &a.run_cnt, &a.spill, &a.lparts, &a.lcnt, &xh))
    return rc;
  a.xh = h->n_hot > 0 ? xh : nullptr;
  a.cold_pol = h->cold_pol;
  a.hot_l1 = h->hot_l1;
  a.has_long = h->long_cap > 0 && !atomic;
  a.t0 = h->t0;
  a.ltag = h->ltag;
  a.lrow = h->lrow;
  a.ltf = h->ltf;
  a.lnp = h->lnp;
  a.lbase = h->lbase;
  a.tail_long = h->nlong_d ? reinterpret_cast<const int32_t*>(h->nlong_d + 1) : nullptr;
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
  // the hot columns' x values for this call (inside the timed kernel span)
  if (grid > 0 && a.xh)
    if (int rc = launch_xhot_fill(h, d_x, xh, stream)) return rc;
  if (grid > 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = h->smem_bytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int nattr = 0;
    // staged plans: the tile kernel launches while k_xhot_fill drains
    // (programmatic dependent launch) and waits for it only before its first
    // gather (griddepcontrol.wait, spmv_kernel.cuh); the ring prologue and the
    // rows part overlap the fill
    if (a.xh && pdl_env()) {
      attr[nattr].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[nattr].val.programmaticStreamSerializationAllowed = 1;
      ++nattr;
      a.pdl = 1;
    }
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
      attr[nattr].id = cudaLaunchAttributeAccessPolicyWindow;
      attr[nattr].val.accessPolicyWindow.base_ptr = const_cast<double*>(d_x);
      attr[nattr].val.accessPolicyWindow.num_bytes = xb;
      attr[nattr].val.accessPolicyWindow.hitRatio =
          xb ? std::min(1.0f, (float)max_persist / (float)xb) : 1.0f;
      attr[nattr].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      attr[nattr].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      ++nattr;
    }
    if (nattr) {
      cfg.attrs = attr;
      cfg.numAttrs = nattr;
    }
    a.nf2_slots = h->nf2_slots;
    const SpmvFn fn = h->nf2 ? spmv_fn_nf2(a.sigma) : spmv_fn(a.sigma, h->vr, h->nf, h->gm);
    if (int rc = func_attrs((const void*)fn, h->device, h->smem_bytes, h->carveout_pct)) return rc;
    CSR5G_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
  }
  if (ev1) CSR5G_CUDA(cudaEventRecord(ev1, stream));
  if (grid > 0)
    if (int rc = scratch_done(h, stream)) return rc;
  // the rows shared between warps were merged inside the kernel
  // (resolve_item); a handle with nothing to multiply has no record
  if (!atomic && items == 0 && grid == 0) {  // no record: row -1 (all ones), value 0.0
    CSR5G_CUDA(cudaMemsetAsync(&a.send->row, 0xff, sizeof(int64_t), stream));
    CSR5G_CUDA(cudaMemsetAsync(&a.send->value, 0, sizeof(double), stream));
  }
  return CSR5G_OK;
}

// One tile through the trace instantiation of the general kernel (one warp,
// a two-stage ring): every head's row and final value (csr5g_spmv_tile).
int launch_tile_trace(Handle* h, int64_t k, const double* d_x, int64_t* d_rows, double* d_vals,
                      int32_t* d_count, cudaStream_t stream) {
  CSR5G_CUDA(cudaSetDevice(h->device));
  const int sigma = (int)h->info.sigma;
  const int wbytes = h->wide ? 8 : 4;
  const int stage_bytes = (int)((h->B * 12 + 32 * wbytes + 127) / 128 * 128);
  const int closed_bytes = (int)(std::min<int64_t>(h->B, kClosedSlots) * 8);
  const int stages = 2, bar_bytes = 128;
  const int smem = bar_bytes + closed_bytes + kEoSlots * 4 + stages * stage_bytes;
  double* spill = nullptr;
  CSR5G_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&spill), sizeof(double) * (h->B + 1), stream));
  SpmvArgs a{};
  a.row_ptr = h->row_ptr;
  a.tile_ptr = h->tile_ptr;
  a.desc = h->desc;
  a.eo_ptr = h->eo_ptr;
  a.eo = h->eo;
  a.col = h->col;
  a.val = h->val;
  a.x = d_x;
  a.spill = spill;
  a.pcs = h->pcs;
  a.pos0 = h->t0 * h->B;
  a.next_row_after = h->next_row_after;
  a.m = h->info.m;
  a.tile_ptr_len = h->info.tile_ptr_len;
  a.sigma = sigma;
  a.B = (int)h->B;
  a.nwarps = 1;
  a.stages = stages;
  a.stage_bytes = stage_bytes;
  a.bar_bytes = bar_bytes;
  a.x_mode = 4;
  a.x_frac = 1.0f;
  a.trace_tile = k;
  a.trace_row = d_rows;
  a.trace_val = d_vals;
  a.trace_count = d_count;
  const SpmvFn fn = spmv_fn_trace(sigma);
  if (!fn) return fail(CSR5G_EINVAL, "csr5g: no trace kernel for sigma " + std::to_string(sigma));
  if (int rc = func_attrs((const void*)fn, h->device, smem, -1)) return rc;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  CSR5G_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
  CSR5G_CUDA(cudaFreeAsync(spill, stream));
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

