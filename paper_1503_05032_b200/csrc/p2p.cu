// p2p.cu -- NVLink P2P boundary exchange of the multi-GPU driver.
//
// The reference has no distributed backend; this is the shard fix-up the
// north star names: "fixes up the one or two boundary rows per shard with
// NVLink P2P adds".  A row whose nonzeros straddle a shard edge gets one
// partial from every shard it touches; its owner is the shard holding its
// first nonzero (mg.py).  Shard r sends at most one partial (its first row,
// when it does not own it) to one static destination, and receives partials
// from a contiguous range of later shards (a row can span whole shards).
//
// Every rank owns one mailbox in its own HBM (cudaMalloc, exported with a CUDA
// IPC handle, opened by every peer with peer access over NVLink):
//   slot[g]  csr5g_partial  the record shard g stored here (remote store)
//   ready[g] u32            epoch of the call that stored slot[g]
//   ack      u32            epoch of the last call whose record the destination consumed
//   err      u32            protocol violations seen by k_fixup_p2p (tests read it)
// Per call (epoch e, host counter, one per binding):
//   sender r:  stream-wait ack >= e-1 (the owner consumed the previous record;
//              single-buffered slot), then the SpMV, whose calibration stores the
//              record into dest's slot[r], fences at system scope and stores
//              ready[r] = e with release semantics (spmv.cu write_run).
//   owner o:   stream-wait ready[g] >= e for every sender g (cuStreamWaitValue32
//              on LOCAL memory: the front end waits, no SM spins), then
//              k_fixup_p2p adds the partials to y[last_row] in shard order
//              (deterministic) and stores ack = e into every sender's mailbox.
// No collective and no host synchronisation per call; the transfers are one
// 16-byte store plus one flag each way per shard edge.  Ranks sharing one GPU
// (functional tests) must not rely on stream waits across processes: mg.py
// then separates the two phases with a host barrier, so every wait is already
// satisfied when it is enqueued (B200_PROFILING: no cross-rank waits on one GPU).
//
// NVLS variant of the fused mode (csr5g_mailbox_mcast_*): the x ping-pong of
// every rank is bound to one NVSwitch multicast object; a kernel's mirror
// store is a single multimem.st to the multicast mapping, which the switch
// replicates to every rank's copy -- 8 bytes out per value instead of
// 8 * (G - 1).  The flags stay peer-to-peer.  Built only where the device
// reports multicast support; any failure leaves the peer-store path.
//
// Fused iterative mode (y -> x, square A).  Instead of an all-gather of the
// owned y ranges after the SpMV, every kernel that stores a final y value
// (tile write-back, tail rows, calibration, fix-up) also stores it into each
// peer's next-x buffer over NVLink (Mirrors, internal.cuh): the exchange
// rides on the SpMV's own stores and overlaps its HBM stream.  Each mailbox
// carries the two x buffers of the ping-pong (x_k = vec[k & 1]) and an
// xready[g] flag per rank.  Iteration k on rank r:
//   wait xready[g] >= k for every active peer g (their rows of x_k landed;
//   also: they finished iteration k-1, so nobody still reads the buffer r is
//   about to overwrite on them), SpMV x_k -> y = vec[(k+1) & 1] with mirrors,
//   boundary fix-up (mirrored), then k_signal: system fence and
//   xready[r] = k + 1 on every peer.
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <type_traits>

#include "internal.cuh"

namespace csr5g {

constexpr int kMaxWorld = 64;

struct MailboxDev {
  csr5g_partial slot[kMaxWorld];
  uint32_t ready[kMaxWorld];
  uint32_t xready[kMaxWorld];  // iteration whose x rows rank g has stored here
  uint32_t ack;
  uint32_t err;
};
constexpr size_t kVecOffset = 4096;  // x buffers follow the header in one allocation
static_assert(sizeof(MailboxDev) <= kVecOffset, "mailbox header");

struct Mcast;  // NVSwitch multicast of the x ping-pong (end of this file)

struct Mailbox {
  int device = 0, world = 0, rank = 0;
  int64_t vec_len = 0;                    // x buffers (iterative mode), 0 = none
  Mcast* mc = nullptr;                    // multicast x buffers (end of this file), or none
  double* mc_local = nullptr;             // ... their unicast mapping here
  double* mc_multi = nullptr;             // ... and the multicast mapping (every rank's copy)
  MailboxDev* local = nullptr;            // this rank's mailbox (own HBM)
  MailboxDev* peer[kMaxWorld] = {};       // every rank's mailbox, mapped here
  bool ipc_opened[kMaxWorld] = {};
  uint32_t** d_peer_ack = nullptr;        // device table: &peer[g]->ack
  uint32_t** d_peer_xready = nullptr;     // device table: &peer[g]->xready[rank]
  double* vec(const MailboxDev* d, int64_t which) const {
    if (d == local && mc_local) return mc_local + (which & 1) * vec_len;
    return reinterpret_cast<double*>(reinterpret_cast<char*>(const_cast<MailboxDev*>(d)) +
                                     kVecOffset) +
           (which & 1) * vec_len;
  }
};

void mcast_free(Mailbox* m);  // multicast teardown (end of this file)

struct Binding {
  Mailbox* mb = nullptr;
  int dest = -1, sb = 0, se = 0, active = 1;
  uint32_t epoch = 0;
  int64_t last_iter = -1;  // iterative mode: steps run 0, 1, 2, ... on every rank
};

void free_binding(Binding* b) { delete b; }

namespace {

using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

int wait_value_fn(WaitValueFn* out) {
  static WaitValueFn fn = nullptr;
  static cudaError_t rc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaError_t e = cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &p, 12000,
                                                     cudaEnableDefault, &q);
    if (e == cudaSuccess && q != cudaDriverEntryPointSuccess) e = cudaErrorNotSupported;
    fn = reinterpret_cast<WaitValueFn>(p);
    return e;
  }();
  if (rc != cudaSuccess) return cuda_fail(rc, "cudaGetDriverEntryPoint(cuStreamWaitValue32)");
  *out = fn;
  return CSR5G_OK;
}

// The stream's front end waits until *addr >= value (cyclic compare); no SM spins.
int stream_wait_geq(cudaStream_t s, const uint32_t* addr, uint32_t value) {
  WaitValueFn fn = nullptr;
  if (int rc = wait_value_fn(&fn)) return rc;
  const CUresult r = fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), value,
                        CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS)
    return fail(CSR5G_ECUDA, "cuStreamWaitValue32 failed (CUresult " + std::to_string((int)r) + ")");
  return CSR5G_OK;
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One thread: y[row] += partials of senders [sb, se) in shard order (mirrored
// to the peers' next x in the iterative mode), then ack every sender.
__global__ void k_fixup_p2p(MailboxDev* mb, uint32_t* const* peer_ack, int sb, int se,
                            int64_t row, double* __restrict__ y, uint32_t epoch, Mirrors mir) {
  double acc = y[row];
  for (int g = sb; g < se; ++g) {
    if (ld_acquire_sys(&mb->ready[g]) != epoch) atomicOr(&mb->err, 1u);
    const volatile csr5g_partial* r = &mb->slot[g];
    if (r->row != row) atomicOr(&mb->err, 2u);
    else acc += r->value;
  }
  y[row] = acc;
  mirror_store(mir, row, acc);
  __threadfence_system();
  for (int g = sb; g < se; ++g) st_release_sys(peer_ack[g], epoch);
}

// Iterative mode: this rank's rows of x_{k+1} are stored on every peer ->
// raise xready[rank] = k + 1 there (after a system-scope fence; the SpMV,
// calibration and fix-up kernels that stored the rows precede it in the stream).
__global__ void k_signal(uint32_t* const* peer_xready, int n, uint32_t value) {
  __threadfence_system();
  for (int g = threadIdx.x; g < n; g += blockDim.x)
    if (peer_xready[g]) st_release_sys(peer_xready[g], value);
}

}  // namespace

int mg_post(Handle* h, const double* d_x, double* d_y, cudaStream_t stream, cudaEvent_t ev0,
            cudaEvent_t ev1) {
  Binding* b = h->mg;
  if (!b) return fail(CSR5G_EINVAL, "csr5g: shard is not bound to a mailbox (csr5g_mg_bind)");
  CSR5G_CUDA(cudaSetDevice(h->device));
  ++b->epoch;
  csr5g_partial* const saved = h->send_ext;
  if (b->dest >= 0) {
    if (int rc = stream_wait_geq(stream, &b->mb->local->ack, b->epoch - 1)) return rc;
    h->send_ext = &b->mb->peer[b->dest]->slot[b->mb->rank];
    h->send_flag = &b->mb->peer[b->dest]->ready[b->mb->rank];
  } else {
    h->send_ext = nullptr;
    h->send_flag = nullptr;
  }
  h->send_epoch = b->epoch;
  const int rc = launch_spmv(h, d_x, d_y, CSR5G_MODE_DETERMINISTIC, stream, ev0, ev1);
  h->send_ext = saved;
  h->send_flag = nullptr;
  return rc;
}

int mg_fixup(Handle* h, double* d_y, cudaStream_t stream) {
  Binding* b = h->mg;
  if (!b) return fail(CSR5G_EINVAL, "csr5g: shard is not bound to a mailbox (csr5g_mg_bind)");
  if (b->se <= b->sb) return CSR5G_OK;
  CSR5G_CUDA(cudaSetDevice(h->device));
  for (int g = b->sb; g < b->se; ++g)
    if (int rc = stream_wait_geq(stream, &b->mb->local->ready[g], b->epoch)) return rc;
  k_fixup_p2p<<<1, 1, 0, stream>>>(b->mb->local, b->mb->d_peer_ack, b->sb, b->se, h->last_row,
                                   d_y, b->epoch, h->mir);
  CSR5G_CUDA(cudaGetLastError());
  return CSR5G_OK;
}

namespace {

int iter_check(Handle* h) {
  Binding* b = h->mg;
  if (!b) return fail(CSR5G_EINVAL, "csr5g: shard is not bound to a mailbox (csr5g_mg_bind)");
  Mailbox* m = b->mb;
  if (m->vec_len <= 0) return fail(CSR5G_EINVAL, "csr5g: mailbox has no x buffers (vec_len = 0)");
  if (m->vec_len != h->info.m || h->info.m != h->info.n)
    return fail(CSR5G_EINVAL, "csr5g: iterative mode needs a square matrix and vec_len = m");
  if (b->active - 1 > kMaxMirror)
    return fail(CSR5G_EINVAL, "csr5g: iterative P2P mode supports at most " +
                                  std::to_string(kMaxMirror + 1) + " active ranks");
  for (int g = 0; g < b->active; ++g)
    if (!m->peer[g]) return fail(CSR5G_EINVAL, "csr5g: iterative mode needs every active peer linked");
  return CSR5G_OK;
}

// Peer next-x buffers of iteration it (skip_row: an owner's boundary row is
// mirrored by its fix-up, with the total).
Mirrors iter_mirrors(Handle* h, int64_t it) {
  Binding* b = h->mg;
  Mailbox* m = b->mb;
  Mirrors mir{};
  if (m->mc_multi) {  // one multimem store per value reaches every rank's copy
    mir.mc = m->mc_multi + ((it + 1) & 1) * m->vec_len;
  } else {
    for (int g = 0; g < b->active; ++g)
      if (g != m->rank) mir.p[mir.n++] = m->vec(m->peer[g], it + 1);
  }
  mir.skip_row = b->se > b->sb ? h->last_row : -1;
  return mir;
}

}  // namespace

int mg_iter_post(Handle* h, int64_t it, cudaStream_t stream, cudaEvent_t ev0, cudaEvent_t ev1) {
  if (int rc = iter_check(h)) return rc;
  Binding* b = h->mg;
  Mailbox* m = b->mb;
  // the xready flags and the buffer parity assume consecutive steps from 0
  if (it != b->last_iter + 1)
    return fail(CSR5G_EINVAL, "csr5g: iterative step " + std::to_string(it) + " after step " +
                                  std::to_string(b->last_iter) + " (steps run 0, 1, 2, ...)");
  b->last_iter = it;
  CSR5G_CUDA(cudaSetDevice(h->device));
  for (int g = 0; g < b->active; ++g)
    if (g != m->rank)
      if (int rc = stream_wait_geq(stream, &m->local->xready[g], (uint32_t)it)) return rc;
  h->mir = iter_mirrors(h, it);
  const int rc = mg_post(h, m->vec(m->local, it), m->vec(m->local, it + 1), stream, ev0, ev1);
  h->mir = Mirrors{};
  return rc;
}

int mg_iter_finish(Handle* h, int64_t it, cudaStream_t stream) {
  if (int rc = iter_check(h)) return rc;
  Binding* b = h->mg;
  Mailbox* m = b->mb;
  h->mir = iter_mirrors(h, it);
  h->mir.skip_row = -1;
  int rc = mg_fixup(h, m->vec(m->local, it + 1), stream);
  h->mir = Mirrors{};
  if (rc) return rc;
  k_signal<<<1, 32, 0, stream>>>(m->d_peer_xready, b->active, (uint32_t)(it + 1));
  CSR5G_CUDA(cudaGetLastError());
  return CSR5G_OK;
}

}  // namespace csr5g

using namespace csr5g;

struct csr5g_mailbox_s {
  Mailbox* m;
};

struct csr5g_matrix_s {
  Handle* h;
};

namespace {

int refresh_peer_table(Mailbox* m) {
  uint32_t* acks[kMaxWorld] = {};
  uint32_t* xr[kMaxWorld] = {};
  for (int g = 0; g < m->world; ++g) {
    acks[g] = m->peer[g] ? &m->peer[g]->ack : nullptr;
    xr[g] = (m->peer[g] && g != m->rank) ? &m->peer[g]->xready[m->rank] : nullptr;
  }
  CSR5G_CUDA(cudaMemcpy(m->d_peer_ack, acks, sizeof(uint32_t*) * m->world, cudaMemcpyHostToDevice));
  CSR5G_CUDA(cudaMemcpy(m->d_peer_xready, xr, sizeof(uint32_t*) * m->world, cudaMemcpyHostToDevice));
  return CSR5G_OK;
}

}  // namespace

extern "C" {

int csr5g_mailbox_create(int device, int32_t world, int32_t rank, int64_t vec_len,
                         csr5g_mailbox* out) {
  if (!out) return fail(CSR5G_EINVAL, "csr5g: out is NULL");
  *out = nullptr;
  if (world < 1 || world > kMaxWorld)
    return fail(CSR5G_EINVAL, "csr5g: world must be in [1, " + std::to_string(kMaxWorld) + "]");
  if (rank < 0 || rank >= world) return fail(CSR5G_EINVAL, "csr5g: rank outside [0, world)");
  if (vec_len < 0) return fail(CSR5G_EINVAL, "csr5g: negative vec_len");
  CSR5G_CUDA(cudaSetDevice(device));
  auto* m = new Mailbox;
  m->device = device;
  m->world = world;
  m->rank = rank;
  m->vec_len = vec_len;
  void* base = nullptr;
  cudaError_t e = cudaMalloc(&base, kVecOffset + sizeof(double) * 2 * (size_t)vec_len);
  m->local = static_cast<MailboxDev*>(base);
  if (e == cudaSuccess) e = cudaMemset(m->local, 0, sizeof(MailboxDev));
  if (e == cudaSuccess) e = cudaMalloc(&m->d_peer_ack, sizeof(uint32_t*) * kMaxWorld);
  if (e == cudaSuccess) e = cudaMalloc(&m->d_peer_xready, sizeof(uint32_t*) * kMaxWorld);
  if (e != cudaSuccess) {
    cudaFree(m->local);
    cudaFree(m->d_peer_ack);
    cudaFree(m->d_peer_xready);
    delete m;
    return cuda_fail(e, "csr5g_mailbox_create");
  }
  // every slot starts as "no record" (row -1)
  csr5g_partial none[kMaxWorld];
  for (auto& r : none) r = csr5g_partial{-1, 0.0};
  auto undo = [&](int rc) {  // every buffer allocated above, on any later failure
    cudaFree(m->local);
    cudaFree(m->d_peer_ack);
    cudaFree(m->d_peer_xready);
    delete m;
    return rc;
  };
  if ((e = cudaMemcpy(m->local->slot, none, sizeof none, cudaMemcpyHostToDevice)) != cudaSuccess)
    return undo(cuda_fail(e, "csr5g_mailbox_create: slots"));
  m->peer[rank] = m->local;
  if (int rc = refresh_peer_table(m)) return undo(rc);
  *out = new csr5g_mailbox_s{m};
  return CSR5G_OK;
}

int csr5g_mailbox_vector(csr5g_mailbox mb, int32_t which, double** d_vec) {
  if (!mb || !d_vec) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  if (mb->m->vec_len <= 0) return fail(CSR5G_EINVAL, "csr5g: mailbox has no x buffers");
  *d_vec = mb->m->vec(mb->m->local, which);
  return CSR5G_OK;
}

int csr5g_mailbox_ipc_handle(csr5g_mailbox mb, void* handle64) {
  if (!mb || !handle64) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == CSR5G_IPC_HANDLE_BYTES, "IPC handle size");
  CSR5G_CUDA(cudaSetDevice(mb->m->device));
  cudaIpcMemHandle_t hd;
  CSR5G_CUDA(cudaIpcGetMemHandle(&hd, mb->m->local));
  std::memcpy(handle64, &hd, sizeof hd);
  return CSR5G_OK;
}

int csr5g_mailbox_open_peer(csr5g_mailbox mb, int32_t peer, const void* handle64) {
  if (!mb || !handle64) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  Mailbox* m = mb->m;
  if (peer < 0 || peer >= m->world || peer == m->rank)
    return fail(CSR5G_EINVAL, "csr5g: peer must be another rank in [0, world)");
  if (m->peer[peer]) return fail(CSR5G_EINVAL, "csr5g: peer mailbox already linked");
  CSR5G_CUDA(cudaSetDevice(m->device));
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle64, sizeof hd);
  void* p = nullptr;
  CSR5G_CUDA(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
  m->peer[peer] = static_cast<MailboxDev*>(p);
  m->ipc_opened[peer] = true;
  return refresh_peer_table(m);
}

int csr5g_mailbox_link_local(csr5g_mailbox mb, int32_t peer, csr5g_mailbox peer_mb) {
  if (!mb || !peer_mb) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  Mailbox* m = mb->m;
  if (peer < 0 || peer >= m->world || peer == m->rank || peer_mb->m->rank != peer)
    return fail(CSR5G_EINVAL, "csr5g: peer must be another rank in [0, world)");
  if (m->peer[peer]) return fail(CSR5G_EINVAL, "csr5g: peer mailbox already linked");
  if (peer_mb->m->vec_len != m->vec_len)
    return fail(CSR5G_EINVAL, "csr5g: peer mailbox has another vec_len");
  if (peer_mb->m->device != m->device) {
    int ok = 0;
    CSR5G_CUDA(cudaDeviceCanAccessPeer(&ok, m->device, peer_mb->m->device));
    if (!ok) return fail(CSR5G_ECUDA, "csr5g: no peer access between the two devices");
    CSR5G_CUDA(cudaSetDevice(m->device));
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer_mb->m->device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
      return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    cudaGetLastError();
  }
  m->peer[peer] = peer_mb->m->local;
  CSR5G_CUDA(cudaSetDevice(m->device));
  return refresh_peer_table(m);
}

int csr5g_mailbox_errors(csr5g_mailbox mb, uint32_t* errors) {
  if (!mb || !errors) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  CSR5G_CUDA(cudaSetDevice(mb->m->device));
  CSR5G_CUDA(cudaMemcpy(errors, &mb->m->local->err, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return CSR5G_OK;
}

int csr5g_mailbox_release(csr5g_mailbox mb) {
  if (!mb) return CSR5G_OK;
  Mailbox* m = mb->m;
  cudaSetDevice(m->device);
  cudaDeviceSynchronize();
  mcast_free(m);
  for (int g = 0; g < m->world; ++g)
    if (m->ipc_opened[g]) cudaIpcCloseMemHandle(m->peer[g]);
  cudaFree(m->d_peer_ack);
  cudaFree(m->d_peer_xready);
  cudaFree(m->local);
  delete m;
  delete mb;
  return CSR5G_OK;
}

int csr5g_mg_bind(csr5g_matrix h, csr5g_mailbox mb, int32_t dest, int32_t sender_begin,
                  int32_t sender_end, int32_t active_world) {
  if (!h || !mb) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  Handle* hh = h->h;
  Mailbox* m = mb->m;
  if (hh->device != m->device) return fail(CSR5G_EINVAL, "csr5g: mailbox is on another device");
  if (active_world < 1 || active_world > m->world || m->rank >= active_world)
    return fail(CSR5G_EINVAL, "csr5g: active_world must cover this rank and not exceed world");
  const bool first_owned = hh->first_owned || hh->pcs == 0;
  if ((dest >= 0) == first_owned)
    return fail(CSR5G_EINVAL, first_owned ? "csr5g: shard owns its first row; dest must be -1"
                                          : "csr5g: shard does not own its first row; dest required");
  if (dest >= m->rank) return fail(CSR5G_EINVAL, "csr5g: dest must be an earlier rank");
  if (sender_end > sender_begin &&
      (sender_begin != m->rank + 1 || sender_end > active_world || hh->is_last))
    return fail(CSR5G_EINVAL, "csr5g: senders must be the ranks right after this one");
  for (int g = sender_begin; g < sender_end; ++g)
    if (!m->peer[g]) return fail(CSR5G_EINVAL, "csr5g: sender mailbox not linked");
  if (dest >= 0 && !m->peer[dest]) return fail(CSR5G_EINVAL, "csr5g: dest mailbox not linked");
  if (!hh->mg) hh->mg = new Binding;
  hh->mg->mb = m;
  hh->mg->dest = dest;
  hh->mg->sb = sender_begin;
  hh->mg->se = std::max(sender_begin, sender_end);
  hh->mg->active = active_world;
  return CSR5G_OK;
}

int csr5g_mg_spmv_post(csr5g_matrix h, const double* d_x, double* d_y, void* stream, void* ev0,
                       void* ev1) {
  if (!h || !d_y || (!d_x && h->h->info.n > 0)) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  return mg_post(h->h, d_x, d_y, static_cast<cudaStream_t>(stream),
                 static_cast<cudaEvent_t>(ev0), static_cast<cudaEvent_t>(ev1));
}

int csr5g_mg_spmv_fixup(csr5g_matrix h, double* d_y, void* stream) {
  if (!h || !d_y) return fail(CSR5G_EINVAL, "csr5g: NULL argument");
  return mg_fixup(h->h, d_y, static_cast<cudaStream_t>(stream));
}

int csr5g_mg_spmv(csr5g_matrix h, const double* d_x, double* d_y, void* stream, void* ev0,
                  void* ev1) {
  if (int rc = csr5g_mg_spmv_post(h, d_x, d_y, stream, ev0, ev1)) return rc;
  return csr5g_mg_spmv_fixup(h, d_y, stream);
}

int csr5g_mg_iter_post(csr5g_matrix h, int64_t it, void* stream, void* ev0, void* ev1) {
  if (!h) return fail(CSR5G_EINVAL, "csr5g: NULL handle");
  if (it < 0) return fail(CSR5G_EINVAL, "csr5g: negative iteration");
  return mg_iter_post(h->h, it, static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(ev0),
                      static_cast<cudaEvent_t>(ev1));
}

int csr5g_mg_iter_finish(csr5g_matrix h, int64_t it, void* stream) {
  if (!h) return fail(CSR5G_EINVAL, "csr5g: NULL handle");
  if (it < 0) return fail(CSR5G_EINVAL, "csr5g: negative iteration");
  return mg_iter_finish(h->h, it, static_cast<cudaStream_t>(stream));
}

int csr5g_mg_iter(csr5g_matrix h, int64_t it, void* stream, void* ev0, void* ev1) {
  if (int rc = csr5g_mg_iter_post(h, it, stream, ev0, ev1)) return rc;
  return csr5g_mg_iter_finish(h, it, stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// NVSwitch multicast (NVLS) of the x ping-pong, fused iterative mode
// ---------------------------------------------------------------------------
namespace csr5g {

struct Mcast {
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  CUmemAllocationHandleType ht = CU_MEM_HANDLE_TYPE_NONE;  // shareable type of both
  CUdeviceptr local_va = 0, mc_va = 0;
  size_t bytes = 0;
  int ndev = 0;
  bool have_mc = false, have_mem = false, local_mapped = false, mc_mapped = false, bound = false;
};

namespace {

// driver entry points (no -lcuda: the runtime hands them out)
struct Drv {
  CUresult (*mc_create)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*mc_add)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mc_bind)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t,
                      size_t, unsigned long long) = nullptr;
  CUresult (*mc_unbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*mc_gran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*mem_create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                         unsigned long long) = nullptr;
  CUresult (*mem_gran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*mem_release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*va_reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*va_free)(CUdeviceptr, size_t) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*export_h)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                       unsigned long long) = nullptr;
  CUresult (*import_h)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*dev_get)(CUdevice*, int) = nullptr;
  CUresult (*dev_attr)(int*, CUdevice_attribute, CUdevice) = nullptr;
};

int drv(const Drv** out) {
  static Drv d;
  static cudaError_t rc = [] {
    auto get = [](const char* name, auto** fn) {
      void* p = nullptr;
      cudaDriverEntryPointQueryResult q{};
      cudaError_t e = cudaGetDriverEntryPointByVersion(name, &p, CUDA_VERSION, cudaEnableDefault, &q);
      if (e == cudaSuccess && q != cudaDriverEntryPointSuccess) e = cudaErrorNotSupported;
      *fn = reinterpret_cast<std::remove_pointer_t<decltype(fn)>>(p);
      return e;
    };
    cudaError_t e = cudaSuccess;
    for (cudaError_t r : {get("cuMulticastCreate", &d.mc_create), get("cuMulticastAddDevice", &d.mc_add),
                          get("cuMulticastBindMem", &d.mc_bind), get("cuMulticastUnbind", &d.mc_unbind),
                          get("cuMulticastGetGranularity", &d.mc_gran), get("cuMemCreate", &d.mem_create),
                          get("cuMemGetAllocationGranularity", &d.mem_gran),
                          get("cuMemRelease", &d.mem_release), get("cuMemAddressReserve", &d.va_reserve),
                          get("cuMemAddressFree", &d.va_free), get("cuMemMap", &d.map),
                          get("cuMemUnmap", &d.unmap), get("cuMemSetAccess", &d.set_access),
                          get("cuMemExportToShareableHandle", &d.export_h),
                          get("cuMemImportFromShareableHandle", &d.import_h),
                          get("cuDeviceGet", &d.dev_get), get("cuDeviceGetAttribute", &d.dev_attr)})
      if (r != cudaSuccess) e = r;
    return e;
  }();
  if (rc != cudaSuccess) return cuda_fail(rc, "cudaGetDriverEntryPoint (multicast / VMM)");
  *out = &d;
  return CSR5G_OK;
}

int cu_fail(CUresult r, const char* what) {
  return fail(CSR5G_ECUDA, std::string(what) + " failed (CUresult " + std::to_string((int)r) + ")");
}
#define CSR5G_CU(call)                              \
  do {                                              \
    const CUresult r_ = (call);                     \
    if (r_ != CUDA_SUCCESS) return cu_fail(r_, #call); \
  } while (0)

CUmulticastObjectProp mc_prop(int ndev, size_t bytes, CUmemAllocationHandleType ht) {
  CUmulticastObjectProp p{};
  p.numDevices = (unsigned)ndev;
  p.size = bytes;
  p.handleTypes = (unsigned long long)ht;
  p.flags = 0;
  return p;
}

// the x ping-pong's size rounded to both granularities
int mc_size(const Drv* d, int device, int ndev, int64_t vec_len, CUmemAllocationHandleType ht,
            size_t* bytes) {
  CUmulticastObjectProp mp = mc_prop(ndev, 1, ht);
  size_t g1 = 0, g2 = 0;
  CSR5G_CU(d->mc_gran(&g1, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  ap.requestedHandleTypes = ht;
  CSR5G_CU(d->mem_gran(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t g = std::max<size_t>(std::max<size_t>(g1, g2), 1);
  const size_t want = sizeof(double) * 2 * (size_t)vec_len;
  *bytes = (want + g - 1) / g * g;
  return CSR5G_OK;
}

int map_rw(const Drv* d, int device, CUmemGenericAllocationHandle h, size_t bytes, CUdeviceptr* va) {
  CSR5G_CU(d->va_reserve(va, bytes, 0, 0, 0));
  CUresult r = d->map(*va, bytes, 0, h, 0);
  if (r == CUDA_SUCCESS) {
    CUmemAccessDesc a{};
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = device;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = d->set_access(*va, bytes, &a, 1);
    if (r != CUDA_SUCCESS) d->unmap(*va, bytes);
  }
  if (r != CUDA_SUCCESS) {
    d->va_free(*va, bytes);
    *va = 0;
    return cu_fail(r, "cuMemMap / cuMemSetAccess");
  }
  return CSR5G_OK;
}

}  // namespace

void mcast_free(Mailbox* m) {
  Mcast* c = m->mc;
  if (!c) return;
  const Drv* d = nullptr;
  if (drv(&d) == CSR5G_OK) {
    CUdevice dev = 0;
    d->dev_get(&dev, m->device);
    if (c->mc_mapped) d->unmap(c->mc_va, c->bytes), d->va_free(c->mc_va, c->bytes);
    if (c->local_mapped) d->unmap(c->local_va, c->bytes), d->va_free(c->local_va, c->bytes);
    if (c->bound) d->mc_unbind(c->mc, dev, 0, c->bytes);
    if (c->have_mem) d->mem_release(c->mem);
    if (c->have_mc) d->mem_release(c->mc);
  }
  m->mc_local = m->mc_multi = nullptr;
  delete c;
  m->mc = nullptr;
}

}  // namespace csr5g

int csr5g_mcast_supported(int device, int32_t* out) {
  if (!out) return fail(CSR5G_EINVAL, "csr5g: out is NULL");
  *out = 0;
  const Drv* d = nullptr;
  if (int rc = drv(&d)) return rc;
  CUdevice dev = 0;
  CSR5G_CU(d->dev_get(&dev, device));
  int v = 0;
  CSR5G_CU(d->dev_attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  *out = v;
  return CSR5G_OK;
}

int csr5g_mailbox_mcast_create(csr5g_mailbox mb, int32_t ndev, void* handle64) {
  if (!mb || ndev < 1) return fail(CSR5G_EINVAL, "csr5g: bad multicast arguments");
  Mailbox* m = mb->m;
  if (m->mc) return fail(CSR5G_EINVAL, "csr5g: the mailbox already has a multicast object");
  if (m->vec_len <= 0) return fail(CSR5G_EINVAL, "csr5g: mailbox has no x buffers");
  const Drv* d = nullptr;
  if (int rc = drv(&d)) return rc;
  CSR5G_CUDA(cudaSetDevice(m->device));
  auto* c = new Mcast;
  c->ndev = ndev;
  m->mc = c;
  // several processes need a fabric handle; one process takes the first
  // handle type the driver accepts
  CUresult r = CUDA_ERROR_NOT_SUPPORTED;
  for (CUmemAllocationHandleType ht :
       {CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_NONE}) {
    if (ndev > 1 && ht != CU_MEM_HANDLE_TYPE_FABRIC) break;
    if (mc_size(d, m->device, ndev, m->vec_len, ht, &c->bytes) != CSR5G_OK) continue;
    const CUmulticastObjectProp p = mc_prop(ndev, c->bytes, ht);
    r = d->mc_create(&c->mc, &p);
    if (r == CUDA_SUCCESS) {
      c->ht = ht;
      break;
    }
  }
  if (r != CUDA_SUCCESS) return mcast_free(m), cu_fail(r, "cuMulticastCreate");
  c->have_mc = true;
  if (ndev > 1) {
    if (!handle64) return mcast_free(m), fail(CSR5G_EINVAL, "csr5g: handle64 is NULL");
    r = d->export_h(handle64, c->mc, CU_MEM_HANDLE_TYPE_FABRIC, 0);
    if (r != CUDA_SUCCESS) return mcast_free(m), cu_fail(r, "cuMemExportToShareableHandle (fabric)");
  }
  return CSR5G_OK;
}

int csr5g_mailbox_mcast_import(csr5g_mailbox mb, int32_t ndev, const void* handle64) {
  if (!mb || !handle64 || ndev < 2) return fail(CSR5G_EINVAL, "csr5g: bad multicast arguments");
  Mailbox* m = mb->m;
  if (m->mc) return fail(CSR5G_EINVAL, "csr5g: the mailbox already has a multicast object");
  const Drv* d = nullptr;
  if (int rc = drv(&d)) return rc;
  CSR5G_CUDA(cudaSetDevice(m->device));
  auto* c = new Mcast;
  c->ndev = ndev;
  m->mc = c;
  c->ht = CU_MEM_HANDLE_TYPE_FABRIC;
  if (int rc = mc_size(d, m->device, ndev, m->vec_len, c->ht, &c->bytes)) return mcast_free(m), rc;
  const CUresult r = d->import_h(&c->mc, const_cast<void*>(handle64), CU_MEM_HANDLE_TYPE_FABRIC);
  if (r != CUDA_SUCCESS) return mcast_free(m), cu_fail(r, "cuMemImportFromShareableHandle (fabric)");
  c->have_mc = true;
  return CSR5G_OK;
}

int csr5g_mailbox_mcast_add(csr5g_mailbox mb) {
  if (!mb || !mb->m->mc) return fail(CSR5G_EINVAL, "csr5g: no multicast object");
  Mailbox* m = mb->m;
  const Drv* d = nullptr;
  if (int rc = drv(&d)) return rc;
  CUdevice dev = 0;
  CSR5G_CU(d->dev_get(&dev, m->device));
  CSR5G_CU(d->mc_add(m->mc->mc, dev));
  return CSR5G_OK;
}

// after every rank's device was added: this rank's x ping-pong in fresh
// device memory, bound to the object, mapped unicast (reads) and multicast
// (the kernels' mirror stores); the mailbox's x buffers become these
int csr5g_mailbox_mcast_bind(csr5g_mailbox mb) {
  if (!mb || !mb->m->mc) return fail(CSR5G_EINVAL, "csr5g: no multicast object");
  Mailbox* m = mb->m;
  Mcast* c = m->mc;
  const Drv* d = nullptr;
  if (int rc = drv(&d)) return rc;
  CSR5G_CUDA(cudaSetDevice(m->device));
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = m->device;
  ap.requestedHandleTypes = c->ht;
  CSR5G_CU(d->mem_create(&c->mem, c->bytes, &ap, 0));
  c->have_mem = true;
  CSR5G_CU(d->mc_bind(c->mc, 0, c->mem, 0, c->bytes, 0));
  c->bound = true;
  if (int rc = map_rw(d, m->device, c->mem, c->bytes, &c->local_va)) return rc;
  c->local_mapped = true;
  if (int rc = map_rw(d, m->device, c->mc, c->bytes, &c->mc_va)) return rc;
  c->mc_mapped = true;
  CSR5G_CUDA(cudaMemset(reinterpret_cast<void*>(c->local_va), 0, c->bytes));
  m->mc_local = reinterpret_cast<double*>(c->local_va);
  m->mc_multi = reinterpret_cast<double*>(c->mc_va);
  return CSR5G_OK;
}

namespace csr5g {
namespace {
__global__ void k_mcast_write(double* mc, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    asm volatile("multimem.st.global.f64 [%0], %1;" ::"l"(mc + i), "d"((double)i * 0.5 + 1.0) : "memory");
}
__global__ void k_mcast_check(const double* local, int64_t n, unsigned long long* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (local[i] != (double)i * 0.5 + 1.0) atomicAdd(bad, 1ull);
}
}  // namespace
}  // namespace csr5g

// test hook: multimem stores into the multicast mapping of x buffer 1 land in
// this rank's bound copy (the count of mismatching values; buffer 1 is left
// holding the pattern)
int csr5g_mailbox_mcast_selftest(csr5g_mailbox mb, int64_t* mismatches) {
  if (!mb || !mismatches || !mb->m->mc_multi) return fail(CSR5G_EINVAL, "csr5g: no bound multicast");
  Mailbox* m = mb->m;
  CSR5G_CUDA(cudaSetDevice(m->device));
  unsigned long long* bad = nullptr;
  CSR5G_CUDA(cudaMalloc(&bad, sizeof *bad));
  cudaError_t e = cudaMemset(bad, 0, sizeof *bad);
  if (e == cudaSuccess) {
    k_mcast_write<<<264, 256>>>(m->mc_multi + m->vec_len, m->vec_len);
    e = cudaDeviceSynchronize();
  }
  if (e == cudaSuccess) {
    k_mcast_check<<<264, 256>>>(m->mc_local + m->vec_len, m->vec_len, bad);
    e = cudaDeviceSynchronize();
  }
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&h, bad, sizeof h, cudaMemcpyDeviceToHost);
  cudaFree(bad);
  if (e != cudaSuccess) return cuda_fail(e, "csr5g_mailbox_mcast_selftest");
  *mismatches = (int64_t)h;
  return CSR5G_OK;
}

int csr5g_mailbox_mcast_release(csr5g_mailbox mb) {
  if (!mb) return CSR5G_OK;
  cudaSetDevice(mb->m->device);
  cudaDeviceSynchronize();
  mcast_free(mb->m);
  return CSR5G_OK;
}
