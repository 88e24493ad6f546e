// pipeline.cu -- SpMV on host vectors through a copy/compute pipeline.
//
// The reference's spmv_csr5 takes host vectors (spmv.hpp:58-61).  On the GPU
// a host-vector SpMV is PCIe-bound: x H2D (8n bytes) + y D2H (8m bytes) dwarf
// the ~0.5 ms kernel.  PCIe is full duplex and the two copy directions use
// separate copy engines, so a batch of independent SpMVs runs as a three-stage
// pipeline over two device (x, y) buffer pairs:
//
//   h2d stream   x_k -> dx[k&1]          waits: SpMV k-2 done reading dx[k&1]
//   run stream   spmv(dx[k&1], dy[k&1])  waits: x_k landed, y_{k-2} copied out
//   d2h stream   dy[k&1] -> y_k          waits: SpMV k done
//
// In steady state a step costs max(H2D, D2H, SpMV) instead of their sum; each
// step still moves its own x in and its own y out.  The buffers and streams are
// created on first use and owned by the handle.
#include <algorithm>

#include "internal.cuh"

namespace csr5g {

struct Pipeline {
  int device = 0;
  int64_t n = 0, m = 0;
  double* dx[2] = {nullptr, nullptr};
  double* dy[2] = {nullptr, nullptr};
  cudaStream_t h2d = nullptr, run = nullptr, d2h = nullptr;
  cudaEvent_t x_in[2] = {}, done[2] = {}, y_out[2] = {}, start = nullptr;
};

void free_pipeline(Pipeline* p) {
  if (!p) return;
  for (int b = 0; b < 2; ++b) {
    if (p->dx[b]) cudaFree(p->dx[b]);
    if (p->dy[b]) cudaFree(p->dy[b]);
    for (cudaEvent_t e : {p->x_in[b], p->done[b], p->y_out[b]})
      if (e) cudaEventDestroy(e);
  }
  if (p->start) cudaEventDestroy(p->start);
  for (cudaStream_t s : {p->h2d, p->run, p->d2h})
    if (s) cudaStreamDestroy(s);
  delete p;
}

namespace {

int make_pipeline(Handle* h, Pipeline** out) {
  if (h->pipe) {
    *out = h->pipe;
    return CSR5G_OK;
  }
  Pipeline* p = new Pipeline;
  p->device = h->device;
  p->n = h->info.n;
  p->m = h->info.m;
  auto bad = [&](cudaError_t e, const char* what) {
    free_pipeline(p);
    return cuda_fail(e, what);
  };
  cudaError_t e;
  for (int b = 0; b < 2; ++b) {
    if ((e = cudaMalloc(&p->dx[b], sizeof(double) * std::max<int64_t>(p->n, 1))) != cudaSuccess)
      return bad(e, "cudaMalloc(pipeline x)");
    if ((e = cudaMalloc(&p->dy[b], sizeof(double) * std::max<int64_t>(p->m, 1))) != cudaSuccess)
      return bad(e, "cudaMalloc(pipeline y)");
    for (cudaEvent_t* ev : {&p->x_in[b], &p->done[b], &p->y_out[b]})
      if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess)
        return bad(e, "cudaEventCreate(pipeline)");
  }
  if ((e = cudaEventCreateWithFlags(&p->start, cudaEventDisableTiming)) != cudaSuccess)
    return bad(e, "cudaEventCreate(pipeline)");
  for (cudaStream_t* s : {&p->h2d, &p->run, &p->d2h})
    if ((e = cudaStreamCreateWithFlags(s, cudaStreamNonBlocking)) != cudaSuccess)
      return bad(e, "cudaStreamCreate(pipeline)");
  h->pipe = p;
  *out = p;
  return CSR5G_OK;
}

}  // namespace

int spmv_host_batch(Handle* h, const double* const* xs, double* const* ys, int64_t count,
                    int mode, cudaStream_t stream) {
  CSR5G_CUDA(cudaSetDevice(h->device));
  // concurrent host-vector calls on one handle (reference: spmv_csr5 from
  // several threads) share its pipeline; their enqueues are serialised and the
  // buffer-reuse events order the GPU work
  std::lock_guard<std::mutex> lock(h->pipe_mu);
  Pipeline* p = nullptr;
  int rc = make_pipeline(h, &p);
  if (rc) return rc;
  const size_t xb = sizeof(double) * p->n, yb = sizeof(double) * p->m;
  // everything already queued on the caller's stream comes first
  CSR5G_CUDA(cudaEventRecord(p->start, stream));
  for (cudaStream_t s : {p->h2d, p->run, p->d2h}) CSR5G_CUDA(cudaStreamWaitEvent(s, p->start, 0));
  for (int64_t k = 0; k < count; ++k) {
    const int b = (int)(k & 1);
    // waits on the buffer pair's previous use (this call's step k-2 or an
    // earlier call's; an event never recorded is already complete)
    CSR5G_CUDA(cudaStreamWaitEvent(p->h2d, p->done[b], 0));  // dx[b] read by its SpMV
    if (xb) CSR5G_CUDA(cudaMemcpyAsync(p->dx[b], xs[k], xb, cudaMemcpyHostToDevice, p->h2d));
    CSR5G_CUDA(cudaEventRecord(p->x_in[b], p->h2d));
    CSR5G_CUDA(cudaStreamWaitEvent(p->run, p->x_in[b], 0));
    CSR5G_CUDA(cudaStreamWaitEvent(p->run, p->y_out[b], 0));  // dy[b] copied out
    rc = launch_spmv(h, p->dx[b], p->dy[b], mode, p->run, nullptr, nullptr);
    if (rc) return rc;
    CSR5G_CUDA(cudaEventRecord(p->done[b], p->run));
    CSR5G_CUDA(cudaStreamWaitEvent(p->d2h, p->done[b], 0));
    if (yb) CSR5G_CUDA(cudaMemcpyAsync(ys[k], p->dy[b], yb, cudaMemcpyDeviceToHost, p->d2h));
    CSR5G_CUDA(cudaEventRecord(p->y_out[b], p->d2h));
  }
  // join: the caller's stream continues after the last copy out
  for (int b = 0; b < 2; ++b)
    if (count > b) CSR5G_CUDA(cudaStreamWaitEvent(stream, p->y_out[b], 0));
  return CSR5G_OK;
}

}  // namespace csr5g
