// async_gather_probe.cu -- random 8-byte gathers over a large x: register
// loads (LDG) against asynchronous copies into shared memory (cp.async.cg,
// 16-byte chunks, LDGSTS), which hold no registers while in flight.  Evidence
// tool for DESIGN.md §5 (the random-gather ceiling), not product code.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                          \
  do {                                                                 \
    cudaError_t e = (x);                                               \
    if (e != cudaSuccess) {                                            \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
      exit(1);                                                         \
    }                                                                  \
  } while (0)

// LDG baseline: every thread K independent gathers per step
template <int K>
__global__ void __launch_bounds__(512) k_ldg(const int32_t* __restrict__ idx,
                                             const double* __restrict__ x, int64_t N, double* out) {
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < N; b += T * K) {
    int32_t c[K];
#pragma unroll
    for (int u = 0; u < K; ++u) c[u] = b + u * T < N ? __ldcs(idx + b + u * T) : 0;
    double v[K];
#pragma unroll
    for (int u = 0; u < K; ++u) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v[u]) : "l"(x + c[u]));
#pragma unroll
    for (int u = 0; u < K; ++u) acc += v[u];
  }
  if (acc == 12345.678) out[0] = acc;
}

// cp.async: each warp streams its share of idx in batches of 32*G gathers;
// batch b lands in ring stage b % S (16-byte chunks holding x[c]); the
// oldest batch is consumed once S-1 newer ones are in flight.
template <int G, int S>
__global__ void k_async(const int32_t* __restrict__ idx, const double* __restrict__ x, int64_t N,
                        double* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int64_t w = (int64_t)blockIdx.x * nw + wib, W = (int64_t)gridDim.x * nw;
  const int64_t per = N / W / (32 * G) * (32 * G);
  const int64_t b0 = w * per;
  unsigned char* ring = smem + (size_t)wib * S * 32 * G * 16;
  double acc = 0.0;
  const int64_t nb = per / (32 * G);
  auto issue = [&](int64_t batch) {
    unsigned char* st = ring + (size_t)(batch % S) * 32 * G * 16;
#pragma unroll
    for (int u = 0; u < G; ++u) {
      const int32_t c = __ldcs(idx + b0 + batch * 32 * G + u * 32 + lane);
      const double* src = x + (c & ~1);
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(st + (u * 32 + lane) * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int64_t b = 0; b < S - 1 && b < nb; ++b) issue(b);
  for (int64_t b = 0; b < nb; ++b) {
    if (b + S - 1 < nb)
      issue(b + S - 1);
    else
      asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
    const double* st = reinterpret_cast<const double*>(ring + (size_t)(b % S) * 32 * G * 16);
#pragma unroll
    for (int u = 0; u < G; ++u) acc += st[(u * 32 + lane) * 2];
  }
  if (acc == 12345.678) out[0] = acc;
}

template <int G, int S>
void run_async(int warps, const int32_t* idx, const double* x, int64_t N, int sms, double* out) {
  const size_t smem = (size_t)warps * S * 32 * G * 16;
  auto fn = k_async<G, S>;
  if (smem > 227 * 1024) return;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fn<<<sms, warps * 32, smem>>>(idx, x, N, out);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a));
  fn<<<sms, warps * 32, smem>>>(idx, x, N, out);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  CK(cudaGetLastError());
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  const int64_t W = (int64_t)sms * warps;
  const int64_t done = N / W / (32 * G) * (32 * G) * W;
  printf("cp.async G=%2d S=%d warps/SM %2d smem %6zu: %6.1f G gathers/s (%lld in flight/SM)\n", G,
         S, warps, smem, done / ms / 1e6, (long long)warps * (S - 1) * 32 * G);
}

template <int K>
void run_ldg(int blocks_per_sm, const int32_t* idx, const double* x, int64_t N, int sms, double* out) {
  k_ldg<K><<<sms * blocks_per_sm, 512>>>(idx, x, N, out);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a));
  k_ldg<K><<<sms * blocks_per_sm, 512>>>(idx, x, N, out);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  printf("LDG K=%2d %d x 512 threads/SM: %6.1f G gathers/s\n", K, blocks_per_sm, N / ms / 1e6);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (int64_t)1 << 27;
  const int64_t N = argc > 2 ? atoll(argv[2]) : (int64_t)1 << 29;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<int32_t> h(N);
  uint64_t s = 88172645463325252ull;
  for (int64_t i = 0; i < N; ++i) {
    s ^= s << 13, s ^= s >> 7, s ^= s << 17;
    h[i] = (int32_t)(s % (uint64_t)n);
  }
  int32_t* idx;
  double *x, *out;
  CK(cudaMalloc(&idx, N * 4));
  CK(cudaMalloc(&x, n * 8 + 16));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemcpy(idx, h.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(x, 0, n * 8 + 16));
  printf("x %.1f MB, %lld uniform random gathers\n", n * 8 / 1e6, (long long)N);
  run_ldg<8>(1, idx, x, N, sms, out);
  run_ldg<8>(2, idx, x, N, sms, out);
  run_ldg<8>(4, idx, x, N, sms, out);
  run_ldg<16>(2, idx, x, N, sms, out);
  run_ldg<16>(4, idx, x, N, sms, out);
  for (int warps : {8, 16, 32}) {
    run_async<8, 4>(warps, idx, x, N, sms, out);
    run_async<8, 8>(warps, idx, x, N, sms, out);
    run_async<16, 4>(warps, idx, x, N, sms, out);
    run_async<4, 8>(warps, idx, x, N, sms, out);
  }
  return 0;
}
