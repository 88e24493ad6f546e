// gather_probe.cu -- microbenchmark: random fp64 gather throughput on one GPU.
//
// Measures the ceiling the SpMV tile kernel works against on irregular
// matrices: G gathers/s of x[idx[i]] with idx uniformly random over n, for
// several load flavours, warps per SM and loads in flight per thread.
// Not part of the product; evidence for DESIGN.md (build: make probe).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));        \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
  double v;
  if (MODE == 0)
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if (MODE == 1)
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if (MODE == 2)
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// each warp walks its chunk of idx in steps of 32*K; per step every lane
// issues K independent gathers, then reduces them
template <int MODE, int K>
__global__ void k_gather(const int32_t* __restrict__ idx, const double* __restrict__ x, int64_t N,
                         int nwarps, double* out) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= nwarps) return;
  const int64_t per = (N + nwarps - 1) / nwarps;
  const int64_t b = w * per, e = b + per < N ? b + per : N;
  double acc = 0.0;
  for (int64_t s = b; s + 32 * K <= e; s += 32 * K) {
    int32_t c[K];
#pragma unroll
    for (int u = 0; u < K; ++u) c[u] = __ldcs(idx + s + u * 32 + lane);
    double v[K];
#pragma unroll
    for (int u = 0; u < K; ++u) v[u] = ld<MODE>(x + c[u]);
#pragma unroll
    for (int u = 0; u < K; ++u) acc += v[u];
  }
  if (acc == 12345.678) out[0] = acc;
}

template <int MODE, int K>
float run(const int32_t* idx, const double* x, int64_t N, int sms, int wps, int carve, double* out) {
  auto fn = k_gather<MODE, K>;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
  const int nwarps = sms * wps;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  fn<<<sms, wps * 32>>>(idx, x, N, nwarps, out);
  CK(cudaEventRecord(a));
  for (int r = 0; r < 3; ++r) fn<<<sms, wps * 32>>>(idx, x, N, nwarps, out);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / 3;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 24);
  const int64_t N = argc > 2 ? atoll(argv[2]) : (int64_t)1 << 28;
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
  CK(cudaMalloc(&x, n * 8));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemcpy(idx, h.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(x, 0, n * 8));
  printf("n=%lld (x %.1f MB) N=%lld gathers\n", (long long)n, n * 8 / 1e6, (long long)N);
  const char* names[] = {"nc", "nc.no_alloc", "cg", "plain"};
  for (int carve : {0, 50, 100}) {
    for (int wps : {8, 16, 32}) {
      float t0 = run<0, 16>(idx, x, N, sms, wps, carve, out);
      float t1 = run<1, 16>(idx, x, N, sms, wps, carve, out);
      float t2 = run<2, 16>(idx, x, N, sms, wps, carve, out);
      float t8 = run<1, 8>(idx, x, N, sms, wps, carve, out);
      float t32 = run<1, 32>(idx, x, N, sms, wps, carve, out);
      printf("carve %3d%% warps/SM %2d | K16 %s %.1f  %s %.1f  %s %.1f | no_alloc K8 %.1f K32 %.1f  (G gathers/s)\n",
             carve, wps, names[0], N / t0 / 1e6, names[1], N / t1 / 1e6, names[2], N / t2 / 1e6,
             N / t8 / 1e6, N / t32 / 1e6);
    }
  }
  return 0;
}
