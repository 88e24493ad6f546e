// sector_probe.cu -- how many L2 sectors (and DRAM bytes) one random 8-byte
// gather costs, per load flavour.  Evidence tool for DESIGN.md §5, not
// product code.  Run under
//   ncu --metrics lts__t_requests_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,\
// dram__bytes_read.sum,gpu__time_duration.sum --csv build/sector_probe
// Each kernel launch performs N uniform random gathers x[idx[i]] over n
// doubles (idx streamed coalesced), with one load flavour.
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

template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
  double v;
  if (MODE == 0) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 2) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 3) asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 4) asm volatile("ld.global.cv.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 5) asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 6) asm volatile("ld.global.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 7) asm volatile("ld.global.nc.L2::128B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  if (MODE == 8) {
    float f;
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(f) : "l"(p));
    v = f;
  }
  if (MODE == 9) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(p), "l"(pol));
  }
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(512) k_gather(const int32_t* __restrict__ idx,
                                                const double* __restrict__ x, int64_t N,
                                                double* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
  double acc = 0.0;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); b * 8 < N; b += stride / 8) {
    int32_t c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = b + (int64_t)u * gridDim.x * blockDim.x;
      c[u] = i < N ? __ldcs(idx + i) : 0;
    }
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ld<MODE>(x + c[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  if (acc == 12345.678) out[0] = acc;
}

template <int MODE>
void run(const char* name, const int32_t* idx, const double* x, int64_t N, int sms, double* out) {
  k_gather<MODE><<<sms * 4, 512>>>(idx, x, N, out);  // warm
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a));
  k_gather<MODE><<<sms * 4, 512>>>(idx, x, N, out);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  printf("mode %d %-28s %8.3f ms  %6.1f G gathers/s\n", MODE, name, ms, N / ms / 1e6);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (int64_t)1 << 27;  // doubles in x
  const int64_t N = argc > 2 ? atoll(argv[2]) : (int64_t)1 << 29;  // gathers
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
  printf("x %.1f MB, %lld gathers\n", n * 8 / 1e6, (long long)N);
  run<0>("ld.global.nc", idx, x, N, sms, out);
  run<1>("ld.global.nc.L1::no_allocate", idx, x, N, sms, out);
  run<2>("ld.global.cg", idx, x, N, sms, out);
  run<3>("ld.global.ca", idx, x, N, sms, out);
  run<4>("ld.global.cv", idx, x, N, sms, out);
  run<5>("ld.relaxed.gpu", idx, x, N, sms, out);
  run<6>("ld.global.L2::64B", idx, x, N, sms, out);
  run<7>("ld.global.nc.L2::128B", idx, x, N, sms, out);
  run<8>("ld.global.nc.f32", idx, x, N, sms, out);
  run<9>("nc.no_alloc.evict_first", idx, x, N, sms, out);
  CK(cudaGetLastError());
  return 0;
}
