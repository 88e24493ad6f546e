// die_probe.cu -- does a B200 die's L2 cache what its own SMs read?
//
// Evidence tool for DESIGN.md §5 (random-gather ceiling), not product code.
// B200 is two dies of 74 SMs, each with half of the 126 MB L2.  If an SM's
// misses are filled into its own die's L2 (so a line read by SMs on both dies
// is held twice), random gathers over all of x see ~63 MB of L2, not 126 MB.
//
// 1. Die map: one CTA per SM chases dependent L2-hit loads (ld.cg) into 2 KB
//    chunks of a warm buffer and records the latency per (SM, chunk).  A chunk
//    homed on the SM's own die answers ~30 cycles sooner; SMs whose near/far
//    pattern correlates with SM 0's are on SM 0's die.
// 2. Gathers: uniform random 8-byte gathers over x (n doubles) with every warp
//    drawing from
//      all   -- the whole of x (what an SpMV on a permuted graph does);
//      die   -- the half of x assigned to its SM's die;
//      mixed -- a half chosen by a hash of the SM id (same per-SM working set
//               as `die`, but each half is read from both dies).
//    die >> mixed ~ all  <=>  the L2 capacity a die's SMs see is its own half.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/die_probe.cu
#include <cuda_runtime.h>

#include <cmath>
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

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

constexpr int kChunk = 2048 / 8;  // doubles per 2 KB chunk

// lane 0 of the CTA on SM s: lat[s * C + c] = mean latency of R dependent
// L2-hit loads into chunk c (the buffer holds zeros, so each address depends
// on the previous load's value)
__global__ void k_diemap(const double* __restrict__ buf, int C, int R, float* lat,
                         int* sm_of_cta) {
  extern __shared__ char pad[];
  if (threadIdx.x != 0) return;
  const uint32_t s = smid();
  sm_of_cta[blockIdx.x] = (int)s;
  if (pad[0] == 123) return;  // keeps the shared memory allocation
  double v = 0.0;
  for (int c = 0; c < C; ++c) {
    const double* p = buf + (size_t)c * kChunk;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p + (int)v));  // warm TLB/line
    const long long t0 = clock64();
    for (int r = 0; r < R; ++r) {
      const double* q = p + ((r * 17) & (kChunk - 1)) + (int)v;
      asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(q));
    }
    const long long t1 = clock64();
    lat[(size_t)s * C + c] = (float)(t1 - t0) / R + (float)v;
  }
}

// every warp: `per` gathers of x[base + (idx & mask)] with the half chosen by
// `mode` (0 all, 1 die, 2 mixed)
__global__ void k_gather(const int32_t* __restrict__ idx, const double* __restrict__ x, int64_t N,
                         int64_t half, const int8_t* __restrict__ die_of_sm, int mode,
                         double* out) {
  extern __shared__ char pad[];
  const int lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int w = blockIdx.x * nw + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * nw;
  const uint32_t s = smid();
  int64_t base = 0, span = 2 * half;
  if (mode == 1) {
    base = die_of_sm[s] ? half : 0;
    span = half;
  } else if (mode == 2) {
    base = ((s * 2654435761u) >> 7) & 1 ? half : 0;
    span = half;
  }
  const int64_t per = (N / nwarps) & ~(int64_t)511;
  const int64_t b = (int64_t)w * per;
  double acc = pad[0] == 123 ? 1.0 : 0.0;
  constexpr int K = 16;
  for (int64_t i = b; i < b + per; i += 32 * K) {
    int32_t c[K];
#pragma unroll
    for (int u = 0; u < K; ++u) c[u] = __ldcs(idx + i + u * 32 + lane);
    double v[K];
#pragma unroll
    for (int u = 0; u < K; ++u) {
      const double* p = x + base + (int64_t)((uint32_t)c[u] % (uint32_t)span);
      asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[u]) : "l"(p));
    }
#pragma unroll
    for (int u = 0; u < K; ++u) acc += v[u];
  }
  if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
  int sms = 0, max_smem = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
  const int one_cta = max_smem - 1024;  // forces one CTA per SM
  CK(cudaFuncSetAttribute(k_diemap, cudaFuncAttributeMaxDynamicSharedMemorySize, one_cta));

  // ---- 1. die map ----
  const int C = 512, R = 16;
  double* buf;
  float* lat;
  int* sm_of_cta;
  CK(cudaMalloc(&buf, (size_t)C * kChunk * 8));
  CK(cudaMemset(buf, 0, (size_t)C * kChunk * 8));
  CK(cudaMalloc(&lat, (size_t)256 * C * 4));
  CK(cudaMemset(lat, 0, (size_t)256 * C * 4));
  CK(cudaMalloc(&sm_of_cta, sms * 4));
  k_diemap<<<sms, 32, one_cta>>>(buf, C, R, lat, sm_of_cta);  // warm
  k_diemap<<<sms, 32, one_cta>>>(buf, C, R, lat, sm_of_cta);
  CK(cudaDeviceSynchronize());
  std::vector<float> L((size_t)256 * C);
  std::vector<int> smo(sms);
  CK(cudaMemcpy(L.data(), lat, L.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(smo.data(), sm_of_cta, sms * 4, cudaMemcpyDeviceToHost));
  std::vector<int> seen(256, 0);
  for (int s : smo) seen[s]++;
  int distinct = 0;
  for (int s = 0; s < 256; ++s) distinct += seen[s] > 0;
  printf("die map: %d CTAs on %d distinct SMs\n", sms, distinct);
  // centre each SM's latency vector; correlate with the first SM's
  auto centred = [&](int s) {
    std::vector<double> v(C);
    double mu = 0;
    for (int c = 0; c < C; ++c) mu += L[(size_t)s * C + c];
    mu /= C;
    for (int c = 0; c < C; ++c) v[c] = L[(size_t)s * C + c] - mu;
    return v;
  };
  int s0 = -1;
  for (int s = 0; s < 256 && s0 < 0; ++s)
    if (seen[s]) s0 = s;
  const std::vector<double> r0 = centred(s0);
  double n0 = 0;
  for (double d : r0) n0 += d * d;
  std::vector<int8_t> die(256, 0);
  int cnt[2] = {0, 0};
  double min_abs_corr = 1.0;
  for (int s = 0; s < 256; ++s) {
    if (!seen[s]) continue;
    const std::vector<double> r = centred(s);
    double dot = 0, nn = 0;
    for (int c = 0; c < C; ++c) dot += r[c] * r0[c], nn += r[c] * r[c];
    const double corr = dot / std::sqrt(nn * n0 + 1e-30);
    die[s] = corr > 0 ? 0 : 1;
    cnt[die[s]]++;
    min_abs_corr = std::fmin(min_abs_corr, std::fabs(corr));
  }
  // near/far latency split seen from SM s0
  std::vector<float> l0(L.begin() + (size_t)s0 * C, L.begin() + (size_t)(s0 + 1) * C);
  double near = 0, far = 0;
  int nn = 0, nf = 0;
  for (int c = 0; c < C; ++c)
    if (r0[c] < 0) near += l0[c], ++nn;
    else far += l0[c], ++nf;
  printf("die map: %d SMs on SM %d's die, %d on the other; min |corr| %.3f; "
         "SM %d: %d near chunks %.1f cyc, %d far chunks %.1f cyc\n",
         cnt[0], s0, cnt[1], min_abs_corr, s0, nn, near / std::max(nn, 1), nf,
         far / std::max(nf, 1));
  printf("die0 SMs:");
  for (int s = 0; s < 256; ++s)
    if (seen[s] && die[s] == 0) printf(" %d", s);
  printf("\ndie1 SMs:");
  for (int s = 0; s < 256; ++s)
    if (seen[s] && die[s] == 1) printf(" %d", s);
  printf("\n");

  // ---- 2. gathers ----
  int8_t* d_die;
  CK(cudaMalloc(&d_die, 256));
  CK(cudaMemcpy(d_die, die.data(), 256, cudaMemcpyHostToDevice));
  const int64_t N = (int64_t)1 << 28;
  std::vector<int32_t> h(N);
  uint64_t st = 88172645463325252ull;
  for (int64_t i = 0; i < N; ++i) {
    st ^= st << 13, st ^= st >> 7, st ^= st << 17;
    h[i] = (int32_t)(st >> 33);
  }
  int32_t* idx;
  double *x, *out;
  const int64_t nmax = (int64_t)1 << 25;  // 268 MB of x at most
  CK(cudaMalloc(&idx, N * 4));
  CK(cudaMalloc(&x, nmax * 8));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemcpy(idx, h.data(), N * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(x, 0, nmax * 8));
  const int smem = 96 * 1024;  // the SpMV's random plans leave ~150 KB of L1
  CK(cudaFuncSetAttribute(k_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const char* names[] = {"all", "die", "mixed"};
  const double mbs[] = {33.5, 50, 67, 84, 100, 117, 134, 168, 201, 268};
  for (int wps : {16, 32}) {
    for (double mb : mbs) {
      const int64_t n = (int64_t)(mb * 1e6 / 8) & ~(int64_t)1;
      printf("warps/SM %2d  x %6.1f MB |", wps, n * 8 / 1e6);
      for (int mode = 0; mode < 3; ++mode) {
        k_gather<<<sms, wps * 32, smem>>>(idx, x, N, n / 2, d_die, mode, out);
        CK(cudaEventRecord(a));
        for (int r = 0; r < 3; ++r) k_gather<<<sms, wps * 32, smem>>>(idx, x, N, n / 2, d_die, mode, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        const int64_t per = (N / (sms * wps)) & ~(int64_t)511;
        printf("  %s %6.1f G/s", names[mode], (double)per * sms * wps / (ms / 3) / 1e6);
      }
      printf("\n");
    }
  }
  CK(cudaGetLastError());
  return 0;
}
