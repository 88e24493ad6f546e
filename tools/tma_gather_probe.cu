// tma_gather_probe.cu -- random 8-byte gathers through the LSU (LDG) against
// TMA tile::gather4 (sm_100a: one instruction fetches 4 rows of a 2D tensor;
// x viewed as [n/2][2] doubles, one 16-byte row per gathered value).  The
// question: does moving the gathers off the L1TEX t-stage (~1 sector per
// clock per SM for scattered loads) raise the gather rate?
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/tma_gather_probe.cu -lcuda
//   ./tma_gather_probe [x_MB ...]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e = (x);                                                                 \
    if (e != cudaSuccess) {                                                              \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
      std::exit(1);                                                                      \
    }                                                                                    \
  } while (0)

__global__ void k_ldg(const double* __restrict__ x, const int32_t* __restrict__ idx, int64_t g,
                      double* out) {
  double s = 0.0;
  const int64_t step = (int64_t)gridDim.x * blockDim.x * 8;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < g; i += step) {
    const int4 a = *reinterpret_cast<const int4*>(idx + i);
    const int4 b = *reinterpret_cast<const int4*>(idx + i + 4);
    const int c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[u]) : "l"(x + c[u]));
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  if (s == 12345.678) *out = s;
}

#ifndef STAGES
#define STAGES 4
#endif
constexpr int kStages = STAGES;
constexpr int kBytesPerRound = 32 * 4 * 32;  // 32 lanes x 4 rows x 32 B (128-byte aligned slots)

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one warp = one gather stream: each round, every lane issues one gather4
// (its 4 indices), lane 0 arms the stage's mbarrier for the round's bytes
__global__ void __launch_bounds__(1024, 1) k_tma(const __grid_constant__ CUtensorMap tm,
                                                const int32_t* __restrict__ idx, int64_t g,
                                                double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + w * kStages;
  unsigned char* buf = smem + 1024 + (size_t)w * kStages * kBytesPerRound;
  if (lane == 0)
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(bars + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t per_round = 128;  // gathers per warp round
  const int64_t gw = (int64_t)gridDim.x * nw;
  const int64_t wid = (int64_t)blockIdx.x * nw + w;
  const int64_t rounds = g / per_round;
  double s = 0.0;
  auto issue = [&](int64_t r, int st) {
    const int32_t* p = idx + r * per_round + lane * 4;
    const int4 q = *reinterpret_cast<const int4*>(p);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bars + st)),
                   "r"(kBytesPerRound)
                   : "memory");
    __syncwarp();
    unsigned char* dst = buf + (size_t)st * kBytesPerRound + lane * 128;
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(saddr(dst)),
        "l"(&tm), "r"(0), "r"(q.x >> 2), "r"(q.y >> 2), "r"(q.z >> 2), "r"(q.w >> 2),
        "r"(saddr(bars + st))
        : "memory");
  };
  int64_t r = wid, k = 0;
  for (int st = 0; st < kStages && wid + st * gw < rounds; ++st) issue(wid + st * gw, st);
  for (; r < rounds; r += gw, ++k) {
    const int st = (int)(k % kStages);
    const uint32_t ph = (uint32_t)((k / kStages) & 1);
    uint32_t ok = 0;
    do {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(saddr(bars + st)), "r"(ph)
          : "memory");
    } while (!ok);
    const int32_t* p = idx + r * per_round + lane * 4;
    const int4 q = *reinterpret_cast<const int4*>(p);
    const double* row = reinterpret_cast<const double*>(buf + (size_t)st * kBytesPerRound + lane * 128);
    s += row[0 + (q.x & 3)] + row[4 + (q.y & 3)] + row[8 + (q.z & 3)] + row[12 + (q.w & 3)];
    __syncwarp();
    const int64_t nr = r + (int64_t)kStages * gw;
    if (nr < rounds) issue(nr, st);
  }
  if (s == 12345.678) *out = s;
}

// one gather4 of rows (3, 10, 77, 1000): the 16-byte rows land in order
__global__ void k_verify(const __grid_constant__ CUtensorMap tm, double* out) {
  __shared__ __align__(128) double buf[16];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bar)), "r"(128)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(saddr(buf)),
        "l"(&tm), "r"(0), "r"(3), "r"(10), "r"(77), "r"(1000), "r"(saddr(&bar))
        : "memory");
    uint32_t ok = 0;
    do {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(saddr(&bar)), "r"(0)
          : "memory");
    } while (!ok);
    for (int i = 0; i < 16; ++i) out[i] = buf[i];
  }
}

int main(int argc, char** argv) {
  std::vector<double> mbs;
  for (int i = 1; i < argc; ++i) mbs.push_back(std::atof(argv[i]));
  if (mbs.empty()) mbs = {32, 64, 128, 1024};
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
  auto encode = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                              const cuuint32_t*, CUtensorMapInterleave,
                                              CUtensorMapSwizzle, CUtensorMapL2promotion,
                                              CUtensorMapFloatOOBfill)>(fn);
  const int64_t g = 1ll << 28;
  int32_t* idx = nullptr;
  double *out = nullptr;
  CK(cudaMalloc(&idx, g * 4));
  CK(cudaMalloc(&out, 8));
  for (double mb : mbs) {
    const int64_t n = (int64_t)(mb * 1e6 / 8) & ~int64_t(3);
    double* x = nullptr;
    CK(cudaMalloc(&x, n * 8));
    std::vector<double> hx(n);
    for (int64_t i = 0; i < n; ++i) hx[i] = (double)(i % 1000) * 0.001;
    CK(cudaMemcpy(x, hx.data(), n * 8, cudaMemcpyHostToDevice));
    std::vector<int32_t> hi(g);
    uint64_t st = 88172645463325252ull;
    for (int64_t i = 0; i < g; ++i) {
      st ^= st << 13, st ^= st >> 7, st ^= st << 17;
      hi[i] = (int32_t)(st % (uint64_t)n);
    }
    CK(cudaMemcpy(idx, hi.data(), g * 4, cudaMemcpyHostToDevice));
    CUtensorMap tm;
    const cuuint64_t dims[2] = {4, (cuuint64_t)(n / 4)};
    const cuuint64_t strides[1] = {32};
    const cuuint32_t box[2] = {4, 1};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      std::printf("encode failed %d\n", (int)r);
      return 1;
    }
    {
      double* vo = nullptr;
      CK(cudaMalloc(&vo, 128));
      std::vector<double> hx2(n);
      for (int64_t i = 0; i < n; ++i) hx2[i] = (double)i;
      CK(cudaMemcpy(x, hx2.data(), n * 8, cudaMemcpyHostToDevice));
      k_verify<<<1, 32>>>(tm, vo);
      CK(cudaDeviceSynchronize());
      double hv[16];
      CK(cudaMemcpy(hv, vo, 128, cudaMemcpyDeviceToHost));
      std::printf("gather4 rows 3,10,77,1000 ->");
      for (double v : hv) std::printf(" %.0f", v);
      std::printf("  (want 12-15 40-43 308-311 4000-4003)\n");
      CK(cudaFree(vo));
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int warps : {16, 32}) {
      k_ldg<<<sms * 4, warps * 8>>>(x, idx, g, out);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      k_ldg<<<sms * 4, warps * 8>>>(x, idx, g, out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      std::printf("x %7.1f MB  LDG  %2d warps/SM: %7.1f G gathers/s\n", mb, warps, g / ms / 1e6);
    }
    for (int warps : {8, 12, 16}) {
      if ((size_t)warps * kStages * kBytesPerRound + 1024 > 227 * 1024) continue;
      const size_t smem = 1024 + (size_t)warps * kStages * kBytesPerRound;
      CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_tma<<<sms, warps * 32, smem>>>(tm, idx, g, out);
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      k_tma<<<sms, warps * 32, smem>>>(tm, idx, g, out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      std::printf("x %7.1f MB  TMA gather4 %2d warps/SM: %7.1f G gathers/s\n", mb, warps, g / ms / 1e6);
    }
    // correctness of the gather4 path: sum over the first rounds vs host
    CK(cudaFree(x));
  }
  std::printf("done\n");
  return 0;
}
