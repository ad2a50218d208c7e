// peaks.cu -- measured roofline denominators on this box: the FP32 SIMT
// peak (scalar FFMA and packed FFMA2), the FP64 DFMA peak and the tcgen05 kind::tf32 dense
// tensor peak, each as a long register/TMEM-resident loop timed with CUDA events.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../../paper_2307_16870_b200/csrc peaks.cu -o peaks
//   ./peaks            -> one JSON line (TFLOP/s, SM clock during the run is sampled by the caller)
//
// Every loop is built so that the compiler cannot fold it (the accumulators depend on runtime
// inputs and are stored at the end) and so that the issue rate, not latency, binds: 8 independent
// FMA chains per thread (latency 4, issue interval 2 per SMSP => 2 chains per SMSP suffice), 4
// warps per SMSP. The tensor loop issues M=128 N=256 K=8 TF32 MMAs from one thread per CTA, one
// CTA per SM, with operands resident in shared memory (the MMA reads them every time).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace eamps;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr int kChains = 8;

__global__ void k_ffma(float* out, float a, float b, int iters) {
  float acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = fmaf(acc[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.f) out[threadIdx.x] = s;
}

// packed FP32x2 FMA (sm_100: fma.rn.f32x2 -> FFMA2), two FMAs per lane per instruction
__device__ __forceinline__ unsigned long long ffma2(unsigned long long x, unsigned long long y, unsigned long long z) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;\n" : "=l"(d) : "l"(x), "l"(y), "l"(z));
  return d;
}

__global__ void k_ffma2(float* out, float a, float b, int iters) {
  unsigned long long acc[kChains];
  const float2 av = make_float2(a, a), bv = make_float2(b, b);
  const unsigned long long A = *reinterpret_cast<const unsigned long long*>(&av);
  const unsigned long long B = *reinterpret_cast<const unsigned long long*>(&bv);
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    float2 v = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
    acc[c] = *reinterpret_cast<unsigned long long*>(&v);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = ffma2(acc[c], A, B);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    float2 v = *reinterpret_cast<float2*>(&acc[c]);
    s += v.x + v.y;
  }
  if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void k_dfma(double* out, double a, double b, int iters) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.0) out[threadIdx.x] = s;
}

// tcgen05 kind::tf32, cta_group::1, M = 128, N = NN, K = 8 per instruction; A (128 x 8) and B
// (NN x 8) K-major SWIZZLE_NONE in shared memory; D (128 x NN fp32) in TMEM.
template <int NN>
__global__ void __launch_bounds__(128, 1) k_tc_tf32(float* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  constexpr int M = 128, K = 8;
  uint8_t* sa = sm;                        // 128 x 8 x 4 B = 4 KB
  uint8_t* sb = sm + M * K * 4;            // NN x 8 x 4 B
  const int tid = threadIdx.x, warp = tid >> 5;
  // canonical K-major: core matrix = 8 rows x 16 B; SBO = 128 B (next 8 rows), LBO = rows*16 B (next 4 k)
  const uint32_t sboA = 128, lboA = M * 16, sboB = 128, lboB = NN * 16;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<float*>(sa + tc::kmaj_off(r, k, lboA, sboA)) = tc::tf32_trunc(1.0f + 0.001f * ((r * 7 + k) % 13));
  }
  for (int i = tid; i < NN * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<float*>(sb + tc::kmaj_off(r, k, lboB, sboB)) = tc::tf32_trunc(0.5f - 0.001f * ((r * 5 + k) % 11));
  }
  tc::fence_async_smem();
  if (warp == 0) tc::tmem_alloc(&tmem_base, NN < 32 ? 32 : NN);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint64_t ad = tc::make_desc(tc::smem_u32(sa), lboA, sboA);
    const uint64_t bd = tc::make_desc(tc::smem_u32(sb), lboB, sboB);
    constexpr uint32_t idesc = tc::make_idesc_tf32(M, NN, false, false);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) tc::mma_tf32(tmem, ad, bd, idesc, (i | u) ? 1u : 0u);
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  float v[8];
  tc::tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16), v);
  if (v[0] == 12345.f) out[tid] = v[1];
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, NN < 32 ? 32 : NN);
}

template <typename F>
static float time_ms(F launch, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();  // warm-up
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    launch();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  float* fo;
  double* dout;
  CK(cudaMalloc(&fo, 4096 * sizeof(float)));
  CK(cudaMalloc(&dout, 4096 * sizeof(double)));
  const int threads = 512, blocks = sms * 4;   // 64 warps per SM
  const int iters = 4096;
  const double fl_per_thread = 2.0 * 16 * kChains * iters;
  float ms_f = time_ms([&] { k_ffma<<<blocks, threads>>>(fo, 0.999f, 1e-4f, iters); }, 5);
  float ms_f2 = time_ms([&] { k_ffma2<<<blocks, threads>>>(fo, 0.999f, 1e-4f, iters); }, 5);
  const int diters = 512;
  float ms_d = time_ms([&] { k_dfma<<<blocks, threads>>>(dout, 0.999, 1e-4, diters); }, 5);
  const double nthr = (double)blocks * threads;
  const double tf_ffma = nthr * fl_per_thread / (ms_f * 1e-3) / 1e12;
  const double tf_ffma2 = 2.0 * nthr * fl_per_thread / (ms_f2 * 1e-3) / 1e12;
  const double tf_dfma = nthr * (2.0 * 16 * kChains * diters) / (ms_d * 1e-3) / 1e12;
  // tensor: one CTA per SM
  const int titers = 20000;
  const size_t smem256 = 128 * 8 * 4 + 256 * 8 * 4, smem128 = 128 * 8 * 4 + 128 * 8 * 4;
  CK(cudaFuncSetAttribute(k_tc_tf32<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem256));
  CK(cudaFuncSetAttribute(k_tc_tf32<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem128));
  float ms_t256 = time_ms([&] { k_tc_tf32<256><<<sms, 128, smem256>>>(fo, titers); }, 5);
  float ms_t128 = time_ms([&] { k_tc_tf32<128><<<sms, 128, smem128>>>(fo, titers); }, 5);
  const double tf_t256 = (double)sms * titers * 8 * (2.0 * 128 * 256 * 8) / (ms_t256 * 1e-3) / 1e12;
  const double tf_t128 = (double)sms * titers * 8 * (2.0 * 128 * 128 * 8) / (ms_t128 * 1e-3) / 1e12;
  printf("{\"sms\": %d, \"clock_attr_mhz\": %.0f, \"fp32_ffma_tflops\": %.2f, \"fp32_ffma2_tflops\": %.2f, "
         "\"fp64_dfma_tflops\": %.2f, \"tf32_tcgen05_m128n256_tflops\": %.1f, \"tf32_tcgen05_m128n128_tflops\": %.1f, "
         "\"ms\": {\"ffma\": %.3f, \"ffma2\": %.3f, \"dfma\": %.3f, \"tc256\": %.3f, \"tc128\": %.3f}}\n",
         sms, clk_khz / 1e3, tf_ffma, tf_ffma2, tf_dfma, tf_t256, tf_t128, ms_f, ms_f2, ms_d, ms_t256, ms_t128);
  return 0;
}
