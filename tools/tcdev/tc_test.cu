// Development check of the tcgen05 kind::tf32 building blocks (tc_common.cuh): C = A B with
// 3xTF32, A 128 x K, B K x N (row-major FP32 in global), A staged K-major or MN-major, B staged
// K-major or MN-major. Not part of the library.
#include "tc_common.cuh"
using namespace eamps::tc;

__global__ void __launch_bounds__(128) k_tc_test(const float* A, const float* B, float* C, int K, int N, int a_mn,
                                                 int b_mn, int swap) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int M = 128;
  uint8_t* sAh = sm;
  uint8_t* sAl = sAh + M * K * 4;
  uint8_t* sBh = sAl + M * K * 4;
  uint8_t* sBl = sBh + N * K * 4;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  uint32_t a_lbo = a_mn ? (M / 4) * 128 : (M / 8) * 128, a_sbo = 128;
  const uint32_t b_lbo = b_mn ? (N / 4) * 128 : (N / 8) * 128, b_sbo = 128;
  for (int x = tid; x < M * K; x += blockDim.x) {
    int r = x / K, k = x % K;
    float h, l;
    split_tf32(A[x], h, l);
    uint32_t o = a_mn ? mnmaj_off(r, k, a_lbo, a_sbo) : kmaj_off(r, k, a_lbo, a_sbo);
    *reinterpret_cast<float*>(sAh + o) = h;
    *reinterpret_cast<float*>(sAl + o) = l;
  }
  for (int x = tid; x < K * N; x += blockDim.x) {
    int k = x / N, n = x % N;
    float h, l;
    split_tf32(B[x], h, l);
    uint32_t o = b_mn ? mnmaj_off(n, k, b_lbo, b_sbo) : kmaj_off(n, k, b_lbo, b_sbo);
    *reinterpret_cast<float*>(sBh + o) = h;
    *reinterpret_cast<float*>(sBl + o) = l;
  }
  const uint32_t dl = swap ? a_sbo : a_lbo, ds = swap ? a_lbo : a_sbo;  // descriptor fields only
  if (warp == 0) tmem_alloc(&tbase, N < 32 ? 32 : N);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t idesc = make_idesc_tf32(M, N, a_mn, b_mn);
    for (int s = 0; s < K / 8; ++s) {
      const uint32_t aoff = a_mn ? s * a_lbo : 2 * s * a_lbo;
      const uint32_t boff = b_mn ? s * b_lbo : 2 * s * b_lbo;
      const uint64_t ah = make_desc(smem_u32(sAh) + aoff, dl, ds);
      const uint64_t al = make_desc(smem_u32(sAl) + aoff, dl, ds);
      const uint64_t bh = make_desc(smem_u32(sBh) + boff, b_lbo, b_sbo);
      const uint64_t bl = make_desc(smem_u32(sBl) + boff, b_lbo, b_sbo);
      mma_tf32(tmem, ah, bh, idesc, s > 0);
      mma_tf32(tmem, ah, bl, idesc, 1);
      mma_tf32(tmem, al, bh, idesc, 1);
    }
    mma_commit(&mbar);
  }
  __syncwarp();
  mbar_wait(&mbar, 0);
  fence_after_sync();
  const int row = warp * 32 + (tid & 31);
  for (int c = 0; c < N; c += 8) {
    float v[8];
    tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    for (int i = 0; i < 8; ++i) C[row * N + c + i] = v[i];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, N < 32 ? 32 : N);
}

extern "C" int tc_test(const float* A, const float* B, float* C, int K, int N, int a_mn, int b_mn, int swap) {
  size_t smem = (size_t)(128 * K * 2 + N * K * 2) * 4;
  cudaFuncSetAttribute(k_tc_test, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_tc_test<<<1, 128, smem>>>(A, B, C, K, N, a_mn, b_mn, swap);
  cudaError_t e = cudaDeviceSynchronize();
  return (int)e;
}
