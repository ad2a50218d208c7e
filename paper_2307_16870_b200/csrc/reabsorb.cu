// reabsorb.cu -- step a5: the Hastings update that writes the truncated factors
// back into the site store with the new, dynamic bond dimension k (U
// left-normalised, V^dagger right-normalised; SURVEY §8(c) algorithm item 7):
//   nu            = sqrt(sum_{j<k} sigma_pi_j^2)          (selector)
//   lambda_i[j]   = sigma_pi_j / nu
//   B_{i+1}[j,t,c] = conj(V[(t,c), pi_j])                   (rows of V_k^H, right-normalised)
//   B_i[(a,s), j]  = (Theta' V[:, pi_j]) / nu               (an m x n x k GEMM; avoids lambda^-1)
// One launch per wave. The grid is sized on the host for the worst case k <= min(m, n, cap)
// (the host does not know k without a sync); tiles beyond the selector's k exit at once.
#include "eamps_internal.cuh"

namespace eamps {

namespace {

__global__ void __launch_bounds__(256) k_reabsorb(const GateDesc* __restrict__ desc, const int32_t* __restrict__ prefix,
                                                  int G, uint8_t* slab) {
  const int tile = blockIdx.x;
  int lo = 0, hi = G - 1;
  while (lo < hi) {
    int md = (lo + hi + 1) >> 1;
    if (prefix[md] <= tile) lo = md; else hi = md - 1;
  }
  const GateDesc gd = desc[lo];
  const int k = gd.k;
  if (k <= 0) return;
  const int m = gd.m, n = gd.n, np = gd.n_pad;
  const int kmax_tiles_j = (min(m, n) + 63) / 64;
  const int gemm_tiles = ((m + 63) / 64) * kmax_tiles_j;
  int local = tile - prefix[lo];
  const float2* __restrict__ V = reinterpret_cast<const float2*>(slab + gd.ws_V);
  const int32_t* __restrict__ pi = reinterpret_cast<const int32_t*>(slab + gd.ws_pi);
  const float inv_nu = (float)(1.0 / gd.nu);
  const int tid = threadIdx.x;

  if (local >= gemm_tiles) {
    // copy row j of B_{i+1}' = conj(V[:, pi_j]) and lambda_i[j]
    const int j = local - gemm_tiles;
    if (j >= k) return;
    const float2* vj = V + (int64_t)pi[j] * np;
    float2* Br = reinterpret_cast<float2*>(slab + gd.off_newR) + (int64_t)j * n;
    for (int c = tid; c < n; c += 256) {
      float2 v = vj[c];
      Br[c] = make_float2(v.x, -v.y);
    }
    if (tid == 0) {
      const double* s2 = reinterpret_cast<const double*>(slab + gd.ws_sig2);
      reinterpret_cast<float*>(slab + gd.off_newLam)[j] = (float)(sqrt(s2[j]) / gd.nu);
    }
    return;
  }
  const int row0 = (local / kmax_tiles_j) * 64, j0 = (local % kmax_tiles_j) * 64;
  if (j0 >= k || row0 >= m) return;
  const float2* __restrict__ thp = reinterpret_cast<const float2*>(slab + gd.ws_thetap);
  float2* __restrict__ Bl = reinterpret_cast<float2*>(slab + gd.off_newL);

  __shared__ float2 As[16][65];
  __shared__ float2 Bs[16][65];
  __shared__ int32_t pis[64];
  if (tid < 64) pis[tid] = (j0 + tid < k) ? pi[j0 + tid] : -1;
  __syncthreads();
  const int ty = tid >> 4, tx = tid & 15;
  float2 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = make_float2(0.f, 0.f);
  for (int k0 = 0; k0 < n; k0 += 16) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      int e = tid + it * 256;
      int i = e & 63, kk = e >> 6;
      int row = row0 + i, col = k0 + kk;
      As[kk][i] = (row < m && col < n) ? thp[(int64_t)col * m + row] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      int e = tid + it * 256;
      int kk = e & 15, jj = e >> 4;
      int col = k0 + kk, p = pis[jj];
      Bs[kk][jj] = (p >= 0 && col < n) ? V[(int64_t)p * np + col] : make_float2(0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float2 av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          acc[a][b].x = fmaf(av[a].x, bv[b].x, fmaf(-av[a].y, bv[b].y, acc[a][b].x));
          acc[a][b].y = fmaf(av[a].x, bv[b].y, fmaf(av[a].y, bv[b].x, acc[a][b].y));
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int row = row0 + ty + 16 * a;
    if (row >= m) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int j = j0 + tx + 16 * b;
      if (j < k) Bl[(int64_t)row * k + j] = make_float2(acc[a][b].x * inv_nu, acc[a][b].y * inv_nu);
    }
  }
}

}  // namespace

void launch_reabsorb(const GateDesc* d_desc, const int32_t* d_tile_prefix, int G, int total_tiles, int d,
                     uint8_t* slab, DevState* st, cudaStream_t s) {
  (void)d; (void)st;
  if (total_tiles <= 0) return;
  k_reabsorb<<<total_tiles, 256, 0, s>>>(d_desc, d_tile_prefix, G, slab);
}

}  // namespace eamps
