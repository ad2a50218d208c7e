// reabsorb.cu -- step a5: the Hastings update that writes the truncated factors
// back into the site store with the new, dynamic bond dimension k (U
// left-normalised, V^dagger right-normalised; SURVEY §8(c) algorithm item 7):
//   nu            = sqrt(sum_{j<k} sigma_pi_j^2)          (selector)
//   lambda_i[j]   = sigma_pi_j / nu
//   B_{i+1}[j,t,c] = conj(V_k[(t,c), j])                    (rows of V_k^H, right-normalised)
//   B_i[(a,s), j]  = (Theta' V_k[:, j]) / nu                (an m x n x k GEMM; avoids lambda^-1)
// with V_k = V[:, pi_0..pi_{k-1}] re-orthonormalised first by one Newton-Schulz step,
//   V_k <- V_k (3 I - V_k^H V_k) / 2 = V_k + V_k E,  E = (I - V_k^H V_k) / 2   (FP64 Gram),
// which takes the FP32-accumulated Jacobi rotations from ||V_k^H V_k - I|| ~ eps32 sqrt(n S) to
// O(that^2): the kept right factor is then right-normalised to storage precision, so the update
// does not inject the FP32 drift of V into the state.
// Grids are sized on the host for the worst case k <= min(m, n) (the host does not know k
// without a sync); tiles beyond the selector's k exit at once.
#include "eamps_internal.cuh"

namespace eamps {

namespace {

__device__ __forceinline__ int find_gate(const int32_t* prefix, int G, int tile) {
  int lo = 0, hi = G - 1;
  while (lo < hi) {
    int md = (lo + hi + 1) >> 1;
    if (prefix[md] <= tile) lo = md; else hi = md - 1;
  }
  return lo;
}

// E[a][b] = (delta_ab - sum_i conj(V[i, pi_a]) V[i, pi_b]) / 2, row-major k x k (FP32 storage of
// an FP64-accumulated Gram; E is O(eps32 sqrt(n S)), so its FP32 rounding is negligible)
__global__ void __launch_bounds__(256) k_vk_gram(const GateDesc* __restrict__ desc, const int32_t* __restrict__ prefix,
                                                 int G, uint8_t* slab) {
  const int g = find_gate(prefix, G, blockIdx.x);
  const GateDesc gd = desc[g];
  const int k = gd.k;
  if (k <= 0) return;
  const int kmt = (min(gd.m, gd.n) + 31) / 32;
  const int local = blockIdx.x - prefix[g];
  const int a0 = (local / kmt) * 32, b0 = (local % kmt) * 32;
  if (a0 >= k || b0 >= k) return;
  const int n = gd.n, np = gd.n_pad;
  const float2* __restrict__ V = reinterpret_cast<const float2*>(slab + gd.ws_V);
  const int32_t* __restrict__ pi = reinterpret_cast<const int32_t*>(slab + gd.ws_pi);
  float2* E = reinterpret_cast<float2*>(slab + gd.ws_E);
  __shared__ float2 Va[64][33], Vb[64][33];
  __shared__ int32_t pa[32], pb[32];
  const int tid = threadIdx.x;
  if (tid < 32) pa[tid] = (a0 + tid < k) ? pi[a0 + tid] : -1;
  else if (tid < 64) pb[tid - 32] = (b0 + tid - 32 < k) ? pi[b0 + tid - 32] : -1;
  __syncthreads();
  const int p = tid >> 3, q4 = (tid & 7) * 4;
  double2 dacc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) dacc[j] = make_double2(0.0, 0.0);
  for (int r0 = 0; r0 < n; r0 += 64) {
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int i = tid & 63, c = (tid >> 6) + 4 * it;
      int row = r0 + i;
      Va[i][c] = (row < n && pa[c] >= 0) ? V[(int64_t)pa[c] * np + row] : make_float2(0.f, 0.f);
      Vb[i][c] = (row < n && pb[c] >= 0) ? V[(int64_t)pb[c] * np + row] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    float2 acc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = make_float2(0.f, 0.f);
    for (int i = 0; i < 64; ++i) {
      float2 x = Va[i][p];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 y = Vb[i][q4 + j];
        acc[j].x = fmaf(x.x, y.x, fmaf(x.y, y.y, acc[j].x));
        acc[j].y = fmaf(x.x, y.y, fmaf(-x.y, y.x, acc[j].y));
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) { dacc[j].x += acc[j].x; dacc[j].y += acc[j].y; }
    __syncthreads();
  }
  const int a = a0 + p;
  if (a < k) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int b = b0 + q4 + j;
      if (b >= k) continue;
      double re = ((a == b) ? 1.0 : 0.0) - dacc[j].x, im = -dacc[j].y;
      E[(int64_t)a * k + b] = make_float2((float)(0.5 * re), (float)(0.5 * im));
    }
  }
}

// V_k'[:, b] = V[:, pi_b] + sum_a V[:, pi_a] E[a][b], stored compactly (n x k, ld n) in ws_theta
__global__ void __launch_bounds__(256) k_vk_apply(const GateDesc* __restrict__ desc, const int32_t* __restrict__ prefix,
                                                  int G, uint8_t* slab) {
  const int g = find_gate(prefix, G, blockIdx.x);
  const GateDesc gd = desc[g];
  const int k = gd.k;
  if (k <= 0) return;
  const int n = gd.n, np = gd.n_pad;
  const int kmt = (min(gd.m, gd.n) + 63) / 64;
  const int local = blockIdx.x - prefix[g];
  const int row0 = (local / kmt) * 64, b0 = (local % kmt) * 64;
  if (row0 >= n || b0 >= k) return;
  const float2* __restrict__ V = reinterpret_cast<const float2*>(slab + gd.ws_V);
  const int32_t* __restrict__ pi = reinterpret_cast<const int32_t*>(slab + gd.ws_pi);
  const float2* __restrict__ E = reinterpret_cast<const float2*>(slab + gd.ws_E);
  float2* Vk = reinterpret_cast<float2*>(slab + gd.ws_theta);
  __shared__ float2 As[16][65];
  __shared__ float2 Bs[16][65];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  float2 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = make_float2(0.f, 0.f);
  for (int a0 = 0; a0 < k; a0 += 16) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      int e = tid + it * 256;
      int i = e & 63, kk = e >> 6;
      int row = row0 + i, a = a0 + kk;
      As[kk][i] = (row < n && a < k) ? V[(int64_t)pi[a] * np + row] : make_float2(0.f, 0.f);
      int bb = e & 63;
      int b = b0 + bb;
      Bs[kk][bb] = (a < k && b < k) ? E[(int64_t)a * k + b] : make_float2(0.f, 0.f);
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
    if (row >= n) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int bc = b0 + tx + 16 * b;
      if (bc >= k) continue;
      float2 v = V[(int64_t)pi[bc] * np + row];
      Vk[(int64_t)bc * n + row] = make_float2(v.x + acc[a][b].x, v.y + acc[a][b].y);
    }
  }
}

__global__ void __launch_bounds__(256) k_reabsorb(const GateDesc* __restrict__ desc, const int32_t* __restrict__ prefix,
                                                  int G, uint8_t* slab) {
  const int g = find_gate(prefix, G, blockIdx.x);
  const GateDesc gd = desc[g];
  const int k = gd.k;
  if (k <= 0) return;
  const int m = gd.m, n = gd.n;
  const int kmax_tiles_j = (min(m, n) + 63) / 64;
  const int gemm_tiles = ((m + 63) / 64) * kmax_tiles_j;
  const int local = blockIdx.x - prefix[g];
  const float2* __restrict__ Vk = reinterpret_cast<const float2*>(slab + gd.ws_theta);  // n x k, ld n
  const float inv_nu = (float)(1.0 / gd.nu);
  const int tid = threadIdx.x;

  if (local >= gemm_tiles) {
    // rows j0 .. j0+63 of B_{i+1}' = conj(V_k[:, j]) (contiguous copy) and lambda_i[j]
    const int j0 = (local - gemm_tiles) * 64;
    if (j0 >= k) return;
    const int j1 = min(k, j0 + 64);
    const float2* src = Vk + (int64_t)j0 * n;
    float2* dst = reinterpret_cast<float2*>(slab + gd.off_newR) + (int64_t)j0 * n;
    const int64_t cnt = (int64_t)(j1 - j0) * n;
    for (int64_t x = tid; x < cnt; x += 256) {
      float2 v = src[x];
      dst[x] = make_float2(v.x, -v.y);
    }
    if (tid < j1 - j0) {
      const double* s2 = reinterpret_cast<const double*>(slab + gd.ws_sig2);
      reinterpret_cast<float*>(slab + gd.off_newLam)[j0 + tid] = (float)(sqrt(s2[j0 + tid]) / gd.nu);
    }
    return;
  }
  const int row0 = (local / kmax_tiles_j) * 64, j0 = (local % kmax_tiles_j) * 64;
  if (j0 >= k || row0 >= m) return;
  const float2* __restrict__ thp = reinterpret_cast<const float2*>(slab + gd.ws_thetap);
  float2* __restrict__ Bl = reinterpret_cast<float2*>(slab + gd.off_newL);

  __shared__ float2 As[16][65];
  __shared__ float2 Bs[16][65];
  const int ty = tid >> 4, tx = tid & 15;
  double2 dacc[4][4];  // FP32 chunk products, FP64 chunk sums (DESIGN "Precision")
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) dacc[a][b] = make_double2(0.0, 0.0);
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
      int col = k0 + kk, j = j0 + jj;
      Bs[kk][jj] = (j < k && col < n) ? Vk[(int64_t)j * n + col] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    float2 acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = make_float2(0.f, 0.f);
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
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) { dacc[a][b].x += acc[a][b].x; dacc[a][b].y += acc[a][b].y; }
    __syncthreads();
  }
  const double inv = 1.0 / gd.nu;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int row = row0 + ty + 16 * a;
    if (row >= m) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      int j = j0 + tx + 16 * b;
      if (j < k) Bl[(int64_t)row * k + j] = make_float2((float)(dacc[a][b].x * inv), (float)(dacc[a][b].y * inv));
    }
  }
  (void)inv_nu;
}

}  // namespace

void launch_reabsorb(const GateDesc* d_desc, const int32_t* d_pre_gram, int tiles_gram, const int32_t* d_pre_apply,
                     int tiles_apply, const int32_t* d_pre_reab, int tiles_reab, int G, uint8_t* slab, cudaStream_t s) {
  if (G <= 0) return;
  if (tiles_gram > 0) k_vk_gram<<<tiles_gram, 256, 0, s>>>(d_desc, d_pre_gram, G, slab);
  if (tiles_apply > 0) k_vk_apply<<<tiles_apply, 256, 0, s>>>(d_desc, d_pre_apply, G, slab);
  if (tiles_reab > 0) k_reabsorb<<<tiles_reab, 256, 0, s>>>(d_desc, d_pre_reab, G, slab);
}

}  // namespace eamps
