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
  // Vb rows padded to 36 float2 (16-byte aligned): a thread's 4 partner columns q4 .. q4+3 are two
  // 16-byte loads instead of four 8-byte ones (ncu r02: short scoreboard 13 warps per issue)
  __shared__ float2 Va[64][33];
  __shared__ __align__(16) float2 Vb[64][36];
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
#pragma unroll 4
    for (int i = 0; i < 64; ++i) {
      const float2 x = Va[i][p];
      const float4 y01 = *reinterpret_cast<const float4*>(&Vb[i][q4]);
      const float4 y23 = *reinterpret_cast<const float4*>(&Vb[i][q4 + 2]);
      const float2 y[4] = {make_float2(y01.x, y01.y), make_float2(y01.z, y01.w), make_float2(y23.x, y23.y),
                           make_float2(y23.z, y23.w)};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[j].x = fmaf(x.x, y[j].x, fmaf(x.y, y[j].y, acc[j].x));
        acc[j].y = fmaf(x.x, y[j].y, fmaf(-x.y, y[j].x, acc[j].y));
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

__global__ void __launch_bounds__(256, 2) k_reabsorb(const GateDesc* __restrict__ desc, const int32_t* __restrict__ prefix,
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
  // 128 registers (2 CTAs per SM; at 177 one CTA per SM left the FP32 pipe latency-bound, ncu r02)
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


// ---- small gates (m, n <= 64; config 2 chi <= 32, the small bonds of every circuit): the three
// steps above fused in ONE CTA per gate with everything in shared memory -- V_k gathered once,
// E = (I - V_k^H V_k)/2, V_k' = V_k + V_k E, B_i' = Theta' V_k' / nu, B_{i+1}' = V_k'^H, lambda_i.
// Same arithmetic in the same order as k_vk_gram / k_vk_apply / k_reabsorb (one 64-row FP32 chunk
// of the Gram for n <= 64 then FP64, FP32 accumulation of V_k E in ascending a, FP32 16-column
// chunk products with FP64 sums for B_i'), so the results are those of the tiled path; what goes
// is three launches of mostly idle 64 x 64 tiles and the global round trips of E and V_k'.
// Columns of V_k / V_k' are stored with stride n + 1 (odd: no shared-memory bank pile-up).
__global__ void __launch_bounds__(256) k_reabsorb_small(const GateDesc* __restrict__ desc,
                                                        const int32_t* __restrict__ list, uint8_t* slab) {
  const GateDesc gd = desc[list[blockIdx.x]];
  const int k = gd.k;
  if (k <= 0) return;
  const int m = gd.m, n = gd.n, np = gd.n_pad, ld = n + 1;
  extern __shared__ __align__(16) float2 rs_sm[];
  float2* Vs = rs_sm;                      // V[:, pi_c], column c at Vs[c * ld + row]
  float2* Vk = Vs + (size_t)k * ld;        // V_k'
  float2* Es = Vk + (size_t)k * ld;        // E[a][b] at Es[a * k + b]
  float2* Ts = Es + (size_t)k * k;         // Theta' (m x n, column-major, ld m)
  const float2* __restrict__ V = reinterpret_cast<const float2*>(slab + gd.ws_V);
  const int32_t* __restrict__ pi = reinterpret_cast<const int32_t*>(slab + gd.ws_pi);
  const float2* __restrict__ thp = reinterpret_cast<const float2*>(slab + gd.ws_thetap);
  const int tid = threadIdx.x;
  for (int x = tid; x < n * k; x += 256) {
    const int c = x / n, row = x % n;
    Vs[c * ld + row] = V[(int64_t)pi[c] * np + row];
  }
  for (int x = tid; x < m * n; x += 256) Ts[x] = thp[x];
  __syncthreads();
  // E[a][b] = (delta_ab - sum_i conj(V[i, pi_a]) V[i, pi_b]) / 2
  for (int x = tid; x < k * k; x += 256) {
    const int a = x / k, b = x % k;
    float2 acc = make_float2(0.f, 0.f);
    for (int i = 0; i < n; ++i) {
      const float2 u = Vs[a * ld + i], y = Vs[b * ld + i];
      acc.x = fmaf(u.x, y.x, fmaf(u.y, y.y, acc.x));
      acc.y = fmaf(u.x, y.y, fmaf(-u.y, y.x, acc.y));
    }
    const double dre = (double)acc.x, dim = (double)acc.y;
    const double re = ((a == b) ? 1.0 : 0.0) - dre, im = -dim;
    Es[x] = make_float2((float)(0.5 * re), (float)(0.5 * im));
  }
  __syncthreads();
  // V_k'[:, b] = V[:, pi_b] + sum_a V[:, pi_a] E[a][b]
  for (int x = tid; x < n * k; x += 256) {
    const int b = x / n, row = x % n;
    float2 acc = make_float2(0.f, 0.f);
    for (int a = 0; a < k; ++a) {
      const float2 av = Vs[a * ld + row], bv = Es[a * k + b];
      acc.x = fmaf(av.x, bv.x, fmaf(-av.y, bv.y, acc.x));
      acc.y = fmaf(av.x, bv.y, fmaf(av.y, bv.x, acc.y));
    }
    const float2 v = Vs[b * ld + row];
    Vk[b * ld + row] = make_float2(v.x + acc.x, v.y + acc.y);
  }
  __syncthreads();
  // B_i'[row][j] = (Theta' V_k')[row][j] / nu: FP32 products in 16-column chunks, FP64 sums
  float2* __restrict__ Bl = reinterpret_cast<float2*>(slab + gd.off_newL);
  const double inv = 1.0 / gd.nu;
  for (int x = tid; x < m * k; x += 256) {
    const int row = x / k, j = x % k;
    double2 dacc = make_double2(0.0, 0.0);
    for (int c0 = 0; c0 < n; c0 += 16) {
      float2 acc = make_float2(0.f, 0.f);
      const int c1 = min(n, c0 + 16);
      for (int c = c0; c < c1; ++c) {
        const float2 av = Ts[(size_t)c * m + row], bv = Vk[j * ld + c];
        acc.x = fmaf(av.x, bv.x, fmaf(-av.y, bv.y, acc.x));
        acc.y = fmaf(av.x, bv.y, fmaf(av.y, bv.x, acc.y));
      }
      dacc.x += acc.x;
      dacc.y += acc.y;
    }
    Bl[x] = make_float2((float)(dacc.x * inv), (float)(dacc.y * inv));
  }
  // B_{i+1}'[j][col] = conj(V_k'[col][j]) and lambda_i[j] = sigma_pi_j / nu
  float2* __restrict__ Br = reinterpret_cast<float2*>(slab + gd.off_newR);
  for (int x = tid; x < k * n; x += 256) {
    const int j = x / n, col = x % n;
    const float2 v = Vk[j * ld + col];
    Br[x] = make_float2(v.x, -v.y);
  }
  if (tid < k) {
    const double* s2 = reinterpret_cast<const double*>(slab + gd.ws_sig2);
    reinterpret_cast<float*>(slab + gd.off_newLam)[tid] = (float)(sqrt(s2[tid]) / gd.nu);
  }
}

}  // namespace

bool reabsorb_small_fits(int m, int n) {
  static const bool off = getenv("EAMPS_NO_REABSORB_SMALL") != nullptr;   // dev A/B switch
  return !off && m <= 64 && n <= 64;
}

size_t reabsorb_small_smem(int m, int n) {
  const size_t k = (size_t)std::min(m, n);
  return 8 * (2 * k * (size_t)(n + 1) + k * k + (size_t)m * n);
}

void launch_reabsorb_small(const GateDesc* d_desc, const int32_t* d_list, int count, size_t smem, uint8_t* slab,
                           cudaStream_t s) {
  if (count <= 0) return;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(k_reabsorb_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)reabsorb_small_smem(64, 64));
  k_reabsorb_small<<<count, 256, smem, s>>>(d_desc, d_list, slab);
}

int launch_reabsorb(const GateDesc* d_desc, const int32_t* d_pre_gram, int tiles_gram, const int32_t* d_pre_apply,
                    int tiles_apply, const int32_t* d_pre_reab, int tiles_reab, int G, uint8_t* slab, cudaStream_t s) {
  if (G <= 0) return 0;
  int launches = 0;
  if (tiles_gram > 0) { k_vk_gram<<<tiles_gram, 256, 0, s>>>(d_desc, d_pre_gram, G, slab); ++launches; }
  if (tiles_apply > 0) { k_vk_apply<<<tiles_apply, 256, 0, s>>>(d_desc, d_pre_apply, G, slab); ++launches; }
  if (tiles_reab > 0) { k_reabsorb<<<tiles_reab, 256, 0, s>>>(d_desc, d_pre_reab, G, slab); ++launches; }
  return launches;
}

}  // namespace eamps
