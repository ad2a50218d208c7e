// refine_large.cu -- FP64 spectrum of deep large-n spectra (steps a2/a3): the
// singular values of theta for gates of the large regime with 256 < n <= 4096 whose spectrum is
// deep, as the eigenvalues of the FP64 Gram G = theta^H theta of theta RECONTRACTED in FP64 from the
// complex64 site tensors and gate.
//
// Why (reading 19, "Relative accuracy of small singular values"): the large regime's FP32
// pipeline (FP32-rounded Cholesky factor B = L, 3xTF32 block rotations accumulated over ~13 sweeps x
// 63 rounds) delivers right singular vectors whose error (~1e-6 sigma_max normwise) exceeds the gaps
// of a deep, dense spectrum: at chi = 1024 (theta 2048 x 2048, sigma_k ~ k^-1.5, sigma_min =
// 1.1e-5 sigma_max, neighbouring sigma 7.5e-9 sigma_max apart) the deep right singular vectors are
// mixed over windows of many neighbours, so the Rayleigh quotient of a deep v_j is an average over
// its window (7.9e-4 relative error with the pairwise polish). A Jacobi refinement warm-started from
// that V would have to re-solve the mixed deep subspace from scratch (a numpy model: 3+ cyclic
// sweeps of the 2048 x 2048 C). The eigenvalues of G do not depend on V at all: a backward-stable
// FP64 Hermitian eigensolver gives sigma_j^2 with an absolute error of a few eps64 ||G||, i.e. a
// relative error ~1e-16 / (sigma_j / sigma_max)^2 = 1e-6 at 1.1e-5 (numpy/LAPACK on the chi = 1024
// recipe: 9.4e-9 relative in sigma, this file's recurrence re-run in numpy: 3.8e-9); the FP64
// recontraction removes the FP32 theta's own 2.6e-6.
// What (one wave; gates picked on the device, at most 4096 columns):
//   k_rlg_pick     the trigger (deepest sigma >= 1e-6 sigma_max below kRatio sigma_max)
//   k_rlg_theta    theta64[(a,s),(t,c)] = lambda_a sum_{s',t'} U[s d+t, s' d+t'] sum_b B_i[a,s',b] B_{i+1}[b,t',c]
//                  (E2 of PAPER.md:32-41 / contract.cu with FP64 products and sums)
//   k_rlg_gram     G = theta64^H theta64 (FP64, lower triangle in 32 x 32 tiles)
//   k_rlg_tridiag  one-stage Householder tridiagonalisation Q^H G Q = T (LAPACK zhetd2 recurrence,
//                  lower), all CTAs of a cooperative grid on one gate at a time; the rank-2 update of
//                  step k-1 is applied lazily during step k (each CTA re-derives the pivot row k
//                  itself), so every step costs one grid barrier
//   k_rlg_bisect   eigenvalues of the real symmetric tridiagonal T by Sturm-count multisection
//                  (one thread per eigenvalue index)
//   k_rlg_finish   sigma^2 in descending order + FP64 tails (a3 redone)
// The j-th largest eigenvalue replaces the sigma^2 of the j-th column of the existing order pi (rank
// matching): the kept columns (the top of a deep spectrum) are well separated and unchanged in order;
// the deep columns are mixed among themselves anyway and are never kept (reading 20).
// V itself is not rotated (as refine.cu). PAPER.md:114 ("performing its SVD", "singular values in
// decreasing order"); north_star tolerance "singular values: relative 1e-5 for sigma >= 1e-6 sigma_max".
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "eamps_internal.cuh"
#include "sort_tails.cuh"

namespace eamps {

namespace {

// EAMPS_DEBUG_SYNC=1 (development): synchronise and check after every launch of this file, naming it
void rl_dbg(cudaStream_t s, const char* what) {
  static const bool on = getenv("EAMPS_DEBUG_SYNC") != nullptr;
  if (!on) return;
  cudaStreamSynchronize(s);
  const cudaError_t e = cudaGetLastError();
  fprintf(stderr, "[eamps debug] after %s: %s\n", what, cudaGetErrorString(e));
}

constexpr int kMinN = 257, kMaxN = 4096;   // the refinement of Jacobi spectra (n <= 256: refine.cu)
constexpr int kEigMinN = 129;              // the eigen route
// measured (config 2, r02): chi = 256 (n = 512, sigma_min/sigma_max = 8.6e-5) 2.8e-6 and chi = 512
// (n = 1024, 3.1e-5) 5.8e-6 with Rayleigh + polish -- inside the 1e-5 bar; chi = 1024 (n = 2048,
// 1.1e-5) 7.9e-4. The FP64 eigensolver runs for spectra deeper than 2e-5 sigma_max.
constexpr double kRatio = 2e-5;
constexpr int TT = 512;          // tridiagonalisation threads per CTA
constexpr int BT = 128;          // bisection threads per CTA
constexpr int kMaxGroups = 148, kDefaultGroups = 8;
constexpr int kBisWide = 148 * 256;   // eigenvalues in a launch from which 1 lane per eigenvalue pays

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {   // conj(a) b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

struct RlgLayout {               // per-gate scratch at ws_log (the large regime's dead TC / Gram scratch)
  int64_t g, th, d, e, eig, tau, p, part, y, slot, rs, cs;
};
// G in tile-major lower storage: 32 x 32 tiles (I >= J), tile (I, J) at tile index I (I + 1) / 2 + J,
// row-major inside (diagonal tiles hold both triangles of their block).
constexpr int TB = 32;
__host__ __device__ inline int64_t g_tiles(int n) { const int64_t nt = (n + TB - 1) / TB; return nt * (nt + 1) / 2; }
__device__ __forceinline__ int64_t g_at(int i, int j) {   // i >= j (or the same tile)
  const int I = i / TB, J = j / TB;
  return ((int64_t)I * (I + 1) / 2 + J) * (TB * TB) + (i % TB) * TB + (j % TB);
}
constexpr int kSlots = 128;      // inverse-iteration factor slots per gate (vectors in flight)
__host__ __device__ inline RlgLayout rlg_layout(const GateDesc& gd) {
  RlgLayout L;
  const int64_t n = gd.n, m = gd.m;
  L.g = gd.ws_log;
  L.th = L.g + 16 * n * n;
  L.d = L.th + 16 * m * n;
  L.e = L.d + 8 * n;
  L.eig = L.e + 8 * n;
  L.tau = L.eig + 8 * n;               // n double2: Householder tau_k
  L.p = L.tau + 16 * n;                // 2 x n double2 (by step parity)
  L.part = L.p + 32 * n;               // 2 x 1024 double2 (by step parity)
  L.y = L.part + 32 * 1024;            // n x n doubles: eigenvectors of T (row j = vector j)
  L.slot = L.y + 8 * n * n;            // kSlots x n x (double4 factors + 1 pivot byte)
  L.rs = (L.slot + (int64_t)kSlots * n * 33 + 255) & ~(int64_t)255;   // tile row partials: tiles x TB double2
  L.cs = L.rs + g_tiles(gd.n) * TB * 16;                                // tile column partials
  return L;
}

// ---- trigger --------------------------------------------------------------------------------
// cand[0..nc): wave-local gate indices (large regime, n in range); flag[c] = 1 if the gate is deep;
// list[0] = count, list[1..] = wave-local gate indices.
// mode 0 (refinement of a Jacobi spectrum): large-regime gates of the Jacobi route in range whose
// spectrum is deep; mode 1 (eigen route): every gate marked eig.
__global__ void k_rlg_pick(const GateDesc* __restrict__ desc, const uint8_t* slab, const int32_t* __restrict__ cand,
                           int nc, int32_t* flag, int32_t* list, int mode) {
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= nc) return;
  const GateDesc& gd = desc[cand[c]];
  const int n = gd.n;
  const double* gS = reinterpret_cast<const double*>(slab + gd.ws_sig2);   // sorted descending
  const double smax = mode == 0 ? gS[0] : 0.0;
  double deep = smax;
  for (int j = lane; mode == 0 && j < n; j += 32)
    if (gS[j] >= 1e-12 * smax) deep = fmin(deep, gS[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) deep = fmin(deep, __shfl_xor_sync(0xffffffffu, deep, o));
  const int on = mode == 1 ? gd.eig != 0
                            : (gd.regime == 1 && !gd.eig && n >= kMinN && n <= kMaxN && smax > 0.0 &&
                               deep < kRatio * kRatio * smax);
  if (lane == 0) {
    flag[c] = on;
    if (on) list[1 + atomicAdd(&list[0], 1)] = cand[c];
  }
}

// ---- theta64: the contraction in FP64 (64 x 64 tile of X over TA = 64/D left indices a and
// TC = 64/D right indices c for all (s', t'); gate mix + lambda in the epilogue; FP32 inputs are
// exact in FP64, products and sums in FP64) ------------------------------------------------------
constexpr int KC = 16;
constexpr size_t kThetaSmem = (size_t)64 * 65 * sizeof(double2);

template <int D, int MINB>
__global__ void __launch_bounds__(256, MINB) k_rlg_theta(const GateDesc* __restrict__ desc, const int32_t* __restrict__ cand,
                                                   const int32_t* __restrict__ flag, uint8_t* slab, const DevState* st,
                                                   const float2* __restrict__ us) {
  constexpr int TA = 64 / D, TC = 64 / D;
  if (!flag[blockIdx.y]) return;
  const GateDesc gd = desc[cand[blockIdx.y]];
  const int l = gd.l, mid = gd.mid, r = gd.r, m = gd.m;
  const int ntc = (r + TC - 1) / TC, nta = (l + TA - 1) / TA;
  if ((int)blockIdx.x >= nta * ntc) return;
  const int a0 = (blockIdx.x / ntc) * TA, c0 = (blockIdx.x % ntc) * TC;
  extern __shared__ __align__(16) uint8_t sm[];
  double2(*As)[65] = reinterpret_cast<double2(*)[65]>(sm);              // stage s: rows 2 KC s ..
  double2(*Bs)[65] = reinterpret_cast<double2(*)[65]>(sm) + KC;         // stage s: rows 2 KC s + KC ..
  double2(*Cs)[65] = reinterpret_cast<double2(*)[65]>(sm);              // [64][65] (epilogue)
  __shared__ double2 Us[D * D * D * D];
  const SiteEntry* sites = reinterpret_cast<const SiteEntry*>(slab + st->sites_off);
  const BondEntry* bonds = reinterpret_cast<const BondEntry*>(slab + st->bonds_off);
  const float2* __restrict__ Bi = reinterpret_cast<const float2*>(slab + sites[gd.site].off);
  const float2* __restrict__ Bj = reinterpret_cast<const float2*>(slab + sites[gd.site + 1].off);
  const float* __restrict__ lam = reinterpret_cast<const float*>(slab + bonds[gd.site].off);
  double2* __restrict__ th = reinterpret_cast<double2*>(slab + rlg_layout(gd).th);
  const int tid = threadIdx.x;
  for (int x = tid; x < D * D * D * D; x += 256) {
    const float2 u = us[(int64_t)gd.u_index * D * D * D * D + x];
    Us[x] = make_double2(u.x, u.y);
  }
  const int ty = tid >> 4, tx = tid & 15;
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);
  // two shared-memory stages, the next chunk prefetched into registers during the current one's
  // products: one barrier per chunk, the global latency under the FP64 pipe
  float2 pa[4], pb[4];
  auto fetch = [&](int b0) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int e = tid + it * 256;
      const int kk = e & (KC - 1), rho = e >> 4;
      const int a = a0 + rho / D, sp = rho % D, b = b0 + kk;
      pa[it] = (a < l && b < mid) ? Bi[((int64_t)a * D + sp) * mid + b] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int e = tid + it * 256;
      const int cc = e % TC, rest = e / TC;
      const int tp = rest % D, kk = rest / D;
      const int c = c0 + cc, b = b0 + kk;
      pb[it] = (c < r && b < mid) ? Bj[((int64_t)b * D + tp) * r + c] : make_float2(0.f, 0.f);
    }
  };
  auto stash = [&](int stg) {
    double2(*Ad)[65] = As + stg * 2 * KC;
    double2(*Bd)[65] = Bs + stg * 2 * KC;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int e = tid + it * 256;
      Ad[e & (KC - 1)][e >> 4] = make_double2(pa[it].x, pa[it].y);
      const int cc = e % TC, rest = e / TC;
      Bd[rest / D][(rest % D) * TC + cc] = make_double2(pb[it].x, pb[it].y);
    }
  };
  const int nch = (mid + KC - 1) / KC;
  fetch(0);
  stash(0);
  __syncthreads();
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) fetch((ch + 1) * KC);
    double2(*Ad)[65] = As + (ch & 1) * 2 * KC;
    double2(*Bd)[65] = Bs + (ch & 1) * 2 * KC;
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      double2 av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = Ad[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bd[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j].x = fma(av[i].x, bv[j].x, fma(-av[i].y, bv[j].y, acc[i][j].x));
          acc[i][j].y = fma(av[i].x, bv[j].y, fma(av[i].y, bv[j].x, acc[i][j].y));
        }
    }
    if (ch + 1 < nch) stash((ch + 1) & 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) Cs[ty + 16 * i][tx + 16 * j] = acc[i][j];
  __syncthreads();
  for (int p = tid; p < TA * TC; p += 256) {
    const int al = p % TA, cl = p / TA;
    const int a = a0 + al, c = c0 + cl;
    if (a >= l || c >= r) continue;
    const double la = lam[a];
#pragma unroll
    for (int s = 0; s < D; ++s)
#pragma unroll
      for (int t = 0; t < D; ++t) {
        double2 o = make_double2(0.0, 0.0);
#pragma unroll
        for (int sp = 0; sp < D; ++sp)
#pragma unroll
          for (int tp = 0; tp < D; ++tp) {
            const double2 u = Us[(s * D + t) * D * D + sp * D + tp];
            const double2 cv = Cs[al * D + sp][tp * TC + cl];
            o.x = fma(u.x, cv.x, fma(-u.y, cv.y, o.x));
            o.y = fma(u.x, cv.y, fma(u.y, cv.x, o.y));
          }
        th[(int64_t)(t * r + c) * m + (a * D + s)] = make_double2(la * o.x, la * o.y);
      }
  }
}

// EAMPS_THETA_MINB2=1: two CTAs per SM (128 registers, a few spills in the prologue) instead of one
// (138 registers, no spills) -- A/B switch
void launch_theta64(int d, int max_tiles, int nc, const GateDesc* d_desc, const int32_t* d_cand, const int32_t* flag,
                    uint8_t* slab, const DevState* st, const float2* d_us, cudaStream_t s) {
  static const bool one = getenv("EAMPS_THETA_MINB2") == nullptr;
  const dim3 g(max_tiles, nc);
  if (d == 2) {
    if (one) k_rlg_theta<2, 1><<<g, 256, kThetaSmem, s>>>(d_desc, d_cand, flag, slab, st, d_us);
    else k_rlg_theta<2, 2><<<g, 256, kThetaSmem, s>>>(d_desc, d_cand, flag, slab, st, d_us);
  } else {
    if (one) k_rlg_theta<4, 1><<<g, 256, kThetaSmem, s>>>(d_desc, d_cand, flag, slab, st, d_us);
    else k_rlg_theta<4, 2><<<g, 256, kThetaSmem, s>>>(d_desc, d_cand, flag, slab, st, d_us);
  }
}

// ---- G = theta64^H theta64: 64 x 64 tiles (bi <= bj), mirrored; K = m in chunks of KC ---------
__global__ void __launch_bounds__(256) k_rlg_gram(const GateDesc* __restrict__ desc, const int32_t* __restrict__ cand,
                                                  const int32_t* __restrict__ flag, uint8_t* slab) {
  if (!flag[blockIdx.y]) return;
  const GateDesc gd = desc[cand[blockIdx.y]];
  const int n = gd.n, m = gd.m, nt = (n + 63) / 64;
  int t = blockIdx.x, bi = 0;
  while (bi < nt && t >= nt - bi) { t -= nt - bi; ++bi; }
  if (bi >= nt) return;
  const int bj = bi + t;
  const RlgLayout L = rlg_layout(gd);
  const double2* __restrict__ th = reinterpret_cast<const double2*>(slab + L.th);
  double2* __restrict__ G = reinterpret_cast<double2*>(slab + L.g);
  extern __shared__ __align__(16) uint8_t sm[];
  double2(*As)[65] = reinterpret_cast<double2(*)[65]>(sm);
  double2(*Bs)[65] = reinterpret_cast<double2(*)[65]>(sm) + KC;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int i0 = bi * 64, j0 = bj * 64;
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);
  double2 pa[4], pb[4];
  auto fetch = [&](int r0) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int e = tid + it * 256;
      const int kk = e & (KC - 1), cc = e >> 4;
      const int row = r0 + kk;
      const int ci = i0 + cc, cj = j0 + cc;
      pa[it] = (row < m && ci < n) ? th[(int64_t)ci * m + row] : make_double2(0.0, 0.0);
      pb[it] = (row < m && cj < n) ? th[(int64_t)cj * m + row] : make_double2(0.0, 0.0);
    }
  };
  auto stash = [&](int stg) {
    double2(*Ad)[65] = As + stg * 2 * KC;
    double2(*Bd)[65] = Bs + stg * 2 * KC;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int e = tid + it * 256;
      Ad[e & (KC - 1)][e >> 4] = pa[it];
      Bd[e & (KC - 1)][e >> 4] = pb[it];
    }
  };
  const int nch = (m + KC - 1) / KC;
  fetch(0);
  stash(0);
  __syncthreads();
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) fetch((ch + 1) * KC);
    double2(*Ad)[65] = As + (ch & 1) * 2 * KC;
    double2(*Bd)[65] = Bs + (ch & 1) * 2 * KC;
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      double2 av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = Ad[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bd[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {   // conj(a) b
          acc[i][j].x = fma(av[i].x, bv[j].x, fma(av[i].y, bv[j].y, acc[i][j].x));
          acc[i][j].y = fma(av[i].x, bv[j].y, fma(-av[i].y, bv[j].x, acc[i][j].y));
        }
    }
    if (ch + 1 < nch) stash((ch + 1) & 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gi = i0 + ty + 16 * i, gj = j0 + tx + 16 * j;   // G[gi][gj]
      if (gi >= n || gj >= n) continue;
      // lower tile storage: an entry is stored where its tile is lower or diagonal; the mirror
      // G[gj][gi] = conj(G[gi][gj]) covers the other half
      if (gi / TB >= gj / TB) G[g_at(gi, gj)] = acc[i][j];
      if (gj / TB >= gi / TB) G[g_at(gj, gi)] = make_double2(acc[i][j].x, -acc[i][j].y);
    }
}

// ---- Householder tridiagonalisation (cooperative grid, one gate at a time) ---------------------
// Monotone arrival counter of a CTA group: barrier number b completes when the counter reaches
// b * members.
__device__ __forceinline__ void rlg_barrier(unsigned int* ctr, unsigned int& nb, int members) {
  __syncthreads();
  ++nb;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    const unsigned int target = nb * (unsigned int)members;
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (v < target) __nanosleep(20);
    } while (v < target);
  }
  __syncthreads();
}

// CTA-wide sum of one double2 per thread (deterministic order; identical in every CTA).
__device__ __forceinline__ double2 cta_sum2(double2 v, double2* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
  for (int i = 0; i < nw; ++i) {
    s.x += red[i].x;
    s.y += red[i].y;
  }
  return s;
}

// CTA-wide sum of one double per thread (deterministic order; identical in every CTA).
__device__ __forceinline__ double cta_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];
  return s;
}

size_t tridiag_smem(int n) { return (size_t)3 * n * sizeof(double2) + 64 * sizeof(double) + 64; }

// The grid is split into groups of cpg CTAs; group g factorises the listed gates g, g + ngrp, ...
// (several gates in flight when the wave has several; all CTAs on one gate when it has one).
// G is the lower triangle in 32 x 32 tiles (g_at). Step k (trailing indices >= k1 = k + 1):
//  (A) every CTA reads column k below the diagonal (x = G[k1:, k]) with the update of step k-1 applied
//      and builds v_k, tau_k, beta_k;
//  (B) the warps stream the trailing lower tiles once: apply the update of step k-1, store, and emit the
//      tile's row partials (G_IJ v_J) and column partials (G_IJ^H v_I, off-diagonal tiles);
//  barrier; (C) p_i = tau (sum of the partials of row block I), partial dots p^H v; v_k kept in
//  column k (dead from now on); barrier; (D) w = p + alpha v, alpha = -tau (p^H v) / 2.
// Half the bytes of full storage per step (each trailing entry read and written once) for one more
// barrier.
__global__ void __launch_bounds__(TT, 1) k_rlg_tridiag(const GateDesc* __restrict__ desc,
                                                       const int32_t* __restrict__ list, uint8_t* slab,
                                                       unsigned int* ctr_base, int cpg) {
  const int cnt = list[0];
  const int grp = blockIdx.x / cpg, lcta = blockIdx.x % cpg, ngrp = gridDim.x / cpg;
  if (grp >= ngrp) return;
  unsigned int* ctr = ctr_base + 32 * grp;   // one 128-byte line per group
  extern __shared__ __align__(16) uint8_t sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gw = lcta * (TT / 32) + warp, W = cpg * (TT / 32);
  unsigned int nb = 0;
  for (int li = grp; li < cnt; li += ngrp) {
    const GateDesc& gd = desc[list[1 + li]];
    const int n = gd.n, nt = (n + TB - 1) / TB;
    const RlgLayout L = rlg_layout(gd);
    double2* A = reinterpret_cast<double2*>(slab + L.g);
    double* dg = reinterpret_cast<double*>(slab + L.d);
    double* eg = reinterpret_cast<double*>(slab + L.e);
    double2* pg = reinterpret_cast<double2*>(slab + L.p);
    double2* partg = reinterpret_cast<double2*>(slab + L.part);
    double2* taug = reinterpret_cast<double2*>(slab + L.tau);
    double2* rsg = reinterpret_cast<double2*>(slab + L.rs);
    double2* csg = reinterpret_cast<double2*>(slab + L.cs);
    double2* vbuf0 = reinterpret_cast<double2*>(sm);
    double2* vbuf1 = vbuf0 + n;
    double2* w = vbuf0 + 2 * n;                                         // w of step k-1
    double* red = reinterpret_cast<double*>(w + n);                     // 32 doubles (16 double2)
    double2* sc = reinterpret_cast<double2*>(red + 32);                 // [0] alpha
    for (int k = 0; k < n - 1; ++k) {
      double2* v = (k & 1) ? vbuf1 : vbuf0;
      const double2* vp = (k & 1) ? vbuf0 : vbuf1;   // v of step k-1 (valid from k = 1)
      const bool upd = k > 0;
      const int k1 = k + 1;
      // (A) column k, rows k .. n-1, with the update of step k-1 (never stored)
      double part = 0.0, dk = 0.0;
      for (int i = k + tid; i < n; i += TT) {
        double2 a = __ldcg(&A[g_at(i, k)]);
        if (upd) {   // a -= v_i conj(w_k) + w_i conj(v_k)
          const double2 t1 = cmulc(w[k], vp[i]);
          const double2 t2 = cmulc(vp[k], w[i]);
          a.x -= t1.x + t2.x;
          a.y -= t1.y + t2.y;
        }
        if (i == k) {
          dk = a.x;
        } else {
          v[i] = a;                                   // x_i = G[i][k]
          if (i >= k + 2) part += a.x * a.x + a.y * a.y;
        }
      }
      const double xn2 = cta_sum(part, red);          // includes a __syncthreads: v[] complete
      if (lcta == 0 && tid == 0) dg[k] = dk;          // i == k is thread 0's
      const double2 al = v[k1];
      double2 tau;
      double beta;
      double2 scale = make_double2(0.0, 0.0);
      if (xn2 == 0.0 && al.y == 0.0) {
        tau = make_double2(0.0, 0.0);
        beta = al.x;
      } else {
        beta = -copysign(sqrt(al.x * al.x + al.y * al.y + xn2), al.x);
        tau = make_double2((beta - al.x) / beta, -al.y / beta);
        const double2 den = make_double2(al.x - beta, al.y);           // 1 / (alpha - beta)
        const double dd = den.x * den.x + den.y * den.y;
        scale = make_double2(den.x / dd, -den.y / dd);
      }
      if (lcta == 0 && tid == 0) eg[k] = beta;
      __syncthreads();   // every thread has read v[k1]
      for (int i = k + 2 + tid; i < n; i += TT) v[i] = cmul(v[i], scale);
      if (tid == 0) v[k1] = make_double2(1.0, 0.0);
      __syncthreads();
      // (B) trailing lower tiles (I >= J >= J0): apply update k-1, store, row / column partials
      const int J0 = k1 / TB, m = nt - J0, ntile = m * (m + 1) / 2;
      for (int q = gw; q < ntile; q += W) {
        int I = 0, rem = q;                          // q -> (I, J), J0 <= J <= I, row-major over I
        {
          int ii = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
          while ((ii + 1) * (ii + 2) / 2 <= q) ++ii;
          while (ii * (ii + 1) / 2 > q) --ii;
          I = ii;
          rem = q - ii * (ii + 1) / 2;
        }
        const int J = J0 + rem, Ib = J0 + I;
        const int j = J * TB + lane;
        const bool jv = j >= k1 && j < n;
        const double2 vj = jv ? v[j] : make_double2(0.0, 0.0);
        const double2 vpj = (upd && jv) ? vp[j] : make_double2(0.0, 0.0);
        const double2 wj = (upd && jv) ? w[j] : make_double2(0.0, 0.0);
        double2* T = A + ((int64_t)Ib * (Ib + 1) / 2 + J) * (TB * TB);
        double2 colacc = make_double2(0.0, 0.0);
        const int64_t toff = ((int64_t)Ib * (Ib + 1) / 2 + J) * TB;
#pragma unroll 1
        for (int c = 0; c < TB / 8; ++c) {
          double2 pr[8];
          double2 a[8];
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) {
            const int i = Ib * TB + 8 * c + rr;
            a[rr] = (jv && i >= k1 && i < n) ? __ldcg(&T[(8 * c + rr) * TB + lane]) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int rr = 0; rr < 8; ++rr) {
            const int i = Ib * TB + 8 * c + rr;
            const bool iv = i >= k1 && i < n;
            if (jv && iv) {
              if (upd) {   // a -= v_i conj(w_j) + w_i conj(v_j)
                const double2 t1 = cmulc(wj, vp[i]);
                const double2 t2 = cmulc(vpj, w[i]);
                a[rr].x -= t1.x + t2.x;
                a[rr].y -= t1.y + t2.y;
                __stcg(&T[(8 * c + rr) * TB + lane], a[rr]);
              }
              if (Ib != J) {   // column partial: conj(a) v_i
                const double2 cv = cmulc(a[rr], v[i]);
                colacc.x += cv.x;
                colacc.y += cv.y;
              }
            }
            pr[rr] = cmul(a[rr], vj);     // 0 where masked
          }
          // transpose-reduce the 8 row products over the 32 lanes: lane ends with the sum of row
          // 4 b4 + 2 b3 + b2 (b_x = bit x of the lane), complete after the xor-2 / xor-1 steps
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const bool hi = lane & 16;
            const double2 keep = hi ? pr[q4 + 4] : pr[q4], send = hi ? pr[q4] : pr[q4 + 4];
            pr[q4].x = keep.x + __shfl_xor_sync(0xffffffffu, send.x, 16);
            pr[q4].y = keep.y + __shfl_xor_sync(0xffffffffu, send.y, 16);
          }
#pragma unroll
          for (int q2 = 0; q2 < 2; ++q2) {
            const bool hi = lane & 8;
            const double2 keep = hi ? pr[q2 + 2] : pr[q2], send = hi ? pr[q2] : pr[q2 + 2];
            pr[q2].x = keep.x + __shfl_xor_sync(0xffffffffu, send.x, 8);
            pr[q2].y = keep.y + __shfl_xor_sync(0xffffffffu, send.y, 8);
          }
          {
            const bool hi = lane & 4;
            const double2 keep = hi ? pr[1] : pr[0], send = hi ? pr[0] : pr[1];
            pr[0].x = keep.x + __shfl_xor_sync(0xffffffffu, send.x, 4);
            pr[0].y = keep.y + __shfl_xor_sync(0xffffffffu, send.y, 4);
          }
          pr[0].x += __shfl_xor_sync(0xffffffffu, pr[0].x, 2);
          pr[0].y += __shfl_xor_sync(0xffffffffu, pr[0].y, 2);
          pr[0].x += __shfl_xor_sync(0xffffffffu, pr[0].x, 1);
          pr[0].y += __shfl_xor_sync(0xffffffffu, pr[0].y, 1);
          if ((lane & 3) == 0) {
            const int r = 4 * ((lane >> 4) & 1) + 2 * ((lane >> 3) & 1) + ((lane >> 2) & 1);
            __stcg(&rsg[toff + 8 * c + r], pr[0]);
          }
        }
        if (Ib != J) __stcg(&csg[toff + lane], colacc);
      }
      rlg_barrier(ctr, nb, cpg);
      // (C) p_i = tau (sum_J rows(I, J) + sum_{I' > I} cols(I', I)); partial dots conj(p_i) v_i
      double2 pdot = make_double2(0.0, 0.0);
      for (int Ib = J0 + gw; Ib < nt; Ib += W) {
        const int i = Ib * TB + lane;
        // up to 2 nt partials per lane: 8 independent loads in flight (a dependent chain of L2 round
        // trips here cost ~20 us per step when one gate has the whole grid: ncu, barrier-stalled)
        double2 sacc = make_double2(0.0, 0.0);
        const int nr = Ib - J0 + 1, ncol = nt - 1 - Ib;
        for (int q0 = 0; q0 < nr + ncol; q0 += 8) {
          double2 t[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int q = q0 + u;
            t[u] = q < nr ? __ldcg(&rsg[((int64_t)Ib * (Ib + 1) / 2 + J0 + q) * TB + lane])
                 : q < nr + ncol ? __ldcg(&csg[((int64_t)(Ib + 1 + q - nr) * (Ib + 2 + q - nr) / 2 + Ib) * TB + lane])
                                 : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            sacc.x += t[u].x;
            sacc.y += t[u].y;
          }
        }
        if (i >= k1 && i < n) {
          const double2 p = cmul(tau, sacc);
          __stcg(&pg[(int64_t)(k & 1) * n + i], p);
          const double2 cp = cmulc(p, v[i]);
          pdot.x += cp.x;
          pdot.y += cp.y;
        }
      }
      // the reflector H_k = I - tau_k v_k v_k^H is kept for the eigenvectors (z = H_0 .. H_{n-2} y):
      // v_k in column k (dead from now on; every CTA read it in (A) before the barrier), tau_k in taug
      if (lcta == 0) {
        for (int i = k1 + tid; i < n; i += TT) __stcg(&A[g_at(i, k)], v[i]);
        if (tid == 0) taug[k] = tau;
      }
      const double2 dsum = cta_sum2(pdot, reinterpret_cast<double2*>(red));
      if (tid == 0) __stcg(&partg[(k & 1) * 1024 + lcta], dsum);
      rlg_barrier(ctr, nb, cpg);
      // (D) w = p + alpha v, alpha = -1/2 tau (p^H v) (zhetd2; p already carries tau). The group's
      // partials summed by warp 0 in a fixed order (identical in every CTA of the group)
      if (warp == 0) {
        double2 s = make_double2(0.0, 0.0);
        for (int c = lane; c < cpg; c += 32) {
          const double2 q = __ldcg(&partg[(k & 1) * 1024 + c]);
          s.x += q.x;
          s.y += q.y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
          s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
        }
        const double2 t = cmul(tau, s);
        if (lane == 0) sc[0] = make_double2(-0.5 * t.x, -0.5 * t.y);
      }
      __syncthreads();
      const double2 alpha = sc[0];
      for (int j = k1 + tid; j < n; j += TT) {
        const double2 p = __ldcg(&pg[(int64_t)(k & 1) * n + j]);
        const double2 av = cmul(alpha, v[j]);
        w[j] = make_double2(p.x + av.x, p.y + av.y);
      }
      __syncthreads();
    }
    // the last diagonal entry: G[n-1][n-1] with the update of step n-2
    if (lcta == 0 && tid == 0) {
      double2 a = __ldcg(&A[g_at(n - 1, n - 1)]);
      if (n >= 2) {
        const double2* vl = ((n - 2) & 1) ? vbuf1 : vbuf0;
        const double2 t1 = cmulc(w[n - 1], vl[n - 1]);
        const double2 t2 = cmulc(vl[n - 1], w[n - 1]);
        a.x -= t1.x + t2.x;
      }
      dg[n - 1] = a.x;
    }
    rlg_barrier(ctr, nb, cpg);   // the next gate reuses the shared buffers and the partials
  }
}

// ---- eigenvalues of the symmetric tridiagonal (d, e) by Sturm-count multisection ---------------
// count(x) = #{eigenvalues < x} = #{negative pivots of T - x I = L D L^T}. A group of 8 lanes per
// eigenvalue index j; each lane runs the Sturm recurrences of 2 of the 16 interior points of the
// bracket (two independent chains), so a pass narrows [lo, hi) 17-fold; the bracket is identical
// in the 8 lanes (same inputs, same arithmetic).
// LPE = lanes per eigenvalue (8: a latency-bound launch with few eigenvalues; 1: a throughput-bound
// one -- plain trisection with 2 points per thread does 4x less Sturm work per digit than the 17-way
// multisection).
template <int LPE>
__global__ void __launch_bounds__(BT) k_rlg_bisect(const GateDesc* __restrict__ desc, const int32_t* __restrict__ cand,
                                                   const int32_t* __restrict__ flag, uint8_t* slab) {
  constexpr int kBisPerCta = BT / LPE;   // eigenvalues per CTA
  constexpr int NP = 2 * LPE;             // points per pass
  if (!flag[blockIdx.y]) return;
  const GateDesc gd = desc[cand[blockIdx.y]];
  const int n = gd.n;
  if ((int)blockIdx.x * kBisPerCta >= n) return;
  const RlgLayout L = rlg_layout(gd);
  const double* dg = reinterpret_cast<const double*>(slab + L.d);
  const double* eg = reinterpret_cast<const double*>(slab + L.e);
  double* eig = reinterpret_cast<double*>(slab + L.eig);
  extern __shared__ __align__(16) uint8_t bis_sm[];
  double* ds = reinterpret_cast<double*>(bis_sm);     // n
  double* e2s = ds + n;                               // n
  __shared__ double red[3][BT / 32];
  double lo = 1e300, hi = -1e300, emax = 0.0;
  for (int i = threadIdx.x; i < n; i += BT) {
    const double di = dg[i], el = i > 0 ? fabs(eg[i - 1]) : 0.0, er = i < n - 1 ? fabs(eg[i]) : 0.0;
    ds[i] = di;
    e2s[i] = er * er;
    lo = fmin(lo, di - el - er);   // Gershgorin
    hi = fmax(hi, di + el + er);
    emax = fmax(emax, er * er);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = lo;
    red[1][threadIdx.x >> 5] = hi;
    red[2][threadIdx.x >> 5] = emax;
  }
  __syncthreads();
  for (int i = 0; i < BT / 32; ++i) {
    lo = fmin(lo, red[0][i]);
    hi = fmax(hi, red[1][i]);
    emax = fmax(emax, red[2][i]);
  }
  const double span = fmax(fabs(lo), fabs(hi));
  lo -= 2.0 * 2.2e-16 * span * n + 1e-300;
  hi += 2.0 * 2.2e-16 * span * n + 1e-300;
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax);
  const int lane = threadIdx.x & 31, sub = lane & (LPE - 1);
  const int j = blockIdx.x * kBisPerCta + threadIdx.x / LPE;
  const bool act = j < n;
  // invariant: count(lo) <= j < count(hi)
  for (int it = 0; it < (LPE == 8 ? 18 : 48); ++it) {   // 17^18 > 2^73, 3^48 > 2^76
    const double wdt = hi - lo;
    if (__all_sync(0xffffffffu, wdt <= 2.2e-16 * fmax(fabs(lo), fabs(hi)) + 1e-300)) break;   // warp-uniform
    const double x1 = lo + wdt * (2 * sub + 1) / (double)(NP + 1), x2 = lo + wdt * (2 * sub + 2) / (double)(NP + 1);
    double q1 = ds[0] - x1, q2 = ds[0] - x2;
    int c1 = q1 < 0.0, c2 = q2 < 0.0;
    for (int i = 1; i < n; ++i) {
      const double e2 = e2s[i - 1], di = ds[i];
      if (fabs(q1) < pivmin) q1 = -pivmin;
      if (fabs(q2) < pivmin) q2 = -pivmin;
      q1 = (di - x1) - e2 / q1;
      q2 = (di - x2) - e2 / q2;
      c1 += q1 < 0.0;
      c2 += q2 < 0.0;
    }
    // bit p of mask: count(x_p) > j (monotone in p); OR over the LPE lanes of the group
    unsigned int mask = ((act && c1 > j) ? 1u : 0u) << (2 * sub) | ((act && c2 > j) ? 2u : 0u) << (2 * sub);
#pragma unroll
    for (int o = 1; o < LPE; o <<= 1) mask |= __shfl_xor_sync(0xffffffffu, mask, o);
    const int p = mask ? __ffs(mask) - 1 : NP;    // first point with count > j
    const double nlo = p == 0 ? lo : lo + wdt * p / (double)(NP + 1);
    const double nhi = p == NP ? hi : lo + wdt * (p + 1) / (double)(NP + 1);
    lo = nlo;
    hi = nhi;
  }
  if (act && sub == 0) eig[j] = 0.5 * (lo + hi);   // ascending
}

// ---- sigma^2 (descending) + tails; mode 1 (eigen route): pi = identity (column j of V will be the
// eigenvector of the j-th largest eigenvalue) and the depth check: a spectrum reaching below
// kEigMin sigma_max (sigma >= 1e-6 sigma_max) leaves the eigen route (desc.eig = 0, fb[c] = 1) for the
// Jacobi route + refinements, whose relative accuracy does not degrade as 1 / sigma^2 -------------
constexpr double kEigMin = 3e-6;
__global__ void __launch_bounds__(256) k_rlg_finish(GateDesc* __restrict__ desc, const int32_t* __restrict__ cand,
                                                    const int32_t* __restrict__ flag, uint8_t* slab, int mode,
                                                    int32_t* fb) {
  if (!flag[blockIdx.x]) {
    if (mode == 1 && threadIdx.x == 0) fb[blockIdx.x] = 0;
    return;
  }
  GateDesc& gdr = desc[cand[blockIdx.x]];
  const GateDesc gd = gdr;
  const int n = gd.n;
  const RlgLayout L = rlg_layout(gd);
  const double* eig = reinterpret_cast<const double*>(slab + L.eig);
  __shared__ double keys[kMaxN];
  __shared__ double part[256];
  __shared__ int s_deep;
  double* gS = reinterpret_cast<double*>(slab + gd.ws_sig2);
  int32_t* gP = reinterpret_cast<int32_t*>(slab + gd.ws_pi);
  if (threadIdx.x == 0) s_deep = 0;
  __syncthreads();
  const double smax = fmax(eig[n - 1], 0.0);
  for (int j = threadIdx.x; j < n; j += 256) {
    const double v = fmax(eig[n - 1 - j], 0.0);
    keys[j] = v;
    gS[j] = v;
    if (mode == 1) {
      gP[j] = j;
      if (v >= 1e-12 * smax && v < kEigMin * kEigMin * smax) s_deep = 1;
    }
  }
  __syncthreads();
  cta_tails(keys, n, reinterpret_cast<double*>(slab + gd.ws_T), part);
  if (mode == 1 && threadIdx.x == 0) {
    fb[blockIdx.x] = s_deep;
    if (s_deep) gdr.eig = 0;
    gdr.sweeps = 0;
  }
}

// ---- eigenvectors of T for the kept columns (eigen route, after the select: k = desc.k) ----------
// Inverse iteration: T - lambda_j I = P L U (Gaussian elimination with partial pivoting, LAPACK
// dgttrf), two solves from a fixed pseudo-random start, unit 2-norm. lambda_j is the bisection value
// (accurate to a few ulps of ||T||), so y_j is accurate to ~eps64 ||T|| / gap_j in angle. One thread
// per vector, kSlots factor slots per gate; row j of Y = y_j.
__global__ void __launch_bounds__(32) k_rlg_invit(const GateDesc* __restrict__ desc, const int32_t* __restrict__ cand,
                                                  uint8_t* slab, int want) {
  const GateDesc& gd = desc[cand[blockIdx.y]];
  if (gd.eig != want) return;
  const int n = gd.n, k = gd.k;
  const int slot = blockIdx.x * 32 + threadIdx.x;
  if (slot >= k) return;
  const RlgLayout L = rlg_layout(gd);
  const double* __restrict__ dg = reinterpret_cast<const double*>(slab + L.d);
  const double* __restrict__ eg = reinterpret_cast<const double*>(slab + L.e);
  const double* __restrict__ eig = reinterpret_cast<const double*>(slab + L.eig);
  double4* F = reinterpret_cast<double4*>(slab + L.slot) + (int64_t)slot * n;     // (dl, d, du, du2)
  uint8_t* piv = reinterpret_cast<uint8_t*>(slab + L.slot + (int64_t)kSlots * n * 32) + (int64_t)slot * n;
  double tnorm = 0.0;
  for (int i = 0; i < n; ++i)
    tnorm = fmax(tnorm, fabs(dg[i]) + (i > 0 ? fabs(eg[i - 1]) : 0.0) + (i < n - 1 ? fabs(eg[i]) : 0.0));
  const double tiny = fmax(tnorm, 1e-300) * 2.220446049250313e-16;
  for (int j = slot; j < k; j += kSlots) {
    const double lam = eig[n - 1 - j];
    double* y = reinterpret_cast<double*>(slab + L.y) + (int64_t)j * n;
    // factor (dgttrf)
    double dcur = dg[0] - lam, ducur = n > 1 ? eg[0] : 0.0;
    for (int i = 0; i < n - 1; ++i) {
      const double dl = eg[i], dn = dg[i + 1] - lam, dun = i + 1 < n - 1 ? eg[i + 1] : 0.0;
      double4 f;
      if (fabs(dcur) >= fabs(dl)) {
        const double d0 = dcur != 0.0 ? dcur : tiny;
        const double fact = dl / d0;
        f = make_double4(fact, d0, ducur, 0.0);
        piv[i] = 0;
        dcur = dn - fact * ducur;
        ducur = dun;
      } else {
        const double fact = dcur / dl;
        f = make_double4(fact, dl, dn, dun);        // row swap: U row i = (dl, dn, dun)
        piv[i] = 1;
        dcur = ducur - fact * dn;
        ducur = -fact * dun;
      }
      F[i] = f;
    }
    F[n - 1] = make_double4(0.0, dcur != 0.0 ? (fabs(dcur) < tiny ? copysign(tiny, dcur) : dcur) : tiny, 0.0, 0.0);
    for (int i = 0; i < n - 1; ++i)   // tiny pivots: perturb (the vector direction is what matters)
      if (fabs(F[i].y) < tiny) F[i].y = copysign(tiny, F[i].y);
    // start vector: fixed pseudo-random in [0.5, 1.5)
    for (int i = 0; i < n; ++i) {
      unsigned int h = (unsigned int)i * 2654435761u ^ ((unsigned int)j * 40503u + 0x9e3779b9u);
      h ^= h >> 15;
      h *= 2246822519u;
      h ^= h >> 13;
      y[i] = 0.5 + (double)(h & 0xffffu) / 65536.0;
    }
    for (int it = 0; it < 2; ++it) {
      // L: forward with the row interchanges
      for (int i = 0; i < n - 1; ++i) {
        const double fact = F[i].x;
        if (piv[i] == 0) {
          y[i + 1] -= fact * y[i];
        } else {
          const double t = y[i];
          y[i] = y[i + 1];
          y[i + 1] = t - fact * y[i];
        }
      }
      // U: back substitution (diag d, super du, second super du2)
      double nrm = 0.0;
      for (int i = n - 1; i >= 0; --i) {
        const double4 f = F[i];
        double v = y[i];
        if (i + 1 < n) v -= f.z * y[i + 1];
        if (i + 2 < n) v -= f.w * y[i + 2];
        v /= f.y;
        y[i] = v;
        nrm = fma(v, v, nrm);
      }
      const double sc = 1.0 / sqrt(nrm);
      for (int i = 0; i < n; ++i) y[i] *= sc;
    }
  }
}

// Clusters of (numerically) degenerate eigenvalues among the kept ones: inverse iteration from
// different starts returns independent vectors of the cluster's invariant subspace; modified
// Gram-Schmidt makes them orthonormal. One CTA per gate (most gates have no cluster).
__global__ void __launch_bounds__(256) k_rlg_mgs(const GateDesc* __restrict__ desc, const int32_t* __restrict__ cand,
                                                 uint8_t* slab, int want) {
  const GateDesc& gd = desc[cand[blockIdx.x]];
  if (gd.eig != want) return;
  const int n = gd.n, k = gd.k;
  const RlgLayout L = rlg_layout(gd);
  const double* gS = reinterpret_cast<const double*>(slab + gd.ws_sig2);
  double* Y = reinterpret_cast<double*>(slab + L.y);
  __shared__ double red[8];
  const double gap = 1e-9 * gS[0];
  int c0 = 0;
  for (int j = 1; j < k; ++j) {
    if (gS[j - 1] - gS[j] > gap) {
      c0 = j;
      continue;
    }
    double* yj = Y + (int64_t)j * n;
    for (int l = c0; l < j; ++l) {
      const double* yl = Y + (int64_t)l * n;
      double s = 0.0;
      for (int i = threadIdx.x; i < n; i += 256) s = fma(yl[i], yj[i], s);
      const double dot = cta_sum(s, red);
      for (int i = threadIdx.x; i < n; i += 256) yj[i] -= dot * yl[i];
      __syncthreads();
    }
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += 256) s = fma(yj[i], yj[i], s);
    const double sc = 1.0 / sqrt(cta_sum(s, red));
    for (int i = threadIdx.x; i < n; i += 256) yj[i] *= sc;
    __syncthreads();
  }
}

// Back-transformation z_j = Q y_j = H_0 (H_1 ( .. H_{n-2} y_j)), H_q = I - tau_q v_q v_q^H (v_q in
// column q of the factorised G, entries q+1 .. n-1), then V[:, j] = z_j in FP32 (unit norm: Q unitary).
// kVpc vectors per CTA in shared memory; each thread owns the same rows of every vector, so only the
// dot products v_q^H z need the CTA (one barrier per reflector, double-buffered partials).
// VPC vectors per CTA, RPT rows per thread (n <= 256 RPT): (16, 2) for n <= 512, (8, 4) for n <= 1024,
// (4, 8) for n <= 2048 -- the shared-memory z stays <= 128 KB and each reflector's loads and barrier
// serve as many vectors as fit.
constexpr int kVpc = 4;   // the largest-n configuration (attribute sizing)
template <int VPC, int RPT>
__global__ void __launch_bounds__(256) k_rlg_backtr(const GateDesc* __restrict__ desc, const int32_t* __restrict__ cand,
                                                    uint8_t* slab, int want) {
  constexpr int kVpc = VPC;
  const GateDesc& gd = desc[cand[blockIdx.y]];
  if (gd.eig != want) return;
  const int n = gd.n, k = gd.k, np = gd.n_pad;
  const int j0 = blockIdx.x * kVpc;
  if (j0 >= k) return;
  const int nv = min(kVpc, k - j0);
  const RlgLayout L = rlg_layout(gd);
  const double2* __restrict__ A = reinterpret_cast<const double2*>(slab + L.g);
  const double2* __restrict__ taug = reinterpret_cast<const double2*>(slab + L.tau);
  const double* __restrict__ Y = reinterpret_cast<const double*>(slab + L.y);
  extern __shared__ __align__(16) uint8_t sm[];
  double2* z = reinterpret_cast<double2*>(sm);                     // [kVpc][n]
  __shared__ double2 red[2][8][kVpc];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int q = 0; q < kVpc; ++q)
    for (int i = tid; i < n; i += 256)
      z[q * n + i] = make_double2(q < nv ? Y[(int64_t)(j0 + q) * n + i] : 0.0, 0.0);
  // thread tid owns rows i = tid + 256 q (q < kRowsPT): the same rows of z for every r, so the update
  // and the next dot product need no barrier between them; reflector r-1's entries of those rows are
  // loaded while reflector r is applied (its L2 latency off the per-reflector critical path)
  constexpr int kRowsPT = RPT;
  double2 cur[kRowsPT], nxt[kRowsPT];
  auto load_col = [&](int r, double2* dst) {
#pragma unroll
    for (int q = 0; q < kRowsPT; ++q) {
      const int i = tid + 256 * q;
      dst[q] = (r >= 0 && i > r && i < n) ? __ldg(&A[g_at(i, r)]) : make_double2(0.0, 0.0);
    }
  };
  load_col(n - 2, cur);
  for (int r = n - 2; r >= 0; --r) {
    load_col(r - 1, nxt);
    double2 acc[kVpc];
#pragma unroll
    for (int q = 0; q < kVpc; ++q) acc[q] = make_double2(0.0, 0.0);
#pragma unroll
    for (int qq = 0; qq < kRowsPT; ++qq) {
      const int i = tid + 256 * qq;
      if (i <= r || i >= n) continue;
#pragma unroll
      for (int q = 0; q < kVpc; ++q) {
        const double2 c = cmulc(cur[qq], z[q * n + i]);
        acc[q].x += c.x;
        acc[q].y += c.y;
      }
    }
    // transpose-reduce the kVpc per-lane partials over the warp: halving stages (offsets 16, 8, ..)
    // leave lane L with vector q(L)'s sum over the lanes sharing its high bits, then a plain xor
    // reduction over the remaining low bits -- kVpc - 1 + 5 - log2(kVpc) shuffle-adds instead of 5 kVpc
    constexpr int S = kVpc >= 16 ? 4 : kVpc >= 8 ? 3 : kVpc >= 4 ? 2 : kVpc >= 2 ? 1 : 0;
#pragma unroll
    for (int st = 0; st < S; ++st) {
      const int o = 16 >> st, half = kVpc >> (st + 1);
      const bool hi = lane & o;
#pragma unroll
      for (int j = 0; j < (kVpc >> 1); ++j) {
        if (j >= half) break;
        const double2 keep = hi ? acc[j + half] : acc[j], send = hi ? acc[j] : acc[j + half];
        acc[j].x = keep.x + __shfl_xor_sync(0xffffffffu, send.x, o);
        acc[j].y = keep.y + __shfl_xor_sync(0xffffffffu, send.y, o);
      }
    }
#pragma unroll
    for (int o = 16 >> S; o >= 1; o >>= 1) {
      acc[0].x += __shfl_xor_sync(0xffffffffu, acc[0].x, o);
      acc[0].y += __shfl_xor_sync(0xffffffffu, acc[0].y, o);
    }
    const int b = r & 1;
    if ((lane & ((32 >> S) - 1)) == 0) {
      int qi = 0;
#pragma unroll
      for (int st = 0; st < S; ++st) qi = 2 * qi + ((lane >> (4 - st)) & 1);
      red[b][warp][qi] = acc[0];
    }
    __syncthreads();
    const double2 tau = taug[r];
    double2 f[kVpc];
#pragma unroll
    for (int q = 0; q < kVpc; ++q) {
      double2 sdot = make_double2(0.0, 0.0);
      for (int w = 0; w < 8; ++w) {
        sdot.x += red[b][w][q].x;
        sdot.y += red[b][w][q].y;
      }
      f[q] = cmul(tau, sdot);
    }
#pragma unroll
    for (int qq = 0; qq < kRowsPT; ++qq) {
      const int i = tid + 256 * qq;
      if (i <= r || i >= n) continue;
#pragma unroll
      for (int q = 0; q < kVpc; ++q) {
        const double2 t = cmul(f[q], cur[qq]);
        z[q * n + i].x -= t.x;
        z[q * n + i].y -= t.y;
      }
    }
#pragma unroll
    for (int qq = 0; qq < kRowsPT; ++qq) cur[qq] = nxt[qq];
  }
  __syncthreads();
  float2* V = reinterpret_cast<float2*>(slab + gd.ws_V);
  for (int q = 0; q < nv; ++q)
    for (int i = tid; i < np; i += 256) {
      const double2 v = i < n ? z[q * n + i] : make_double2(0.0, 0.0);
      V[(int64_t)(j0 + q) * np + i] = make_float2((float)v.x, (float)v.y);
    }
}

// ---- the eigen route for n <= 128 (QR-regime thetas, config 2 chi = 64): one CTA per gate, G in
// shared memory (packed lower triangle, 132 KB at n = 128). Same recurrences as k_rlg_tridiag /
// k_rlg_bisect / k_rlg_finish (zhetd2, Sturm counts), the reflectors stored to the gate's tile-layout G
// columns and tau array exactly as k_rlg_tridiag does, so k_rlg_invit / k_rlg_mgs / k_rlg_backtr serve
// both. Depth check: a spectrum reaching below kEigMinSmall sigma_max (sigma >= 1e-6 sigma_max) is
// flagged (desc.eig = 2, k = n): all its eigenvectors are computed before the select and the FP64
// Rayleigh-Ritz refinement (refine.cu, relative accuracy) replaces its sigma.
constexpr int kSmallMaxN = 128;
constexpr double kEigMinSmall = 2e-4;   // = refine.cu's trigger: deeper spectra get the relative-accurate RR
__host__ __device__ inline int pk_lo(int i, int j) { return i * (i + 1) / 2 + j; }   // j <= i
size_t eig_cta_smem(int n) {
  return (size_t)n * (n + 1) / 2 * 16 + (size_t)3 * n * 16 + (size_t)4 * n * 8 + 64 * 8 + 256 * 8 + 128;
}

__global__ void __launch_bounds__(256, 1) k_eig_cta(GateDesc* __restrict__ desc, const int32_t* __restrict__ cand,
                                                    uint8_t* slab, int32_t* fb) {
  GateDesc& gdr = desc[cand[blockIdx.x]];
  if (gdr.eig != 1) return;
  const GateDesc gd = gdr;
  const int n = gd.n;
  const RlgLayout L = rlg_layout(gd);
  double2* G = reinterpret_cast<double2*>(slab + L.g);
  double* dg = reinterpret_cast<double*>(slab + L.d);
  double* eg = reinterpret_cast<double*>(slab + L.e);
  double* eig = reinterpret_cast<double*>(slab + L.eig);
  double2* taug = reinterpret_cast<double2*>(slab + L.tau);
  extern __shared__ __align__(16) uint8_t sm[];
  double2* A = reinterpret_cast<double2*>(sm);                         // packed lower
  double2* v = A + n * (n + 1) / 2;
  double2* w = v + n;
  double2* p = w + n;
  double* ds = reinterpret_cast<double*>(p + n);
  double* e2 = ds + n;
  double* keys = e2 + n;                                               // 2 n doubles (sort-free: ascending -> desc)
  double* red = keys + 2 * n;                                          // 64
  double* part = red + 64;                                             // 256
  __shared__ double2 s_sc;
  __shared__ int s_deep;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = warp; i < n; i += 8)
    for (int j = lane; j <= i; j += 32) A[pk_lo(i, j)] = G[g_at(i, j)];
  __syncthreads();
  for (int k = 0; k < n - 1; ++k) {
    const int k1 = k + 1;
    double part2 = 0.0;
    for (int i = k1 + tid; i < n; i += 256) {
      const double2 x = A[pk_lo(i, k)];
      v[i] = x;
      if (i >= k + 2) part2 += x.x * x.x + x.y * x.y;
    }
    const double xn2 = cta_sum(part2, red);
    const double2 al = v[k1];
    double2 tau;
    double beta;
    double2 scale = make_double2(0.0, 0.0);
    if (xn2 == 0.0 && al.y == 0.0) {
      tau = make_double2(0.0, 0.0);
      beta = al.x;
    } else {
      beta = -copysign(sqrt(al.x * al.x + al.y * al.y + xn2), al.x);
      tau = make_double2((beta - al.x) / beta, -al.y / beta);
      const double2 den = make_double2(al.x - beta, al.y);
      const double dd = den.x * den.x + den.y * den.y;
      scale = make_double2(den.x / dd, -den.y / dd);
    }
    if (tid == 0) {
      ds[k] = A[pk_lo(k, k)].x;
      e2[k] = beta;          // beta for now (squared below)
      taug[k] = tau;
    }
    __syncthreads();
    for (int i = k + 2 + tid; i < n; i += 256) v[i] = cmul(v[i], scale);
    if (tid == 0) v[k1] = make_double2(1.0, 0.0);
    __syncthreads();
    // p = tau A22 v: two threads per row (even / odd j), A22 Hermitian from the packed lower triangle
    {
      const int i = k1 + (tid >> 1), h = tid & 1;
      double2 acc = make_double2(0.0, 0.0);
      if (i < n) {
        for (int j = k1 + h; j < n; j += 2) {
          const double2 a = j <= i ? A[pk_lo(i, j)] : make_double2(A[pk_lo(j, i)].x, -A[pk_lo(j, i)].y);
          const double2 vj = v[j];
          acc.x = fma(a.x, vj.x, fma(-a.y, vj.y, acc.x));
          acc.y = fma(a.x, vj.y, fma(a.y, vj.x, acc.y));
        }
      }
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
      if (i < n && h == 0) p[i] = cmul(tau, acc);
    }
    // the reflector for the back-transformation (column k of the tile-layout G, as k_rlg_tridiag)
    for (int i = k1 + tid; i < n; i += 256) G[g_at(i, k)] = v[i];
    __syncthreads();
    double2 pd = make_double2(0.0, 0.0);
    for (int i = k1 + tid; i < n; i += 256) {
      const double2 c = cmulc(p[i], v[i]);
      pd.x += c.x;
      pd.y += c.y;
    }
    const double2 dot = cta_sum2(pd, reinterpret_cast<double2*>(red));
    const double2 t = cmul(tau, dot);
    const double2 alpha = make_double2(-0.5 * t.x, -0.5 * t.y);
    for (int i = k1 + tid; i < n; i += 256) {
      const double2 av = cmul(alpha, v[i]);
      w[i] = make_double2(p[i].x + av.x, p[i].y + av.y);
    }
    __syncthreads();
    // A22 -= v w^H + w v^H (packed lower)
    for (int i = k1 + warp; i < n; i += 8) {
      const double2 vi = v[i], wi = w[i];
      for (int j = k1 + lane; j <= i; j += 32) {
        const double2 t1 = cmulc(w[j], vi), t2 = cmulc(v[j], wi);
        double2& a = A[pk_lo(i, j)];
        a.x -= t1.x + t2.x;
        a.y -= t1.y + t2.y;
      }
    }
    __syncthreads();
  }
  if (tid == 0) ds[n - 1] = A[pk_lo(n - 1, n - 1)].x;
  __syncthreads();
  // d, e to global (inverse iteration), e^2 for the Sturm counts
  for (int i = tid; i < n; i += 256) {
    dg[i] = ds[i];
    if (i < n - 1) {
      eg[i] = e2[i];
      e2[i] = e2[i] * e2[i];
    } else {
      e2[i] = 0.0;
    }
  }
  __syncthreads();
  // Gershgorin interval
  double lo = 1e300, hi = -1e300, emax = 0.0;
  for (int i = tid; i < n; i += 256) {
    const double el = i > 0 ? sqrt(e2[i - 1]) : 0.0, er = i < n - 1 ? sqrt(e2[i]) : 0.0;
    lo = fmin(lo, ds[i] - el - er);
    hi = fmax(hi, ds[i] + el + er);
    emax = fmax(emax, e2[i]);
  }
  {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      emax = fmax(emax, __shfl_xor_sync(0xffffffffu, emax, o));
    }
    __syncthreads();
    if (lane == 0) {
      red[warp] = lo;
      red[8 + warp] = hi;
      red[16 + warp] = emax;
    }
    __syncthreads();
    for (int q = 0; q < 8; ++q) {
      lo = fmin(lo, red[q]);
      hi = fmax(hi, red[8 + q]);
      emax = fmax(emax, red[16 + q]);
    }
  }
  const double span = fmax(fabs(lo), fabs(hi));
  lo -= 2.0 * 2.2e-16 * span * n + 1e-300;
  hi += 2.0 * 2.2e-16 * span * n + 1e-300;
  const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax);
  // 2 lanes per eigenvalue, 2 points per lane: 5-section per pass
  {
    const int j = tid >> 1, sub = tid & 1;
    const bool act = j < n;
    for (int it = 0; it < 40; ++it) {   // 5^40 > 2^92
      const double wdt = hi - lo;
      if (__all_sync(0xffffffffu, wdt <= 2.2e-16 * fmax(fabs(lo), fabs(hi)) + 1e-300)) break;
      const double x1 = lo + wdt * (2 * sub + 1) / 5.0, x2 = lo + wdt * (2 * sub + 2) / 5.0;
      double q1 = ds[0] - x1, q2 = ds[0] - x2;
      int c1 = q1 < 0.0, c2 = q2 < 0.0;
      for (int i = 1; i < n; ++i) {
        const double ee = e2[i - 1], di = ds[i];
        if (fabs(q1) < pivmin) q1 = -pivmin;
        if (fabs(q2) < pivmin) q2 = -pivmin;
        q1 = (di - x1) - ee / q1;
        q2 = (di - x2) - ee / q2;
        c1 += q1 < 0.0;
        c2 += q2 < 0.0;
      }
      unsigned int mask = ((act && c1 > j) ? 1u : 0u) << (2 * sub) | ((act && c2 > j) ? 2u : 0u) << (2 * sub);
      mask |= __shfl_xor_sync(0xffffffffu, mask, 1);
      const int pp = mask ? __ffs(mask) - 1 : 4;
      const double nlo = pp == 0 ? lo : lo + wdt * pp / 5.0;
      const double nhi = pp == 4 ? hi : lo + wdt * (pp + 1) / 5.0;
      lo = nlo;
      hi = nhi;
    }
    if (act && sub == 0) keys[j] = 0.5 * (lo + hi);   // ascending
  }
  if (tid == 0) s_deep = 0;
  __syncthreads();
  // sigma^2 descending, pi = identity, tails, depth check
  double* gS = reinterpret_cast<double*>(slab + gd.ws_sig2);
  int32_t* gP = reinterpret_cast<int32_t*>(slab + gd.ws_pi);
  double* desc_keys = keys + n;
  const double smax = fmax(keys[n - 1], 0.0);
  for (int j = tid; j < n; j += 256) {
    eig[j] = keys[j];
    const double vv = fmax(keys[n - 1 - j], 0.0);
    desc_keys[j] = vv;
    gS[j] = vv;
    gP[j] = j;
    if (vv >= 1e-12 * smax && vv < kEigMinSmall * kEigMinSmall * smax) s_deep = 1;
  }
  __syncthreads();
  cta_tails(desc_keys, n, reinterpret_cast<double*>(slab + gd.ws_T), part);
  if (tid == 0) {
    gdr.sweeps = 0;
    if (s_deep) {          // all eigenvectors now, then the relative-accurate refinement (refine.cu)
      gdr.eig = 2;
      gdr.k = n;
    }
    if (fb) fb[blockIdx.x] = s_deep;
  }
  (void)s_sc;
}

}  // namespace

bool refine_large_candidate(const GateDesc& gd) { return gd.regime == 1 && gd.n >= kMinN && gd.n <= kMaxN; }

// The eigen route (EAMPS_NO_EIG=1: every large gate takes the tcgen05 Jacobi route, the FP64 Gram
// eigenvalues only refine deep spectra -- the A/B reference).
bool eig_route(const GateDesc& gd) {
  static const bool off = getenv("EAMPS_NO_EIG") != nullptr;
  return !off && gd.regime == 1 && gd.n >= kEigMinN && gd.n <= kMaxN;
}

// must cover rlg_layout: g 16 n^2 | th 16 m n | d, e, eig 24 n | tau 16 n | p 32 n | part 32 KB |
// y 8 n^2 | slots kSlots 33 n | (256-byte alignment) | rs, cs 2 x tiles x TB x 16
size_t refine_large_scratch(int m, int n) {
  return (size_t)16 * n * n + (size_t)16 * m * n + (size_t)72 * n + 32 * 1024 + (size_t)8 * n * n +
         (size_t)kSlots * n * 33 + 256 + 2 * (size_t)g_tiles(n) * TB * 16 + 512;
}

namespace {
// mode 0: refinement of deep Jacobi spectra; mode 1: the eigen route's spectrum (fb: fallback flags).
int rlg_front(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* h_cand, const int32_t* d_cand, int nc,
              uint8_t* slab, DevState* st, const float2* d_us, int d, int32_t* iscr, int mode, int32_t* fb,
              cudaStream_t s, const RlgMarks* mk) {
  if (nc <= 0) return 0;
  int max_tiles = 0, max_gram = 0, max_n = 0;
  for (int c = 0; c < nc; ++c) {
    const GateDesc& g = h_desc[h_cand[c]];
    if (mode == 0 ? !refine_large_candidate(g) : !g.eig) continue;
    const int T = 64 / d;
    max_tiles = std::max(max_tiles, ((g.l + T - 1) / T) * ((g.r + T - 1) / T));
    const int nt = (g.n + 63) / 64;
    max_gram = std::max(max_gram, nt * (nt + 1) / 2);
    max_n = std::max(max_n, g.n);
  }
  if (max_n == 0) return 0;
  int32_t* flag = iscr;
  int32_t* list = iscr + nc;                                                   // nc + 1 ints
  // group barrier counters: one 128-byte line per group, at a 128-byte boundary after the lists
  unsigned int* ctr = reinterpret_cast<unsigned int*>(
      (reinterpret_cast<uintptr_t>(iscr + 2 * nc + 2) + 127) & ~uintptr_t(127));
  cudaMemsetAsync(list, 0, sizeof(int32_t), s);
  cudaMemsetAsync(ctr, 0, 128 * kMaxGroups, s);
  k_rlg_pick<<<(nc + 7) / 8, 256, 0, s>>>(d_desc, slab, d_cand, nc, flag, list, mode);
  rl_dbg(s, "k_rlg_pick");
  static std::atomic<unsigned long long> attr{0};
  const size_t tsm = tridiag_smem(kMaxN);
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(k_rlg_theta<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kThetaSmem);
    cudaFuncSetAttribute(k_rlg_theta<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kThetaSmem);
    cudaFuncSetAttribute(k_rlg_theta<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kThetaSmem);
    cudaFuncSetAttribute(k_rlg_theta<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kThetaSmem);
    cudaFuncSetAttribute(k_rlg_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kThetaSmem);
    cudaFuncSetAttribute(k_rlg_tridiag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
    cudaFuncSetAttribute(k_rlg_bisect<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * kMaxN);
    cudaFuncSetAttribute(k_rlg_bisect<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * kMaxN);
  }
  launch_theta64(d, max_tiles, nc, d_desc, d_cand, flag, slab, st, d_us, s);
  rl_dbg(s, "k_rlg_theta");
  k_rlg_gram<<<dim3(max_gram, nc), 256, kThetaSmem, s>>>(d_desc, d_cand, flag, slab);
  rl_dbg(s, "k_rlg_gram");
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_rlg_tridiag, TT, tsm);
  int grid = sms * std::max(per, 1);
  if (grid > 1024) grid = 1024;   // the partial-dot buffer holds 1024 CTAs
  // several gates in flight when the wave has several candidates (EAMPS_RLG_GROUPS overrides)
  static const int env_groups = getenv("EAMPS_RLG_GROUPS") ? atoi(getenv("EAMPS_RLG_GROUPS")) : 0;
  // measured (r02, 1 CTA per SM): n = 512: 4 / 8 / 16 / 37 / 74 groups 0.35 / 0.20 / 0.13 / 0.10 / 0.10
  // s per 512 gates of tridiagonalisation; n = 2048: 2 / 4 / 8 / 16 groups 28 / 25 / 23 / 22 ms per
  // gate. About n / 256 CTAs per group (>= 2): the per-step barrier and pivot latency amortised over
  // as many gates in flight as the traffic allows.
  int groups = env_groups > 0 ? env_groups : grid / std::max(2, max_n / 256);
  (void)kDefaultGroups;
  groups = std::max(1, std::min({groups, nc, kMaxGroups, grid}));
  const int cpg = grid / groups;
  const GateDesc* a_desc = d_desc;
  const int32_t* a_list = list;
  uint8_t* a_slab = slab;
  unsigned int* a_ctr = ctr;
  int a_cpg = cpg;
  void* args[] = {&a_desc, &a_list, &a_slab, &a_ctr, &a_cpg};
  if (mk) mk->at[0] = mk->mark(mk->ctx);
  cudaLaunchCooperativeKernel((const void*)k_rlg_tridiag, dim3(grid), dim3(TT), args, tsm, s);
  if (mk) mk->at[1] = mk->mark(mk->ctx);
  rl_dbg(s, "k_rlg_tridiag");
  // the lanes per eigenvalue from the launch's parallelism (upper bound: every candidate picked)
  int tot_n = 0;
  for (int c = 0; c < nc; ++c)
    if (mode == 0 ? refine_large_candidate(h_desc[h_cand[c]]) : h_desc[h_cand[c]].eig != 0) tot_n += h_desc[h_cand[c]].n;
  const size_t bsm = (size_t)16 * max_n;
  if (tot_n >= kBisWide)
    k_rlg_bisect<1><<<dim3((max_n + BT - 1) / BT, nc), BT, bsm, s>>>(d_desc, d_cand, flag, slab);
  else
    k_rlg_bisect<8><<<dim3((max_n + BT / 8 - 1) / (BT / 8), nc), BT, bsm, s>>>(d_desc, d_cand, flag, slab);
  rl_dbg(s, "k_rlg_bisect");
  k_rlg_finish<<<nc, 256, 0, s>>>(d_desc, d_cand, flag, slab, mode, fb);
  rl_dbg(s, "k_rlg_finish");
  return 6;
}
}  // namespace

// cand: device copy of the wave-local candidate gates (nc, max n / tiles from the host copy);
// iscr: wave scratch: flags (nc ints), list (nc + 1 ints), then kMaxGroups 128-byte barrier lines.
int launch_refine_large(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* h_cand, const int32_t* d_cand, int nc,
                        uint8_t* slab, DevState* st, const float2* d_us, int d, int32_t* iscr, cudaStream_t s) {
  return rlg_front(d_desc, h_desc, h_cand, d_cand, nc, slab, st, d_us, d, iscr, 0, nullptr, s, nullptr);
}

// The eigen route's front (a2 + a3 for the gates marked eig): theta64, G, T, eigenvalues, sorted
// sigma^2 and tails, pi = identity; fb[c] = 1 where the spectrum is too deep for it (the gate is
// unmarked on the device and must take the Jacobi route).
int launch_eig_front(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* h_cand, const int32_t* d_cand, int nc,
                     uint8_t* slab, DevState* st, const float2* d_us, int d, int32_t* iscr, int32_t* fb,
                     cudaStream_t s, const RlgMarks* mk) {
  return rlg_front(d_desc, h_desc, h_cand, d_cand, nc, slab, st, d_us, d, iscr, 1, fb, s, mk);
}

// The eigen route's right singular vectors for the kept k (after the select): inverse iteration
// on T, cluster MGS, back-transformation into V (FP32, columns 0 .. k-1).
// want: the gates whose desc.eig == want (1: the kept k after the select; 2: every column, before
// the refinement of a too-deep small spectrum). The host copy only bounds the grid.
int launch_eig_vectors(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* h_cand, const int32_t* d_cand, int nc,
                       uint8_t* slab, cudaStream_t s, int want) {
  int max_n = 0;
  for (int c = 0; c < nc; ++c)
    if (h_desc[h_cand[c]].eig) max_n = std::max(max_n, h_desc[h_cand[c]].n);
  if (max_n == 0) return 0;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(k_rlg_backtr<16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 512 * 16);
    cudaFuncSetAttribute(k_rlg_backtr<8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 1024 * 16);
    cudaFuncSetAttribute(k_rlg_backtr<4, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 2048 * 16);
    cudaFuncSetAttribute(k_rlg_backtr<2, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4096 * 16);
  }
  k_rlg_invit<<<dim3(kSlots / 32, nc), 32, 0, s>>>(d_desc, d_cand, slab, want);
  rl_dbg(s, "k_rlg_invit");
  k_rlg_mgs<<<nc, 256, 0, s>>>(d_desc, d_cand, slab, want);
  rl_dbg(s, "k_rlg_mgs");
  if (max_n <= 512)
    k_rlg_backtr<16, 2><<<dim3((max_n + 15) / 16, nc), 256, (size_t)16 * max_n * 16, s>>>(d_desc, d_cand, slab, want);
  else if (max_n <= 1024)
    k_rlg_backtr<8, 4><<<dim3((max_n + 7) / 8, nc), 256, (size_t)8 * max_n * 16, s>>>(d_desc, d_cand, slab, want);
  else if (max_n <= 2048)
    k_rlg_backtr<4, 8><<<dim3((max_n + 3) / 4, nc), 256, (size_t)4 * max_n * 16, s>>>(d_desc, d_cand, slab, want);
  else
    k_rlg_backtr<2, 16><<<dim3((max_n + 1) / 2, nc), 256, (size_t)2 * max_n * 16, s>>>(d_desc, d_cand, slab, want);
  rl_dbg(s, "k_rlg_backtr");
  return 3;
}

// Opt-in (EAMPS_EIG_SMALL=1): measured slower than the QR-regime Jacobi it would replace (config 2
// chi = 64 x 4096, one B200: 40.3K vs 71.5K updates/s; k_eig_cta 17 ms per 4096 gates, the FP64
// recontraction + Gram and the kept-vector back-transformation another ~60 ms) -- the block-recursive
// FP32 Jacobi runs at 0.57 of the FP32 SIMT peak, the one-CTA FP64 eigensolver at 0.04 of FP64.
bool eig_route_small(const GateDesc& gd) {
  static const bool on = getenv("EAMPS_EIG_SMALL") != nullptr && getenv("EAMPS_NO_EIG") == nullptr;
  return on && gd.regime == 3 && gd.n <= kSmallMaxN && gd.m >= gd.n;
}

// The eigen route's front for n <= 128 (QR-regime thetas): theta64, G (tile layout), then one CTA
// per gate (k_eig_cta). Gates flagged too deep get eig = 2 (all vectors before the refinement).
int launch_eig_small_front(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* h_cand, const int32_t* d_cand,
                           int nc, uint8_t* slab, DevState* st, const float2* d_us, int d, int32_t* iscr,
                           cudaStream_t s, const RlgMarks* mk) {
  int max_tiles = 0, max_gram = 0, max_n = 0;
  for (int c = 0; c < nc; ++c) {
    const GateDesc& g = h_desc[h_cand[c]];
    if (!g.eig) continue;
    const int T = 64 / d;
    max_tiles = std::max(max_tiles, ((g.l + T - 1) / T) * ((g.r + T - 1) / T));
    const int nt = (g.n + 63) / 64;
    max_gram = std::max(max_gram, nt * (nt + 1) / 2);
    max_n = std::max(max_n, g.n);
  }
  if (max_n == 0) return 0;
  int32_t* flag = iscr;
  int32_t* list = iscr + nc;
  cudaMemsetAsync(list, 0, sizeof(int32_t), s);
  k_rlg_pick<<<(nc + 7) / 8, 256, 0, s>>>(d_desc, slab, d_cand, nc, flag, list, 1);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(k_rlg_theta<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kThetaSmem);
    cudaFuncSetAttribute(k_rlg_theta<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kThetaSmem);
    cudaFuncSetAttribute(k_rlg_theta<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kThetaSmem);
    cudaFuncSetAttribute(k_rlg_theta<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kThetaSmem);
    cudaFuncSetAttribute(k_rlg_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kThetaSmem);
    cudaFuncSetAttribute(k_eig_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)eig_cta_smem(kSmallMaxN));
  }
  launch_theta64(d, max_tiles, nc, d_desc, d_cand, flag, slab, st, d_us, s);
  rl_dbg(s, "k_rlg_theta (small)");
  k_rlg_gram<<<dim3(max_gram, nc), 256, kThetaSmem, s>>>(d_desc, d_cand, flag, slab);
  rl_dbg(s, "k_rlg_gram (small)");
  if (mk) mk->at[0] = mk->mark(mk->ctx);
  k_eig_cta<<<nc, 256, eig_cta_smem(max_n), s>>>(d_desc, d_cand, slab, nullptr);
  if (mk) mk->at[1] = mk->mark(mk->ctx);
  rl_dbg(s, "k_eig_cta");
  return 4;
}

}  // namespace eamps
