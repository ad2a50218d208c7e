// precond_large.cu -- step a2, large regime: the R-preconditioner of the tcgen05 block Jacobi
// (the large-theta counterpart of svd_qr.cu's Householder preconditioner).
//
//   G = theta^H theta               (FP64 products of the FP32 theta, FP64 sums; k_pc_gram)
//   G = L L^H                       (blocked left-looking Cholesky in FP64; k_pc_chol_*)
//   B = L (= R^H for theta = Q R)   (FP32, n x n, the block Jacobi's working matrix; k_pc_b_from_l)
//   block Jacobi on B's columns, no V accumulation: B W = U Sigma gives R = W Sigma U^H and
//   theta = (Q W) Sigma U^H, so theta's right singular vectors are the normalised converged
//   columns of B (k_pc_vnorm); sigma then comes from the Rayleigh quotient with the ORIGINAL theta
//   and the FP64-anchored polish (launch_spectrum_polish), exactly as in the QR regime.
// Q is never formed. Accuracy: the FP64 Gram and Cholesky give R with relative backward error
// ~ eps64 kappa(theta)^2 (config 2 chi = 1024: 1e-16 x 1.2e10 ~ 1e-6 of the smallest sigma's
// direction, below the FP32 Jacobi's own tolerance), and the Rayleigh quotient is second order in
// the direction error. A pivot below n eps64 max_i G_ii (theta numerically rank-deficient) zeroes its
// column of L: that direction gets sigma = 0 (it lies in the FP32 noise of theta anyway).
// The preconditioner removes the V half of every rotation and cuts the sweeps (the QR regime:
// 12 -> 9 at chi = 64). PAPER.md:65 (M = U Lambda V^dagger), :114 ("performing its SVD");
// SURVEY §8(a) a2.
#include "eamps_internal.cuh"

namespace eamps {

namespace {

__device__ __forceinline__ double2 cmul_conj_acc(double2 acc, double2 a, double2 b) {   // acc + conj(a) b
  acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(-a.y, b.x, acc.y));
  return acc;
}

// G[i][j] = sum_r conj(theta[r][i]) theta[r][j] for the 64 x 64 tiles with ti >= tj (the lower
// triangle the Cholesky reads). theta: ws_theta (FP32, ld m); G: ws_log (FP64 complex, ld n).
__global__ void __launch_bounds__(256, 2) k_pc_gram(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                 uint8_t* slab) {
  const GateDesc& gd = desc[list[blockIdx.y]];
  if (gd.jrows <= 0) return;
  const int m = gd.m, n = gd.n, T = (n + 63) / 64;
  const int t = blockIdx.x;
  if (t >= T * (T + 1) / 2) return;
  int ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while (ti * (ti + 1) / 2 > t) --ti;
  while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
  const int tj = t - ti * (ti + 1) / 2;
  const float2* th = reinterpret_cast<const float2*>(slab + gd.ws_theta);
  double2* G = reinterpret_cast<double2*>(slab + gd.ws_log);
  __shared__ double2 Ai[16][65], Aj[16][65];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double2 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = make_double2(0.0, 0.0);
  // the next 16-row chunk is fetched into registers while the current one multiplies (ncu r02: long
  // scoreboard was the top stall with the fetch in front of every chunk)
  float2 pi[4], pj[4];
  auto fetch = [&](int r0) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int x = tid + it * 256;
      const int c = x >> 4, r = r0 + (x & 15);
      const int ci = ti * 64 + c, cj = tj * 64 + c;
      pi[it] = (r < m && ci < n) ? th[(int64_t)ci * m + r] : make_float2(0.f, 0.f);
      pj[it] = (r < m && cj < n) ? th[(int64_t)cj * m + r] : make_float2(0.f, 0.f);
    }
  };
  fetch(0);
  for (int r0 = 0; r0 < m; r0 += 16) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int x = tid + it * 256;
      const int c = x >> 4, rr = x & 15;
      Ai[rr][c] = make_double2(pi[it].x, pi[it].y);
      Aj[rr][c] = make_double2(pj[it].x, pj[it].y);
    }
    __syncthreads();
    if (r0 + 16 < m) fetch(r0 + 16);
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
      double2 xi[4], yj[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) xi[a] = Ai[k][ty + 16 * a];   // 2 addresses per warp (broadcast)
#pragma unroll
      for (int b = 0; b < 4; ++b) yj[b] = Aj[k][tx + 16 * b];   // consecutive: no bank conflicts
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = cmul_conj_acc(acc[a][b], xi[a], yj[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ti * 64 + ty + 16 * a, j = tj * 64 + tx + 16 * b;
      if (i < n && j < n) G[(int64_t)j * n + i] = acc[a][b];
    }
}

// In-place blocked left-looking Cholesky G = L L^H (lower), panels of 32 columns, two launches per
// panel so that the row blocks of a panel run in parallel (chi = 1024 has only tens of gates):
//   k_pc_chol_diag  (one CTA per gate): the diagonal block G_JJ -= L_J,0:c0 L_J,0:c0^H, factored in
//                   shared memory (pivots <= tau -> zero column) and inverted; L_JJ -> G, L_JJ^-1 ->
//                   the gate's scratch (after G);
//   k_pc_chol_panel (one CTA per 32-row block below the diagonal block and gate): the same update,
//                   then X = G_blk L_JJ^-H = G_blk (L_JJ^-1)^H (a small GEMM, no serial solve).
// tau = n eps64 max_i G_ii, from the unfactored G in the first diagonal launch.
struct CholScratch {
  double2 Mi[32][32];
  double tau;
};

__device__ __forceinline__ CholScratch* chol_scratch(uint8_t* slab, const GateDesc& gd) {
  return reinterpret_cast<CholScratch*>(slab + gd.ws_log + (size_t)16 * gd.n * gd.n);
}

// Cholesky of the 32 x 32 diagonal block (w x w used) in shared memory by a 256-thread CTA, in the
// square-root-free (L D L^H) form of the right-looking recurrence: step j subtracts
// A[i][j] conj(A[k][j]) / d_j from every A[i][k], j < k <= i < w, reading the unscaled column j,
// which no thread writes in that step -- one barrier per step instead of three (scale the column,
// barrier, update, barrier). Then L[i][j] = A[i][j] / sqrt(d_j), L[j][j] = sqrt(d_j). A pivot
// d_j <= tau zeroes column j (no update from it), as before. s_rs: 32 doubles of shared memory.
__device__ __forceinline__ void chol32(double2 (*Lp)[33], int w, double tau, double* s_rs) {
  const int tid = threadIdx.x;
  for (int j = 0; j < w; ++j) {
    const double d = Lp[j][j].x;
    const double id = d > tau ? 1.0 / d : 0.0;
    for (int x = tid; x < 32 * 32; x += 256) {
      const int i = x >> 5, k = x & 31;
      if (k > j && k <= i && i < w) {
        const double2 a = Lp[i][j], q = Lp[k][j];   // A[i][k] -= A[i][j] conj(A[k][j]) / d_j
        Lp[i][k].x -= (a.x * q.x + a.y * q.y) * id;
        Lp[i][k].y -= (a.y * q.x - a.x * q.y) * id;
      }
    }
    __syncthreads();
  }
  if (tid < 32) {
    const double d = tid < w ? Lp[tid][tid].x : 0.0;
    s_rs[tid] = d > tau ? rsqrt(d) : 0.0;
  }
  __syncthreads();
  for (int x = tid; x < 32 * 32; x += 256) {
    const int i = x >> 5, j = x & 31;
    if (i < w && j <= i) {
      const double r = s_rs[j];
      const double2 a = Lp[i][j];
      Lp[i][j] = i == j ? make_double2(a.x * r, 0.0) : make_double2(a.x * r, a.y * r);
    }
  }
  __syncthreads();
}

// M = L_JJ^-1 (lower triangular, w x w of the 32 x 32 block, zeros elsewhere) by all 8 warps of a
// 256-thread CTA: column-oriented forward substitution of L M_j = e_j with one lane per row. Warp wp
// takes the columns j = wp, wp + 8, wp + 16, wp + 24 in lockstep; at step k lane k finalises
// M[k][j] = b_k / L[k][k] and broadcasts it, and every lane i > k subtracts L[i][k] M[k][j] --
// the same products in the same order (k ascending) as the row-by-row recurrence
// M[i][j] = -(sum_{j <= k < i} L[i][k] M[k][j]) / L[i][i], but 32 lanes x 8 warps in parallel
// instead of one thread per column (that serial loop was the CTA's critical path: ~22% of the
// kernel's warps waited on the barrier after it, ncu r02). A zero pivot (L[k][k] = 0) zeroes row k
// of M, and a zero L[j][j] the whole column j, as before.
__device__ __forceinline__ void tri_inv32(const double2 (*Lp)[33], double2 (*Mi)[33], int w) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const double dl = (lane < w) ? Lp[lane][lane].x : 0.0;
  const double di = dl > 0.0 ? 1.0 / dl : 0.0;
  double2 b[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) b[c] = make_double2(lane == wp + 8 * c ? 1.0 : 0.0, 0.0);
  for (int k = 0; k < w; ++k) {
    const double2 lik = (lane > k && lane < w) ? Lp[lane][k] : make_double2(0.0, 0.0);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (k < wp + 8 * c) continue;                 // warp-uniform
      double2 m = make_double2(b[c].x * di, b[c].y * di);
      m.x = __shfl_sync(0xffffffffu, m.x, k);
      m.y = __shfl_sync(0xffffffffu, m.y, k);
      if (lane == k) {
        b[c] = m;
      } else if (lane > k) {                        // b_i -= L[i][k] M[k][j]
        b[c].x -= lik.x * m.x - lik.y * m.y;
        b[c].y -= lik.x * m.y + lik.y * m.x;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int j = wp + 8 * c;
    Mi[lane][j] = (j < w && lane >= j && lane < w) ? b[c] : make_double2(0.0, 0.0);
  }
}

// acc (row rr, columns cb .. cb+3 of the 32 x 32 block at rows i0, columns c0) = G_blk - L_blk L_J^H
__device__ __forceinline__ void chol_block_update(const double2* G, int n, int i0, int c0, int w, double2 (&acc)[4],
                                                  double2 (*As)[17], double2 (*Bs)[17]) {
  const int tid = threadIdx.x, rr = tid >> 3, cb = (tid & 7) * 4;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int i = i0 + rr, j = c0 + cb + b;
    acc[b] = (i < n && j < c0 + w) ? G[(int64_t)j * n + i] : make_double2(0.0, 0.0);
  }
  for (int k0 = 0; k0 < c0; k0 += 16) {       // k0 + 16 <= c0 (c0 is a multiple of 32)
    for (int x = tid; x < 32 * 16; x += 256) {
      const int r = x & 31, kk = x >> 5;
      const int k = k0 + kk;
      As[r][kk] = (i0 + r < n) ? G[(int64_t)k * n + i0 + r] : make_double2(0.0, 0.0);
      Bs[r][kk] = (c0 + r < n) ? G[(int64_t)k * n + c0 + r] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < 16; ++kk) {
      const double2 a = As[rr][kk];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double2 q = Bs[cb + b][kk];   // acc -= a conj(q)
        acc[b].x -= a.x * q.x + a.y * q.y;
        acc[b].y -= a.y * q.x - a.x * q.y;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_pc_chol_diag(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                      uint8_t* slab, int c0) {
  const GateDesc& gd = desc[list[blockIdx.x]];
  if (gd.jrows <= 0 || c0 >= gd.n) return;
  const int n = gd.n, w = min(32, n - c0);
  double2* G = reinterpret_cast<double2*>(slab + gd.ws_log);
  CholScratch* W = chol_scratch(slab, gd);
  __shared__ double2 Mi[32][33];
  __shared__ double2 AB[2][32][17];                           // update staging, then Lp
  double2 (*As)[17] = AB[0];
  double2 (*Bs)[17] = AB[1];
  double2 (*Lp)[33] = reinterpret_cast<double2(*)[33]>(&AB[0][0][0]);
  __shared__ double s_red[8];
  __shared__ double s_rs[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rr = tid >> 3, cb = (tid & 7) * 4;
  double tau;
  if (c0 == 0) {
    double dm = 0.0;
    for (int i = tid; i < n; i += 256) dm = fmax(dm, G[(int64_t)i * n + i].x);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    if (lane == 0) s_red[warp] = dm;
    __syncthreads();
    double gmax = 0.0;
    for (int v = 0; v < 8; ++v) gmax = fmax(gmax, s_red[v]);
    tau = (double)n * 2.220446049250313e-16 * gmax;
    if (tid == 0) W->tau = tau;
  } else {
    tau = W->tau;
  }
  double2 acc[4];
  chol_block_update(G, n, c0, c0, w, acc, As, Bs);
#pragma unroll
  for (int b = 0; b < 4; ++b) Lp[rr][cb + b] = acc[b];
  __syncthreads();
  chol32(Lp, w, tau, s_rs);
  tri_inv32(Lp, Mi, w);                         // L_JJ^-1
  __syncthreads();
  for (int x = tid; x < 32 * 32; x += 256) {
    const int i = x >> 5, j = x & 31;
    if (i < w && j <= i) G[(int64_t)(c0 + j) * n + c0 + i] = Lp[i][j];
    W->Mi[i][j] = Mi[i][j];
  }
}

__global__ void __launch_bounds__(256) k_pc_chol_panel(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                       uint8_t* slab, int c0) {
  const GateDesc& gd = desc[list[blockIdx.y]];
  const int i0 = c0 + 32 * (1 + (int)blockIdx.x);
  if (gd.jrows <= 0 || i0 >= gd.n) return;
  const int n = gd.n, w = min(32, n - c0);
  double2* G = reinterpret_cast<double2*>(slab + gd.ws_log);
  const CholScratch* W = chol_scratch(slab, gd);
  __shared__ double2 Mi[32][33];
  __shared__ double2 AB[2][32][17];                           // update staging, then Tt
  double2 (*As)[17] = AB[0];
  double2 (*Bs)[17] = AB[1];
  double2 (*Tt)[33] = reinterpret_cast<double2(*)[33]>(&AB[0][0][0]);
  const int tid = threadIdx.x, rr = tid >> 3, cb = (tid & 7) * 4;
  for (int x = tid; x < 32 * 32; x += 256) Mi[x >> 5][x & 31] = W->Mi[x >> 5][x & 31];
  double2 acc[4];
  chol_block_update(G, n, i0, c0, w, acc, As, Bs);   // (its barriers also publish Mi)
#pragma unroll
  for (int b = 0; b < 4; ++b) Tt[rr][cb + b] = acc[b];
  __syncthreads();
#pragma unroll
  for (int b = 0; b < 4; ++b) {                 // x_j = sum_{k <= j} t_k conj(M[j][k])
    const int j = cb + b;
    double2 x = make_double2(0.0, 0.0);
    for (int k = 0; k <= j && k < w; ++k) {
      const double2 tk = Tt[rr][k], q = Mi[j][k];
      x.x += tk.x * q.x + tk.y * q.y;
      x.y += tk.y * q.x - tk.x * q.y;
    }
    const int i = i0 + rr;
    if (i < n && j < w) G[(int64_t)(c0 + j) * n + i] = x;
  }
}

// Small n (<= 128, the QR regime): the whole blocked Cholesky in one CTA per gate (4096 gates give
// the parallelism; no per-panel launches). In-place left-looking G = L L^H (lower), panels of 32
// columns: (1) every 32-row block of the panel gets G[i][panel] -= L[i][0:c0] L[panel][0:c0]^H;
// (2) the diagonal block is factored in shared memory (pivots <= tau -> zero column) and inverted;
// (3) the blocks below become X = G_blk L_JJ^-H = G_blk (L_JJ^-1)^H (a small GEMM, no serial solve).
__global__ void __launch_bounds__(256, 3) k_pc_chol_cta(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                 uint8_t* slab) {
  const GateDesc& gd = desc[list[blockIdx.x]];
  if (gd.jrows <= 0) return;
  const int n = gd.n;
  double2* G = reinterpret_cast<double2*>(slab + gd.ws_log);
  // B = L in FP32 (n x n_pad, ld n; the block Jacobi's working matrix, k_pc_b_from_l's layout), written
  // as each block of L becomes final -- no separate conversion pass over L (0.47 ms per chi = 64 step)
  float2* Bf = reinterpret_cast<float2*>(slab + gd.ws_theta);
  struct Smem {
    double2 Lp[32][33];   // factored diagonal block L_JJ; later the row block being solved
    double2 Mi[32][33];   // L_JJ^-1 (lower)
    double2 As[32][17], Bs[32][17];
  };
  extern __shared__ __align__(16) uint8_t pc_sm[];
  Smem& S = *reinterpret_cast<Smem*>(pc_sm);
  auto& Lp = S.Lp;
  auto& Mi = S.Mi;
  auto& As = S.As;
  auto& Bs = S.Bs;
  auto& Tt = S.Lp;
  __shared__ double s_red[8];
  __shared__ double s_rs[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // 32 x 32 tile: row rr, columns cb + 8b (b < 4). Columns 8 apart, not 4 consecutive: the 8 threads of a
  // shared-memory phase then read 8 consecutive rows of Bs / Mi (padded strides: distinct banks); with
  // cb = 4 (tid & 7) they read rows 0, 4, .., 28, which share 2 bank groups (4-way conflicts, ncu r02).
  const int rr = tid >> 3, cb = tid & 7;
  // pivot threshold tau = n eps64 max_i G_ii
  double dm = 0.0;
  for (int i = tid; i < n; i += 256) dm = fmax(dm, G[(int64_t)i * n + i].x);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
  if (lane == 0) s_red[warp] = dm;
  __syncthreads();
  double gmax = 0.0;
  for (int w = 0; w < 8; ++w) gmax = fmax(gmax, s_red[w]);
  const double tau = (double)n * 2.220446049250313e-16 * gmax;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int w = min(32, n - c0);
    for (int i0 = c0; i0 < n; i0 += 32) {
      double2 acc[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = i0 + rr, j = c0 + cb + 8 * b;
        acc[b] = (i < n && j < c0 + w) ? G[(int64_t)j * n + i] : make_double2(0.0, 0.0);
      }
      for (int k0 = 0; k0 < c0; k0 += 16) {       // k0 + 16 <= c0 (c0 is a multiple of 32)
        for (int x = tid; x < 32 * 16; x += 256) {
          const int r = x & 31, kk = x >> 5;
          const int k = k0 + kk;
          As[r][kk] = (i0 + r < n) ? G[(int64_t)k * n + i0 + r] : make_double2(0.0, 0.0);
          Bs[r][kk] = (c0 + r < n) ? G[(int64_t)k * n + c0 + r] : make_double2(0.0, 0.0);
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < 16; ++kk) {
          const double2 a = As[rr][kk];
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const double2 q = Bs[cb + 8 * b][kk];   // acc -= a conj(q)
            acc[b].x -= a.x * q.x + a.y * q.y;
            acc[b].y -= a.y * q.x - a.x * q.y;
          }
        }
        __syncthreads();
      }
      if (i0 == c0) {
        // ---- factor the diagonal block in shared memory (right-looking, unblocked)
#pragma unroll
        for (int b = 0; b < 4; ++b) Lp[rr][cb + 8 * b] = acc[b];
        __syncthreads();
        chol32(Lp, w, tau, s_rs);
        // ---- inverse of the lower-triangular L_JJ, column by column (thread j < w owns column j)
        tri_inv32(Lp, Mi, w);
        __syncthreads();
        // ---- write L_JJ (lower part) back, and B's diagonal block (FP32, zeros above the diagonal)
        for (int x = tid; x < 32 * 32; x += 256) {
          const int i = x >> 5, j = x & 31;
          if (i < w && j <= i) G[(int64_t)(c0 + j) * n + c0 + i] = Lp[i][j];
          if (i < w && j < w) {
            const double2 l = Lp[i][j];
            Bf[(int64_t)(c0 + j) * n + c0 + i] = j <= i ? make_float2((float)l.x, (float)l.y) : make_float2(0.f, 0.f);
          }
        }
      } else {
        // ---- X = T (L_JJ^-1)^H: x_j = sum_{k <= j} t_k conj(M[j][k]). The thread's 4 columns run
        // as 4 independent accumulation chains over k <= cb + 24 (M is stored lower-triangular with
        // zeros above the diagonal, so the extra terms add exact zeros): one T load per 4 products,
        // no serial dependence between the columns (ncu r02: this loop was 23% of the kernel's stall
        // samples as 4 back-to-back serial chains with 2 loads per product).
#pragma unroll
        for (int b = 0; b < 4; ++b) Tt[rr][cb + 8 * b] = acc[b];
        __syncthreads();
        double2 x[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) x[b] = make_double2(0.0, 0.0);
        const int kend = min(cb + 25, w);
        for (int k = 0; k < kend; ++k) {
          const double2 tk = Tt[rr][k];
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const double2 q = Mi[cb + 8 * b][k];
            x[b].x += tk.x * q.x + tk.y * q.y;
            x[b].y += tk.y * q.x - tk.x * q.y;
          }
        }
        const int i = i0 + rr;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int j = cb + 8 * b;
          if (i < n && j < w) {
            G[(int64_t)(c0 + j) * n + i] = x[b];
            Bf[(int64_t)(c0 + j) * n + i] = make_float2((float)x[b].x, (float)x[b].y);
          }
        }
      }
      __syncthreads();
    }
  }
  // B: zeros in the blocks above the diagonal blocks and in the pad columns
  const int np = gd.n_pad;
  for (int64_t x = tid; x < (int64_t)n * np; x += 256) {
    const int j = (int)(x / n), i = (int)(x % n);
    if (j >= n || (i >> 5) < (j >> 5)) Bf[x] = make_float2(0.f, 0.f);
  }
}

// ---- n <= 128 (the QR regime; config 2 chi = 64): Gram + Cholesky + B = L fused in ONE CTA per gate,
// G (FP64, packed lower triangle, 132 KB at n = 128) never leaves shared memory. Same arithmetic as
// k_pc_gram + k_pc_chol_cta + k_pc_b_from_l (FP64 products of the FP32 theta, right-looking blocked
// Cholesky with 32-column panels, pivots <= tau = n eps64 max_i G_ii -> zero column), different
// summation order. The three kernels take 2.54 + 4.57 + 0.47 ms per 4096-gate step (chi = 64, r02
// launch list); this variant 9.3 ms (opt-in, see launch_precond_large).
constexpr int kPcFusedMaxN = 128;
__host__ __device__ inline int pc_up(int i, int j) { return i * (i + 1) / 2 + j; }   // j <= i
size_t pc_fused_smem(int n) {
  return (((size_t)n * (n + 1) / 2 * 16 + 15) & ~(size_t)15) + (size_t)32 * (n + 1) * 8 + 64;
}

__global__ void __launch_bounds__(256, 1) k_pc_fused(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                    uint8_t* slab) {
  const GateDesc& gd = desc[list[blockIdx.x]];
  if (gd.jrows <= 0) return;
  const int m = gd.m, n = gd.n, np = gd.n_pad;
  extern __shared__ __align__(16) uint8_t pf_sm[];
  double2* G = reinterpret_cast<double2*>(pf_sm);
  float2* Th = reinterpret_cast<float2*>(pf_sm + (((size_t)n * (n + 1) / 2 * 16 + 15) & ~(size_t)15));
  const int pitch = n + 1;
  __shared__ uint8_t bI[512], bJ[512];
  __shared__ int s_nblk;
  __shared__ double s_red[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float2* __restrict__ th = reinterpret_cast<const float2*>(slab + gd.ws_theta);
  // ---- 1. G = theta^H theta, lower triangle, 4 x 8 register blocks (I: rows 4I.., J: columns 8J..)
  if (tid == 0) {
    int c = 0;
    const int NI = (n + 3) / 4, NJ = (n + 7) / 8;
    for (int I = 0; I < NI; ++I)
      for (int J = 0; J < NJ && 8 * J <= 4 * I + 3; ++J) {
        bI[c] = (uint8_t)I;
        bJ[c] = (uint8_t)J;
        ++c;
      }
    s_nblk = c;
  }
  __syncthreads();
  const int nblk = s_nblk;
  for (int b0 = 0; b0 < nblk; b0 += 256) {
    const int b = b0 + tid;
    const bool act = b < nblk;
    const int i0 = act ? 4 * bI[b] : 0, j0 = act ? 8 * bJ[b] : 0;
    double2 acc[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[a][c] = make_double2(0.0, 0.0);
    for (int r0 = 0; r0 < m; r0 += 32) {
      __syncthreads();
      for (int x = tid; x < 32 * n; x += 256) {
        const int rr = x & 31, c = x >> 5, r = r0 + rr;
        Th[rr * pitch + c] = r < m ? th[(int64_t)c * m + r] : make_float2(0.f, 0.f);
      }
      __syncthreads();
      if (act) {
#pragma unroll 2
        for (int rr = 0; rr < 32; ++rr) {
          double2 xi[4], yj[8];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const float2 v = (i0 + a < n) ? Th[rr * pitch + i0 + a] : make_float2(0.f, 0.f);
            xi[a] = make_double2(v.x, v.y);
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float2 v = (j0 + c < n) ? Th[rr * pitch + j0 + c] : make_float2(0.f, 0.f);
            yj[c] = make_double2(v.x, v.y);
          }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[a][c] = cmul_conj_acc(acc[a][c], xi[a], yj[c]);
        }
      }
    }
    if (act) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int i = i0 + a, j = j0 + c;
          if (i < n && j <= i) G[pc_up(i, j)] = acc[a][c];
        }
    }
  }
  __syncthreads();
  // ---- 2. G = L L^H in place (right-looking, 32-column panels)
  double dm = 0.0;
  for (int i = tid; i < n; i += 256) dm = fmax(dm, G[pc_up(i, i)].x);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
  if (lane == 0) s_red[warp] = dm;
  __syncthreads();
  double gmax = 0.0;
  for (int w = 0; w < 8; ++w) gmax = fmax(gmax, s_red[w]);
  const double tau = (double)n * 2.220446049250313e-16 * gmax;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int w = min(32, n - c0);
    // (a) the diagonal block, one warp, lane = row
    if (warp == 0) {
      for (int j = 0; j < w; ++j) {
        const double d = G[pc_up(c0 + j, c0 + j)].x;
        const bool ok = d > tau;
        const double il = ok ? rsqrt(d) : 0.0;
        __syncwarp();
        if (lane >= j && lane < w) {
          const int q = pc_up(c0 + lane, c0 + j);
          if (lane == j) G[q] = make_double2(ok ? d * il : 0.0, 0.0);
          else G[q] = make_double2(G[q].x * il, G[q].y * il);
        }
        __syncwarp();
        if (lane > j && lane < w) {           // row `lane`: G[i][k] -= G[i][j] conj(G[k][j]), j < k <= i
          const double2 a = G[pc_up(c0 + lane, c0 + j)];
          for (int k = j + 1; k <= lane; ++k) {
            const double2 q = G[pc_up(c0 + k, c0 + j)];
            double2& t = G[pc_up(c0 + lane, c0 + k)];
            t.x -= a.x * q.x + a.y * q.y;
            t.y -= a.y * q.x - a.x * q.y;
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // (b) the rows below: x L_JJ^H = g_i by forward substitution, one thread per row
    for (int i = c0 + w + tid; i < n; i += 256) {
      for (int j = 0; j < w; ++j) {
        double2 x = G[pc_up(i, c0 + j)];
        for (int k = 0; k < j; ++k) {          // x -= L[i][k] conj(L[j][k])
          const double2 a = G[pc_up(i, c0 + k)], q = G[pc_up(c0 + j, c0 + k)];
          x.x -= a.x * q.x + a.y * q.y;
          x.y -= a.y * q.x - a.x * q.y;
        }
        const double l = G[pc_up(c0 + j, c0 + j)].x;
        const double il = l > 0.0 ? 1.0 / l : 0.0;
        G[pc_up(i, c0 + j)] = make_double2(x.x * il, x.y * il);
      }
    }
    __syncthreads();
    // (c) the trailing lower triangle: G[i][s] -= sum_k L[i][k] conj(L[s][k]), c0 + w <= s <= i
    const int r = n - c0 - w;
    const int ntr = r * (r + 1) / 2;
    for (int x = tid; x < ntr; x += 256) {
      int ii = (int)((sqrt(8.0 * x + 1.0) - 1.0) * 0.5);
      while (ii * (ii + 1) / 2 > x) --ii;
      while ((ii + 1) * (ii + 2) / 2 <= x) ++ii;
      const int ss = x - ii * (ii + 1) / 2;
      const int i = c0 + w + ii, sc = c0 + w + ss;
      double2 t = G[pc_up(i, sc)];
      for (int k = 0; k < w; ++k) {
        const double2 a = G[pc_up(i, c0 + k)], q = G[pc_up(sc, c0 + k)];
        t.x -= a.x * q.x + a.y * q.y;
        t.y -= a.y * q.x - a.x * q.y;
      }
      G[pc_up(i, sc)] = t;
    }
    __syncthreads();
  }
  // ---- 3. B = L in FP32 (n x n_pad, ld n), zero above the diagonal and in the pad columns
  float2* B = reinterpret_cast<float2*>(slab + gd.ws_theta);
  for (int x = tid; x < n * np; x += 256) {
    const int j = x / n, i = x % n;
    float2 v = make_float2(0.f, 0.f);
    if (j < n && i >= j) {
      const double2 g = G[pc_up(i, j)];
      v = make_float2((float)g.x, (float)g.y);
    }
    B[x] = v;
  }
}

// B = L in FP32 (n x n_pad, ld n): the lower triangle of L, zeros above it and in the pad columns
__global__ void k_pc_b_from_l(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list, uint8_t* slab) {
  const GateDesc& gd = desc[list[blockIdx.y]];
  if (gd.jrows <= 0) return;
  const int n = gd.n, np = gd.n_pad;
  const double2* G = reinterpret_cast<const double2*>(slab + gd.ws_log);
  float2* B = reinterpret_cast<float2*>(slab + gd.ws_theta);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < (int64_t)n * np;
       x += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(x / n), i = (int)(x % n);
    float2 v = make_float2(0.f, 0.f);
    if (j < n && i >= j) {
      const double2 g = G[(int64_t)j * n + i];
      v = make_float2((float)g.x, (float)g.y);
    }
    B[x] = v;
  }
}

// V[:, j] = b_j / |b_j| (FP64 norm) for j < n, rows n .. n_pad and columns n .. n_pad zero
// A column at or below the Jacobi's rounding floor (|b_j|^2 <= (2^-24 |theta|_F)^2) was never rotated,
// so its direction is not orthogonal to the others: it carries no singular value (v_j = 0).
__global__ void k_pc_vnorm(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list, uint8_t* slab,
                           const double* __restrict__ norm2) {
  const GateDesc& gd = desc[list[blockIdx.y]];
  if (gd.jrows <= 0) return;
  const int n = gd.n, np = gd.n_pad;
  const float2* B = reinterpret_cast<const float2*>(slab + gd.ws_theta);
  float2* V = reinterpret_cast<float2*>(slab + gd.ws_V);
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= np) return;
  double a = 0.0;
  if (j < n)
    for (int i = lane; i < n; i += 32) a += (double)B[(int64_t)j * n + i].x * B[(int64_t)j * n + i].x +
                                            (double)B[(int64_t)j * n + i].y * B[(int64_t)j * n + i].y;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  const float sc = a > norm2[blockIdx.y] * 3.552713678800501e-15 ? (float)(1.0 / sqrt(a)) : 0.f;
  for (int i = lane; i < np; i += 32) {
    const float2 b = (j < n && i < n) ? B[(int64_t)j * n + i] : make_float2(0.f, 0.f);
    V[(int64_t)j * np + i] = make_float2(b.x * sc, b.y * sc);
  }
}

}  // namespace

bool large_precond_enabled() {
  static const bool off = getenv("EAMPS_NO_LARGE_PRECOND") != nullptr || getenv("EAMPS_LARGE_SIMT") != nullptr;
  return !off;
}

// m < n (wide theta): G = theta^H theta is n x n of rank <= m; the Cholesky zeroes the dependent
// pivots and the Jacobi runs on B = L (n x n) whose zero columns carry sigma = 0 -- still no V and
// fewer rows per rotation than the V-accumulating path (m + n). EAMPS_NO_WIDE_PRECOND=1: off (A/B).
bool large_precond_wide() {
  static const bool off = getenv("EAMPS_NO_WIDE_PRECOND") != nullptr;
  return !off;
}

size_t large_precond_scratch(int n) { return (size_t)16 * n * n + sizeof(CholScratch); }

int launch_precond_large(GateDesc* d_desc, const int32_t* d_list, int count, int max_n, uint8_t* slab, cudaStream_t s) {
  if (count <= 0) return 0;
  // EAMPS_PC_FUSED=1: the one-CTA fused variant. Measured slower on the default bench (precond
  // sub-phase 9.3 ms vs 7.5 ms for the three kernels: with 165 KB of shared memory one CTA per SM
  // runs the gate's Gram passes and 32-step panel factorisations with nothing to hide their latency),
  // so the separate kernels stay the default.
  static const bool fused = getenv("EAMPS_PC_FUSED") != nullptr;
  if (fused && max_n <= kPcFusedMaxN) {
    static std::atomic<unsigned long long> fattr{0};
    if (first_on_device(fattr))
      cudaFuncSetAttribute(k_pc_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pc_fused_smem(kPcFusedMaxN));
    k_pc_fused<<<count, 256, pc_fused_smem(max_n), s>>>(d_desc, d_list, slab);
    return 1;
  }
  const int T = (max_n + 63) / 64;
  k_pc_gram<<<dim3(T * (T + 1) / 2, count), 256, 0, s>>>(d_desc, d_list, slab);
  static const bool cta_small = getenv("EAMPS_CHOL_PANELS") == nullptr;   // dev A/B switch
  if (max_n <= 128 && cta_small) {
    constexpr int kCholSmem = (2 * 32 * 33 + 2 * 32 * 17) * 16;
    static std::atomic<unsigned long long> attr{0};
    if (first_on_device(attr)) {
      cudaFuncSetAttribute(k_pc_chol_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, kCholSmem);
    }
    k_pc_chol_cta<<<count, 256, kCholSmem, s>>>(d_desc, d_list, slab);   // also writes B = L
    return 2;
  }
  for (int c0 = 0; c0 < max_n; c0 += 32) {
    k_pc_chol_diag<<<count, 256, 0, s>>>(d_desc, d_list, slab, c0);
    const int rb = (max_n - c0 - 1) / 32;       // row blocks below the diagonal block
    if (rb > 0) k_pc_chol_panel<<<dim3(rb, count), 256, 0, s>>>(d_desc, d_list, slab, c0);
  }
  k_pc_b_from_l<<<dim3(64, count), 256, 0, s>>>(d_desc, d_list, slab);
  return 2 + 2 * ((max_n + 31) / 32);
}

int launch_precond_vnorm(GateDesc* d_desc, const int32_t* d_list, int count, int max_np, uint8_t* slab,
                         const double* norm2, cudaStream_t s) {
  if (count <= 0) return 0;
  k_pc_vnorm<<<dim3((max_np + 7) / 8, count), 256, 0, s>>>(d_desc, d_list, slab, norm2);
  return 1;
}

}  // namespace eamps
