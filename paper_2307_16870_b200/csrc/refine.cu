// refine.cu -- FP64 Rayleigh-Ritz refinement of the singular values (steps a2/a3) for
// gates whose spectrum is deep.
//
// Why: the FP32 Jacobi paths deliver right singular vectors V with a normwise error ~eps32: the
// Cholesky factor B = L is rounded to FP32 before the block Jacobi, an FP32 Householder R carries
// eps32 sigma_max, an FP32-accumulated V drifts by ~1e-6. A small sigma_j (sigma_j / sigma_max <~
// 1e-4) is then contaminated through the Rayleigh quotient ||theta v_j||^2 by the large singular
// directions mixed into v_j, and the pairwise second-order polish cannot undo a mixing that large
// (measured in a numpy model of the pipeline on a graded 128 x 128 theta, sigma down to 3e-6
// sigma_max: Rayleigh 107 % error, pairwise polish 12-54 %, this refinement 1e-8; GPU: up to 100 %
// on the config-4 MPO and the graded edge tests, tests/test_gpu_edge.py).
// What: C = B^H B with B = theta V (theta = lambda (x) Theta', the contraction's FP32 output; V the
// FP32 right singular vectors, unit columns), formed with FP64 products and sums; its eigenvalues by
// a cyclic two-sided Jacobi in FP64 (tournament order, relative off-diagonal tolerance 1e-12).
// By Ostrowski's theorem eig(V^H theta^H theta V) = eig(theta^H theta) up to factors in
// [sigma_min(V)^2, sigma_max(V)^2] = 1 +- ||V^H V - I|| (~1e-6 for the FP32 V), for EVERY
// eigenvalue, however small; C is computed from B column by column in FP64, so its small
// eigenvalues keep their relative accuracy, and two-sided Jacobi on a positive semidefinite C
// computes them with relative accuracy. sigma_j^2 = C_jj after convergence replaces the Rayleigh
// value of column j; then the sort and the FP64 tails (a3) are redone. V itself is not rotated (the
// reabsorb keeps the FP32 V: the state is unchanged to storage precision; the ranks and fidelities
// follow the refined sigma). PAPER.md:114 ("performing its SVD", "singular values in decreasing
// order"), :65; north_star tolerance "singular values: relative 1e-5 for sigma >= 1e-6 sigma_max".
//
// Scope: n <= kRefineMaxN (one CTA per gate; C in shared memory, packed upper triangle, for
// n <= 128, else in the gate's dead preconditioner / rotation-log scratch). Trigger: the smallest
// sigma^2 >= 1e-12 sigma_max^2 is below kRefineRatio^2 sigma_max^2 (config 2 at chi <= 128 never
// triggers; graded / noisy-MPO spectra do).
#include <cuda_runtime.h>

#include <atomic>

#include "eamps_internal.cuh"
#include "sort_tails.cuh"

namespace eamps {

namespace {

constexpr int RT = 256;
constexpr int kRefineMaxN = 256;
constexpr double kRefineRatio = 2e-4;      // QR / large regimes (config 2 chi <= 256: 6.9e-4 .. 8.6e-5 -> no)
constexpr double kRefineRatioAcc = 2e-3;   // small / medium regimes (config 2 chi = 16: 5.5e-3 -> no)
constexpr int kSmemPackedMaxN = 128;

__host__ __device__ inline int npow2_of(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// packed upper triangle (i <= j), row-major: offset of (i, j)
__device__ __forceinline__ int up_off(int i, int j, int n) { return i * n - ((i * (i - 1)) >> 1) + (j - i); }

size_t refine_smem(int n) {
  const int np2 = npow2_of(n);
  size_t s = (size_t)2 * 32 * 33 * sizeof(double2)   // GEMM staging
             + (size_t)np2 * 12 + 16 + RT * 8;        // sort keys | idx | tails scratch
  if (n <= kSmemPackedMaxN) s += (size_t)n * (n + 1) / 2 * sizeof(double2);
  return s + 64;
}

// One gate's refinement (one CTA; the body of k_refine).
__device__ void refine_gate(GateDesc& gd, uint8_t* slab, DevState* st, const float2* __restrict__ d_us,
                            int max_sweeps) {
  const int n = gd.n, m = gd.m, np = gd.n_pad, dd = st->d;
  double* gS = reinterpret_cast<double*>(slab + gd.ws_sig2);
  const int tid = threadIdx.x;
  extern __shared__ __align__(16) uint8_t sm[];
  double2* As = reinterpret_cast<double2*>(sm);                 // [32][33]
  double2* Bs = As + 32 * 33;                                    // [32][33]
  const int np2 = npow2_of(n);
  double* keys = reinterpret_cast<double*>(Bs + 32 * 33);
  int32_t* idx = reinterpret_cast<int32_t*>(keys + np2);
  double* part = reinterpret_cast<double*>(idx + np2 + (np2 & 1));
  double2* Cp = n <= kSmemPackedMaxN
                    ? reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(part + RT) + 15) & ~uintptr_t(15))
                    : reinterpret_cast<double2*>(slab + gd.ws_log);
  // ---- B = theta V with theta RECONTRACTED in FP64 from the complex64 site tensors and gate (the
  // exact inputs of both sides: the FP32 contraction output Theta' carries ~eps32 relative rounding
  // per entry, which alone moves a sigma at 2e-6 sigma_max by ~4e-5 -- measured on a config-4 MPO
  // gate); stored FP32 in the dead theta workspace (ld m), each column keeping its relative accuracy.
  //   X_a[s'][(t',c)] = sum_b B_i[a,s',b] B_{i+1}[b,t',c]
  //   theta[(a,s),(t,c)] = lambda_a sum_{s',t'} U[s d+t, s' d+t'] X_a[s'][(t',c)]   (contract.cu, E2)
  const BondEntry* bonds = reinterpret_cast<const BondEntry*>(slab + st->bonds_off);
  const SiteEntry* sites = reinterpret_cast<const SiteEntry*>(slab + st->sites_off);
  const float* lam = reinterpret_cast<const float*>(slab + bonds[gd.site].off);
  const float2* Bi = reinterpret_cast<const float2*>(slab + sites[gd.site].off);       // (chi_l, d, chi_m)
  const float2* Bj = reinterpret_cast<const float2*>(slab + sites[gd.site + 1].off);   // (chi_m, d, chi_r)
  const float2* U = d_us + (int64_t)gd.u_index * dd * dd * dd * dd;
  const int chl = gd.l, chm = gd.mid, chr = gd.r, d2 = dd * dd;
  const float2* V = reinterpret_cast<const float2*>(slab + gd.ws_V);
  float2* B = reinterpret_cast<float2*>(slab + gd.ws_theta);
  // 1 / |v_j| in FP64 (keys[] as scratch): the columns of an FP32-accumulated V (small / medium
  // regimes) drift from unit norm by ~1e-5 after 15 sweeps, which would scale eig(V^H G V) by the
  // same factor (Ostrowski); with unit columns the remaining non-orthogonality enters at second order
  for (int j = tid; j < n; j += RT) {
    const float2* vj = V + (int64_t)j * np;
    double dsum = 0.0;
    for (int k = 0; k < n; ++k) dsum += (double)vj[k].x * vj[k].x + (double)vj[k].y * vj[k].y;
    keys[j] = dsum > 0.0 ? 1.0 / sqrt(dsum) : 0.0;
  }
  double2* Xa = As;                     // d x n   (As | Bs: 2 x 32 x 33 double2 >= 2 d n for d n <= 1024)
  double2* Ta = As + dd * n;            // d x n
  __syncthreads();
  for (int a = 0; a < chl; ++a) {
    for (int x = tid; x < dd * n; x += RT) {
      const int sp = x / n, col = x % n, tp = col / chr, c = col % chr;
      const float2* bi = Bi + ((int64_t)a * dd + sp) * chm;
      double xr = 0.0, xi = 0.0;
      for (int b = 0; b < chm; ++b) {
        const float2 u = bi[b], v = Bj[((int64_t)b * dd + tp) * chr + c];
        xr = fma((double)u.x, (double)v.x, fma(-(double)u.y, (double)v.y, xr));
        xi = fma((double)u.x, (double)v.y, fma((double)u.y, (double)v.x, xi));
      }
      Xa[x] = make_double2(xr, xi);
    }
    __syncthreads();
    const double la = lam[a];
    for (int x = tid; x < dd * n; x += RT) {
      const int sr = x / n, col = x % n, t = col / chr, c = col % chr;
      double tr = 0.0, ti = 0.0;
      for (int sp = 0; sp < dd; ++sp)
        for (int tp = 0; tp < dd; ++tp) {
          const float2 u = U[(sr * dd + t) * d2 + sp * dd + tp];
          const double2 xv = Xa[sp * n + tp * chr + c];
          tr = fma((double)u.x, xv.x, fma(-(double)u.y, xv.y, tr));
          ti = fma((double)u.x, xv.y, fma((double)u.y, xv.x, ti));
        }
      Ta[x] = make_double2(la * tr, la * ti);
    }
    __syncthreads();
    for (int x = tid; x < dd * n; x += RT) {
      const int sr = x / n, j = x % n;
      const float2* vj = V + (int64_t)j * np;
      const double2* th = Ta + sr * n;
      double wr = 0.0, wi = 0.0;
      for (int k = 0; k < n; ++k) {
        const double2 t = th[k];
        const float2 v = vj[k];
        wr = fma(t.x, (double)v.x, fma(-t.y, (double)v.y, wr));
        wi = fma(t.x, (double)v.y, fma(t.y, (double)v.x, wi));
      }
      const double sc = keys[j];
      B[(int64_t)j * m + a * dd + sr] = make_float2((float)(sc * wr), (float)(sc * wi));
    }
    __syncthreads();
  }
  // ---- C = B^H B (FP64), packed upper triangle: 32 x 32 tiles (bi <= bj), rows in 32-chunks
  const int nt = (n + 31) / 32;
  const int ti = tid & 31, tj0 = (tid >> 5) * 4;       // thread: tile row ti, tile columns tj0..tj0+3
  for (int bi = 0; bi < nt; ++bi) {
    for (int bj = bi; bj < nt; ++bj) {
      double2 acc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = make_double2(0.0, 0.0);
      for (int r0 = 0; r0 < m; r0 += 32) {
        for (int x = tid; x < 32 * 32; x += RT) {
          const int rr = x & 31, cc = x >> 5;
          const int row = r0 + rr, ci = bi * 32 + cc, cj = bj * 32 + cc;
          const float2 a = (row < m && ci < n) ? B[(int64_t)ci * m + row] : make_float2(0.f, 0.f);
          const float2 b = (row < m && cj < n) ? B[(int64_t)cj * m + row] : make_float2(0.f, 0.f);
          As[cc * 33 + rr] = make_double2(a.x, a.y);
          Bs[cc * 33 + rr] = make_double2(b.x, b.y);
        }
        __syncthreads();
#pragma unroll 4
        for (int rr = 0; rr < 32; ++rr) {
          const double2 a = As[ti * 33 + rr];   // conj(a) b
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double2 b = Bs[(tj0 + u) * 33 + rr];
            acc[u].x = fma(a.x, b.x, fma(a.y, b.y, acc[u].x));
            acc[u].y = fma(a.x, b.y, fma(-a.y, b.x, acc[u].y));
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = bi * 32 + ti, j = bj * 32 + tj0 + u;
        if (i < n && j < n && i <= j) Cp[up_off(i, j, n)] = acc[u];
      }
    }
  }
  __syncthreads();
  // ---- cyclic two-sided Jacobi on the Hermitian C (FP64), tournament order: each round rotates
  // n/2 disjoint pairs; every 2x2 block (pair a rows, pair b columns) becomes J_a^H X J_b
  auto cld = [&](int i, int j) {
    const double2 v = Cp[up_off(min(i, j), max(i, j), n)];
    return i <= j ? v : make_double2(v.x, -v.y);
  };
  auto cst = [&](int i, int j, double2 v) {
    Cp[up_off(min(i, j), max(i, j), n)] = i <= j ? v : make_double2(v.x, -v.y);
  };
  const int neven = n + (n & 1);           // odd n: a phantom column (never rotated)
  const int half = neven / 2;
  __shared__ double4 rp[kRefineMaxN / 2];  // c, s, Re e, Im e
  __shared__ int2 rpq[kRefineMaxN / 2];
  __shared__ int s_rot;
  const double tol2 = 1e-24;               // (1e-12)^2: relative off-diagonal tolerance
  double cmax = 0.0;
  for (int j = 0; j < n; ++j) cmax = fmax(cmax, cld(j, j).x);
  const double tiny = cmax * 1e-30;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int rnd = 0; rnd < neven - 1; ++rnd) {
      for (int k = tid; k < half; k += RT) {
        auto pos = [&](int x) { return x == 0 ? 0 : ((x - 1 + rnd) % (neven - 1)) + 1; };
        int p = pos(k), q = pos(neven - 1 - k);
        if (p > q) { const int t = p; p = q; q = t; }
        double c = 1.0, s = 0.0, er = 1.0, ei = 0.0;
        if (q < n) {
          const double al = cld(p, p).x, be = cld(q, q).x;
          const double2 g = cld(p, q);
          const double g2 = g.x * g.x + g.y * g.y;
          if (fmin(al, be) > tiny && g2 > tol2 * al * be) {
            const double ag = sqrt(g2);
            er = g.x / ag;
            ei = g.y / ag;
            const double zeta = (be - al) / (2.0 * ag);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            c = 1.0 / sqrt(1.0 + t * t);
            s = c * t;
            // the pair's own block J^H X J is diagonal: (alpha - t|gamma|, beta + t|gamma|)
            cst(p, p, make_double2(al - t * ag, 0.0));
            cst(q, q, make_double2(be + t * ag, 0.0));
            cst(p, q, make_double2(0.0, 0.0));
            s_rot = 1;
          }
        }
        rp[k] = make_double4(c, s, er, ei);
        rpq[k] = make_int2(p, q);
      }
      __syncthreads();
      // off-diagonal 2x2 blocks (a < b): X = [[C_pa pb, C_pa qb], [C_qa pb, C_qa qb]] -> J_a^H X J_b,
      // J = [[c, s e], [-s conj(e), c]] acting on columns (p, q): (x, y) -> (c x - s conj(e) y, s e x + c y)
      const int nblk = half * (half - 1) / 2;
      for (int x = tid; x < nblk; x += RT) {
        int a = 0, rem = x;
        while (rem >= half - 1 - a) { rem -= half - 1 - a; ++a; }
        const int b = a + 1 + rem;
        const double4 Ja = rp[a], Jb = rp[b];
        if (Ja.y == 0.0 && Jb.y == 0.0) continue;
        const int2 ra = rpq[a], cb = rpq[b];
        // a phantom index (odd n) has no entries: read as 0, never stored (its J is the identity)
        const bool va = ra.y < n, vb = cb.y < n;
        const double2 z = make_double2(0.0, 0.0);
        double2 X00 = cld(ra.x, cb.x), X01 = vb ? cld(ra.x, cb.y) : z;
        double2 X10 = va ? cld(ra.y, cb.x) : z, X11 = (va && vb) ? cld(ra.y, cb.y) : z;
        if (Jb.y != 0.0) {   // columns (right factor J_b): (x, y) -> (c x - s conj(e) y, s x + c conj(e) y)
          auto colrot = [&](double2& u, double2& v) {
            const double2 ev = make_double2(Jb.z * v.x + Jb.w * v.y, Jb.z * v.y - Jb.w * v.x);   // conj(e) v
            const double2 nu = make_double2(Jb.x * u.x - Jb.y * ev.x, Jb.x * u.y - Jb.y * ev.y);
            const double2 nv = make_double2(Jb.y * u.x + Jb.x * ev.x, Jb.y * u.y + Jb.x * ev.y);
            u = nu;
            v = nv;
          };
          colrot(X00, X01);
          colrot(X10, X11);
        }
        if (Ja.y != 0.0) {   // rows (left factor J_a^H): (u, v) -> (c u - s e v, s u + c e v)
          auto rowrot = [&](double2& u, double2& v) {
            const double2 ev = make_double2(Ja.z * v.x - Ja.w * v.y, Ja.z * v.y + Ja.w * v.x);   // e v
            const double2 nu = make_double2(Ja.x * u.x - Ja.y * ev.x, Ja.x * u.y - Ja.y * ev.y);
            const double2 nv = make_double2(Ja.y * u.x + Ja.x * ev.x, Ja.y * u.y + Ja.x * ev.y);
            u = nu;
            v = nv;
          };
          rowrot(X00, X10);
          rowrot(X01, X11);
        }
        cst(ra.x, cb.x, X00);
        if (vb) cst(ra.x, cb.y, X01);
        if (va) cst(ra.y, cb.x, X10);
        if (va && vb) cst(ra.y, cb.y, X11);
      }
      __syncthreads();
    }
    if (!s_rot) break;
    __syncthreads();
  }
  // ---- sigma_j^2 = C_jj; sort descending (pi), FP64 tails: step a3 redone on the refined values
  for (int j = tid; j < np2; j += RT) {
    keys[j] = j < n ? fmax(cld(j, j).x, 0.0) : -1.0;
    idx[j] = j;
  }
  __syncthreads();
  cta_sort_desc(keys, idx, np2);
  int32_t* gP = reinterpret_cast<int32_t*>(slab + gd.ws_pi);
  for (int j = tid; j < n; j += RT) {
    gS[j] = keys[j];
    gP[j] = idx[j];
  }
  cta_tails(keys, n, reinterpret_cast<double*>(slab + gd.ws_T), part);
}


// The trigger, one warp per gate of the wave: the gates whose smallest sigma >= 1e-12 sigma_max is
// below the regime's ratio go to a compact list (count at list[0], gates from list[1]).
__global__ void k_refine_pick(const GateDesc* __restrict__ desc, const uint8_t* slab, int G, int32_t* list) {
  const int g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (g >= G) return;
  const GateDesc& gd = desc[g];
  const int n = gd.n;
  if (n > kRefineMaxN || n < 2) return;
  if (gd.eig == 1) return;   // eigen route: V not formed yet (its too-deep gates come as eig = 2, V complete)
  const double* gS = reinterpret_cast<const double*>(slab + gd.ws_sig2);   // sorted descending
  const double smax = gS[0];
  // the deepest sigma^2 >= 1e-12 sigma_max^2: the last j with gS[j] >= 1e-12 smax (sorted)
  double deep = smax;
  for (int j = lane; j < n; j += 32)
    if (gS[j] >= 1e-12 * smax) deep = fmin(deep, gS[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) deep = fmin(deep, __shfl_xor_sync(0xffffffffu, deep, o));
  // the regimes that accumulate V in FP32 (small 0, medium 2) lose relative accuracy earlier than
  // the preconditioned ones (QR 3, large 1: V = unit columns of the converged B = L)
  const double r = (gd.regime == 0 || gd.regime == 2) ? kRefineRatioAcc : kRefineRatio;
  if (lane == 0 && smax > 0.0 && deep < r * r * smax) list[1 + atomicAdd(&list[0], 1)] = g;
}

__global__ void __launch_bounds__(RT) k_refine(GateDesc* __restrict__ desc, uint8_t* slab, DevState* st,
                                               const int32_t* __restrict__ list, const float2* __restrict__ d_us,
                                               int max_sweeps) {
  const int cnt = list[0];
  for (int li = blockIdx.x; li < cnt; li += gridDim.x) {
    refine_gate(desc[list[1 + li]], slab, st, d_us, max_sweeps);
    __syncthreads();
  }
}
}  // namespace

size_t refine_scratch_bytes(int n) {
  return (n > kSmemPackedMaxN && n <= kRefineMaxN) ? (size_t)n * (n + 1) / 2 * sizeof(double2) : 0;
}

int launch_refine(GateDesc* d_desc, int G, int max_n, uint8_t* slab, DevState* st, const float2* d_us,
                  int32_t* d_list, cudaStream_t s) {
  if (G <= 0 || max_n < 2) return 0;
  // the wave may mix gates with C in shared memory (n <= 128) and in global memory (n <= 256)
  const int nn = max_n < kRefineMaxN ? max_n : kRefineMaxN;
  const size_t a = refine_smem(nn < kSmemPackedMaxN ? nn : kSmemPackedMaxN), b = refine_smem(nn);
  const size_t smem = a > b ? a : b;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr))
    cudaFuncSetAttribute(k_refine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)refine_smem(kSmemPackedMaxN));
  cudaMemsetAsync(d_list, 0, sizeof(int32_t), s);
  k_refine_pick<<<(G + 7) / 8, 256, 0, s>>>(d_desc, slab, G, d_list);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = G < sms ? G : sms;   // grid-stride over the compact list (most waves: none)
  k_refine<<<grid, RT, smem, s>>>(d_desc, slab, st, d_list, d_us, 16);
  return 2;
}

}  // namespace eamps
