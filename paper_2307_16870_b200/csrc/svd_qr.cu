// svd_qr.cu -- step a2 for thetas with m >= n that fit one CTA's shared memory (config 2
// chi = 16 and 64, config 1 bulk gates): QR-preconditioned one-sided Jacobi, no V accumulation.
//
//   theta = Q R (Householder, FP32, in shared memory; Q is never formed)
//   B = R^H (n x n, lower triangular), one-sided Jacobi on B's columns: B W = U Sigma
//   => R = W Sigma U^H and theta = (Q W) Sigma U^H: the right singular vectors of theta are the
//      normalised converged columns of B, v_j = b_j / |b_j| (no V accumulation, no rotation log)
//   sigma_j^2 = |theta v_j|^2 / |v_j|^2 with the ORIGINAL theta (FP64 products): second order in
//   the error of v_j, so the FP32 QR's normwise backward error (~eps sigma_max) does not reach
//   the small singular values; the residual non-orthogonality of the v_j (the Jacobi tolerance)
//   is removed by the FP64-anchored polish (launch_spectrum_polish).
// The preconditioner cuts the sweeps (config 2 chi = 64: 12 -> 9, numpy check of the same
// tournament) and removes the V half of every round. PAPER.md:65 (M = U Lambda V^dagger, V^dagger
// right-normalised) and :114 ("performing its SVD"); SURVEY §8(a) a2.
#include <cstdlib>
#include <type_traits>

#include "jacobi_common.cuh"

namespace eamps {

namespace {

constexpr int QR_T = 512;          // threads per CTA (circle-method kernels)
// block-recursive kernels: one lane group of GT per two residents, n / 4 = R GT / 4 groups
template <int GT, int R, int PK>
__host__ __device__ constexpr int qr_threads() { return PK == 2 ? R * GT * GT / 4 : QR_T; }
constexpr int QR_TILE = 32;        // Rayleigh row tile

// gamma = b_p^H b_q over the group (bit-identical in every lane), then the rotation of the pair in
// registers and the cached-norm update alpha' = alpha - t|gamma|, beta' = beta + t|gamma|.
// With P + iQ = s e, U + iW = c e (e = gamma / |gamma|):
//   x' = c x - s conj(e) y:  Re x' = c Re x - P Re y - Q Im y,  Im x' = c Im x - P Im y + Q Re y
//   y' = s x + c conj(e) y:  Re y' = s Re x + U Re y + W Im y,  Im y' = s Im x + U Im y - W Re y
template <int GT, int R>
__device__ __forceinline__ void pair_step(ColRegs<GT, R>& X, ColRegs<GT, R>& Y, float& al, float& be, float skip,
                                          float tol2, int& rot) {
  float gr, gi;
  cross_planar(X, Y, gr, gi);
  group_sum2<GT>(gr, gi);
  Rot Rt;
  float tg;
  if (jacobi_rot_fast(al, be, gr, gi, skip, tol2, Rt, tg)) {
    rot = 1;
    rot_planar(X, Y, Rt);
    al -= tg;
    be += tg;
  }
}

// One-sided Jacobi sweeps over the n = R GT columns of B (ld m, m even) in the block-recursive
// resident/visitor ordering. Level s (s = n, n/2, ..., 4): the columns split into sets of s
// consecutive columns; in each set the first s/2 are residents, held two per lane group
// (s/4 groups per set), the last s/2 visitors. Round k (k < s/2): group li of the set meets
// visitor (2 li + k) mod (s/2) with both its residents in turn. Then every set splits in halves
// (residents, visitors) for the next level; the last level rotates the pairs (4g, 4g+1) (still
// in registers after level 4) and (4g+2, 4g+3). Every pair is rotated exactly once per sweep, n - 1 rounds of n/2 rotations, as in
// the circle method (a numpy model of both orderings on config 2 thetas: 9 sweeps each). Visitor
// parity alternates between rounds, so round k+1's visitor is idle in round k and is prefetched.
template <int GT, int R>
__device__ __forceinline__ void jacobi_block_recursive(float2* A, int m, int n, float* cn, float skip, float tol2,
                                                       int max_sweeps, int& sweep, bool& converged) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int gid = tid / GT, lg = tid % GT;
  const bool active = gid < n / 4;                  // whole warps (n/4 * GT is a multiple of 32)
  for (; sweep < max_sweeps && !converged; ++sweep) {
    for (int j = warp; j < n; j += nw) {
      float a = 0.f;
      for (int i = lane; i < n; i += 32) {
        const float2 v = A[(size_t)j * m + i];
        a = fmaf(v.x, v.x, fmaf(v.y, v.y, a));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) cn[j] = a;
    }
    __syncthreads();
    int rot = 0;
    for (int s = n; s >= 4; s >>= 1) {
      const int gps = s / 4, h = s / 2;
      const int li = gid % gps, base = (gid / gps) * s;
      ColRegs<GT, R> X1, X2, Y, Yn;
      float a1 = 0.f, a2 = 0.f, bY = 0.f, bn = 0.f;
      int v = base + h + 2 * li;                      // round 0 visitor (2 li < h)
      if (active) {
        X1.load(A + (size_t)(base + 2 * li) * m, lg);
        X2.load(A + (size_t)(base + 2 * li + 1) * m, lg);
        a1 = cn[base + 2 * li];
        a2 = cn[base + 2 * li + 1];
        Y.load(A + (size_t)v * m, lg);
        bY = cn[v];
      }
      // round k: rotate with Yc (visitor v), prefetch round k+1's visitor into Yp (ping-pong, h even)
      auto visit = [&](ColRegs<GT, R>& Yc, ColRegs<GT, R>& Yp, int k) {
        int vi = 2 * li + k + 1;                      // < 2h: (2 li + k + 1) mod h without a division
        if (vi >= h) vi -= h;
        const int vn = base + h + vi;
        if (active) {
          if (k + 1 < h) {
            Yp.load(A + (size_t)vn * m, lg);
            bn = cn[vn];
          }
          pair_step(X1, Yc, a1, bY, skip, tol2, rot);
          pair_step(X2, Yc, a2, bY, skip, tol2, rot);
          Yc.store(A + (size_t)v * m, lg);
          if (lg == 0) cn[v] = bY;
        }
        __syncthreads();
        bY = bn;
        v = vn;
      };
      for (int k = 0; k < h; k += 2) {
        visit(Y, Yn, k);
        visit(Yn, Y, k + 1);
      }
      if (active) {
        if (s == 4) pair_step(X1, X2, a1, a2, skip, tol2, rot);   // last level, first pair (4g, 4g+1)
        X1.store(A + (size_t)(base + 2 * li) * m, lg);
        X2.store(A + (size_t)(base + 2 * li + 1) * m, lg);
        if (lg == 0) {
          cn[base + 2 * li] = a1;
          cn[base + 2 * li + 1] = a2;
        }
      }
      __syncthreads();
    }
    if (active) {                                   // last level, second pair (4g+2, 4g+3)
      ColRegs<GT, R> Y, Z;
      const int c = 4 * gid + 2;
      Y.load(A + (size_t)c * m, lg);
      Z.load(A + (size_t)(c + 1) * m, lg);
      float a3 = cn[c], a4 = cn[c + 1];
      pair_step(Y, Z, a3, a4, skip, tol2, rot);
      Y.store(A + (size_t)c * m, lg);
      Z.store(A + (size_t)(c + 1) * m, lg);
    }
    converged = (__syncthreads_or(rot) == 0);
  }
}

// Element (r, c) of a pair-planar column-major matrix (ld m, m even): column c's row pair r/2 is
// the float4 (Re 2p, Re 2p+1, Im 2p, Im 2p+1).
__device__ __forceinline__ float2 pl_get(const float2* A, int m, int c, int r) {
  const float* f = reinterpret_cast<const float*>(A + (size_t)c * m) + (r >> 1) * 4 + (r & 1);
  return make_float2(f[0], f[2]);
}
__device__ __forceinline__ void pl_set(float2* A, int m, int c, int r, float2 v) {
  float* f = reinterpret_cast<float*>(A + (size_t)c * m) + (r >> 1) * 4 + (r & 1);
  f[0] = v.x;
  f[2] = v.y;
}

// B = L (n x n lower, ld n, FP32 interleaved) written by the Cholesky preconditioner
// (precond_large.cu: G = theta^H theta = L L^H in FP64) -> the CTA's pair-planar A (ld m; rows >= n
// are not read by the Jacobi). Returns |B|_F^2 = tr G = |theta|_F^2.
template <int NT>
__device__ float load_b_planar(const float2* __restrict__ Bg, float2* A, int m, int n, float* s_wn) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nh = n / 2;
  const float4* b4 = reinterpret_cast<const float4*>(Bg);
  float nrm = 0.f;
  for (int x = tid; x < n * nh; x += NT) {
    const int c = x / nh, p = x % nh;
    const float4 t = b4[(size_t)c * nh + p];        // (Re 2p, Im 2p, Re 2p+1, Im 2p+1) of column c
    reinterpret_cast<float4*>(A + (size_t)c * m)[p] = make_float4(t.x, t.z, t.y, t.w);
    nrm = fmaf(t.x, t.x, fmaf(t.y, t.y, fmaf(t.z, t.z, fmaf(t.w, t.w, nrm))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  if (lane == 0) s_wn[warp] = nrm;
  __syncthreads();
  float norm2 = 0.f;
  for (int w = 0; w < NT / 32; ++w) norm2 += s_wn[w];
  return norm2;
}

// Householder QR of theta (m x n, m >= n, m even) in shared memory, PAIR-PLANAR: theta is loaded
// as row pairs (Re 2p, Re 2p+1, Im 2p, Im 2p+1), so every dot product and rank-1 update below is a
// packed FP32x2 instruction on two rows (half the instructions of the interleaved version), then
// B = R^H is formed in place in the same layout (the Jacobi's layout). Same arithmetic as the
// interleaved path: reflector H = I - beta v v^H, v = x - alpha e_1, alpha = -(x0/|x0|) |x|,
// one barrier per reflector (the group of column j+1 publishes the next (|x|^2, x0) pair).
// Returns |theta|_F^2. Needs NT threads, s_wn >= NT / 32 floats.
template <int NT>
__device__ float householder_planar(const float2* __restrict__ gth, float2* A, int m, int n, float2* s_rdiag,
                                    float* s_wn, float* s_xn2, float2* s_x0) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mh = m / 2;
  const float4* g4 = reinterpret_cast<const float4*>(gth);
  float4* A4 = reinterpret_cast<float4*>(A);
  float nrm = 0.f;
  for (int x = tid; x < n * mh; x += NT) {
    const float4 t = g4[x];                        // (Re 2p, Im 2p, Re 2p+1, Im 2p+1)
    A4[x] = make_float4(t.x, t.z, t.y, t.w);
    nrm = fmaf(t.x, t.x, fmaf(t.y, t.y, fmaf(t.z, t.z, fmaf(t.w, t.w, nrm))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  if (lane == 0) s_wn[warp] = nrm;
  __syncthreads();
  float norm2 = 0.f;
  for (int w = 0; w < NT / 32; ++w) norm2 += s_wn[w];
  if (warp == 0) {
    float a = 0.f;
    for (int p = lane; p < mh; p += 32) {
      const float4 t = A4[p];
      a = fmaf(t.x, t.x, fmaf(t.y, t.y, fmaf(t.z, t.z, fmaf(t.w, t.w, a))));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) {
      s_xn2[0] = a;
      s_x0[0] = make_float2(A4[0].x, A4[0].z);
    }
  }
  __syncthreads();
  constexpr int QG = 8;                            // lanes per column
  const int qg = tid / QG, ql = tid % QG, ngr = NT / QG;
  for (int j = 0; j < n; ++j) {
    const float xn2 = s_xn2[j & 1];
    const float2 x0 = s_x0[j & 1];
    const float xn = sqrtf(xn2);
    const float ax0 = sqrtf(x0.x * x0.x + x0.y * x0.y);
    const float2 ph = ax0 > 0.f ? make_float2(x0.x / ax0, x0.y / ax0) : make_float2(1.f, 0.f);
    const float2 alpha = make_float2(-ph.x * xn, -ph.y * xn);
    const float2 v0 = make_float2(x0.x - alpha.x, x0.y - alpha.y);
    const float vn2 = xn2 - ax0 * ax0 + (v0.x * v0.x + v0.y * v0.y);
    const bool skipj = !(xn2 > 0.f) || !(vn2 > 0.f);
    const float beta = skipj ? 0.f : 2.f / vn2;
    if (tid == 0) s_rdiag[j] = skipj ? x0 : alpha;
    const float4* vj = A4 + (size_t)j * mh;
    const int pj = j >> 1;
    const bool odd = j & 1;
    // v on row pair p: column j's rows, with row j -> v0 and row j-1 (j odd) -> 0
    auto vpair = [&](int p) {
      float4 v = vj[p];
      if (p == pj) {
        if (odd) v = make_float4(0.f, v0.x, 0.f, v0.y);
        else v = make_float4(v0.x, v.y, v0.y, v.w);
      }
      return v;
    };
    for (int c0 = j + 1; c0 < n; c0 += ngr) {
      const int c = c0 + qg;
      float4* ac = A4 + (size_t)c * mh;
      float2 ar = make_float2(0.f, 0.f), ai = ar, ai2 = ar;
      if (c < n && !skipj) {
        for (int p = pj + ql; p < mh; p += QG) {
          const float4 v = vpair(p), a = ac[p];
          const float2 vr = make_float2(v.x, v.y), vi = make_float2(v.z, v.w);
          const float2 a_r = make_float2(a.x, a.y), a_i = make_float2(a.z, a.w);
          ar = f2_fma(vr, a_r, ar);                  // Re conj(v) a = vr ar + vi ai
          ar = f2_fma(vi, a_i, ar);
          ai = f2_fma(vr, a_i, ai);                  // Im conj(v) a = vr ai - vi ar
          ai2 = f2_fma(vi, a_r, ai2);
        }
      }
      float wr = ar.x + ar.y, wi = (ai.x + ai.y) - (ai2.x + ai2.y);
#pragma unroll
      for (int o = QG / 2; o > 0; o >>= 1) {
        wr += __shfl_xor_sync(0xffffffffu, wr, o);
        wi += __shfl_xor_sync(0xffffffffu, wi, o);
      }
      const bool nextc = (c == j + 1);
      float t2 = 0.f;
      auto tail2 = [&](int p, const float4& a) {     // |a|^2 over rows >= j+1 of the pair
        if (p == pj) return odd ? 0.f : fmaf(a.y, a.y, a.w * a.w);
        return fmaf(a.x, a.x, fmaf(a.y, a.y, fmaf(a.z, a.z, a.w * a.w)));
      };
      if (c < n && !skipj) {
        const float br = beta * wr, bi = beta * wi;
        const float2 mbr = make_float2(-br, -br), pbi = make_float2(bi, bi), mbi = make_float2(-bi, -bi);
        for (int p = pj + ql; p < mh; p += QG) {
          const float4 v = vpair(p), a = ac[p];
          const float2 vr = make_float2(v.x, v.y), vi = make_float2(v.z, v.w);
          float2 a_r = make_float2(a.x, a.y), a_i = make_float2(a.z, a.w);
          a_r = f2_fma(pbi, vi, f2_fma(mbr, vr, a_r));   // a -= (beta w) v
          a_i = f2_fma(mbi, vr, f2_fma(mbr, vi, a_i));
          const float4 an = make_float4(a_r.x, a_r.y, a_i.x, a_i.y);
          ac[p] = an;
          if (nextc) t2 += tail2(p, an);
        }
      } else if (c < n && nextc) {
        for (int p = pj + ql; p < mh; p += QG) t2 += tail2(p, ac[p]);
      }
      if (c0 == j + 1 && warp == 0) {                 // warp-uniform: holds the group of column j+1
#pragma unroll
        for (int o = QG / 2; o > 0; o >>= 1) t2 += __shfl_xor_sync(0xffffffffu, t2, o);
        __syncwarp();                                 // row j+1 was written by another lane
        if (qg == 0 && ql == 0) {
          s_xn2[(j + 1) & 1] = t2;
          s_x0[(j + 1) & 1] = pl_get(A, m, j + 1, j + 1);
        }
      }
    }
    __syncthreads();
  }
  // ---- B = R^H in place (top n x n block); rows >= n and R's lower part (the reflectors) -> 0
  for (int x = tid; x < n * m; x += NT) {
    const int c = x / m, r = x % m;
    if (r > c) pl_set(A, m, c, r, make_float2(0.f, 0.f));
  }
  __syncthreads();
  for (int x = tid; x < n * n; x += NT) {
    const int c = x / n, r = x % n;                  // R[r][c], r < c  ->  B[c][r] = conj(R[r][c])
    if (r < c) {
      const float2 v = pl_get(A, m, c, r);
      pl_set(A, m, r, c, make_float2(v.x, -v.y));
      pl_set(A, m, c, r, make_float2(0.f, 0.f));
    } else if (r == c) {
      const float2 d = s_rdiag[r];
      pl_set(A, m, r, r, make_float2(d.x, -d.y));
    }
  }
  __syncthreads();
  return norm2;
}

template <int GT, int R, int PK>
__global__ void __launch_bounds__(qr_threads<GT, R, PK>()) k_svd_qr(GateDesc* desc, const int32_t* __restrict__ list, uint8_t* slab,
                                                 DevState* st, int max_sweeps, float tol_min) {
  extern __shared__ __align__(16) uint8_t sm[];
  GateDesc& gd = desc[list[blockIdx.x]];
  const int m = gd.m, n = gd.n, half = n / 2;
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  float2* A = reinterpret_cast<float2*>(sm);                                  // m x n, ld m
  float2* T = A + (size_t)m * n;                                              // QR_TILE x (n+1)
  double* s2 = reinterpret_cast<double*>(T + (size_t)QR_TILE * (n + 1));
  int32_t* six = reinterpret_cast<int32_t*>(s2 + npow2);
  double* part = reinterpret_cast<double*>(six + npow2 + (npow2 & 1));       // QR_T doubles
  uint16_t* sched = reinterpret_cast<uint16_t*>(part + QR_T);                // (n-1) x n/2
  float* cn = reinterpret_cast<float*>(                                        // n cached |b_j|^2
      (reinterpret_cast<uintptr_t>(sched + (n - 1) * half) + 15) & ~uintptr_t(15));
  __shared__ float2 s_rdiag[256];                                             // R_jj
  __shared__ float s_wn[32];
  __shared__ float s_xn2[2];                                                  // by step parity
  __shared__ float2 s_x0[2];
  constexpr int NT = qr_threads<GT, R, PK>();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = NT / 32;
  const float2* __restrict__ gth = reinterpret_cast<const float2*>(slab + gd.ws_theta);
  build_circle_schedule(sched, n);
  float norm2 = 0.f;
  if constexpr (PK == 2) {
    // pair-planar Householder QR and B = R^H (householder_planar): packed FP32x2 row pairs
    if (gd.jrows > 0) norm2 = load_b_planar<NT>(reinterpret_cast<const float2*>(slab + gd.ws_theta), A, m, n, s_wn);
    else norm2 = householder_planar<NT>(gth, A, m, n, s_rdiag, s_wn, s_xn2, s_x0);
  } else if (gd.jrows > 0) {
    // B = L (= R^H) from the FP64 Gram + Cholesky preconditioner (precond_large.cu; n x n, ld n, in
    // the theta workspace) into the top n rows of A (ld m). An FP32 Householder R would carry a
    // normwise backward error ~eps32 sigma_max, i.e. no relative accuracy for sigma_j << sigma_max
    // (measured: 0.19 relative on a config-4 MPO theta with sigma_min ~1e-6 sigma_max); the FP64
    // Cholesky's error is ~eps64 kappa^2 instead.
    const float2* __restrict__ Bg = reinterpret_cast<const float2*>(slab + gd.ws_theta);
    float nrm = 0.f;
    for (int x = tid; x < m * n; x += NT) {
      const int c = x / m, r = x % m;
      const float2 v = r < n ? Bg[(size_t)c * n + r] : make_float2(0.f, 0.f);
      A[x] = v;
      nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, nrm));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if (lane == 0) s_wn[warp] = nrm;
    __syncthreads();
    for (int w = 0; w < nw; ++w) norm2 += s_wn[w];
  } else {
    float nrm = 0.f;
    for (int x = tid; x < m * n; x += NT) {
      const float2 v = gth[x];
      A[x] = v;
      nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, nrm));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    if (lane == 0) s_wn[warp] = nrm;
    __syncthreads();
    for (int w = 0; w < nw; ++w) norm2 += s_wn[w];
    // ---- Householder QR: column j's norm and leading entry come from the previous step
    if (warp == 0) {
      float a = 0.f;
      for (int i = lane; i < m; i += 32) a = fmaf(A[i].x, A[i].x, fmaf(A[i].y, A[i].y, a));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (lane == 0) {
        s_xn2[0] = a;
        s_x0[0] = A[0];
      }
    }
    __syncthreads();
    constexpr int QG = 8;                          // lanes per column in the update
    const int qg = tid / QG, ql = tid % QG, ngr = NT / QG;
    // One barrier per reflector: every thread derives the reflector from the (norm, leading entry)
    // pair the previous step left in s_xn2 / s_x0[j & 1] and keeps v_0 in a register (v's other
    // entries are column j's rows > j, which step j does not modify); the group of column j+1
    // publishes the next pair into the other parity slot. Q is never formed, so v_0 is not stored.
    for (int j = 0; j < n; ++j) {
      // reflector H = I - beta v v^H with v = x - alpha e_1, alpha = -(x0/|x0|) |x|
      const float xn2 = s_xn2[j & 1];
      const float2 x0 = s_x0[j & 1];
      const float xn = sqrtf(xn2);
      const float ax0 = sqrtf(x0.x * x0.x + x0.y * x0.y);
      const float2 ph = ax0 > 0.f ? make_float2(x0.x / ax0, x0.y / ax0) : make_float2(1.f, 0.f);
      const float2 alpha = make_float2(-ph.x * xn, -ph.y * xn);
      const float2 v0 = make_float2(x0.x - alpha.x, x0.y - alpha.y);
      const float vn2 = xn2 - ax0 * ax0 + (v0.x * v0.x + v0.y * v0.y);
      const bool skipj = !(xn2 > 0.f) || !(vn2 > 0.f);
      const float beta = skipj ? 0.f : 2.f / vn2;
      const float2* vj = A + (size_t)j * m;        // v: v0, then column j's rows j+1..m-1
      if (tid == 0) s_rdiag[j] = skipj ? x0 : alpha;
      // columns c > j: w = v^H a_c ; a_c -= beta w v ; the group of column j+1 also returns its new
      // tail norm and leading entry for the next reflector
      for (int c0 = j + 1; c0 < n; c0 += ngr) {
        const int c = c0 + qg;
        float2* ac = A + (size_t)c * m;
        float wr = 0.f, wi = 0.f;
        if (c < n && !skipj) {
          float wr1 = 0.f, wi1 = 0.f;              // two accumulator pairs (shorter FMA chains)
          int i = j + ql;
          for (; i + QG < m; i += 2 * QG) {
            const float2 v = i == j ? v0 : vj[i], a = ac[i];
            const float2 v1 = vj[i + QG], a1 = ac[i + QG];
            wr = fmaf(v.x, a.x, fmaf(v.y, a.y, wr));     // Re conj(v) a
            wi = fmaf(v.x, a.y, fmaf(-v.y, a.x, wi));    // Im conj(v) a
            wr1 = fmaf(v1.x, a1.x, fmaf(v1.y, a1.y, wr1));
            wi1 = fmaf(v1.x, a1.y, fmaf(-v1.y, a1.x, wi1));
          }
          if (i < m) {
            const float2 v = i == j ? v0 : vj[i], a = ac[i];
            wr = fmaf(v.x, a.x, fmaf(v.y, a.y, wr));
            wi = fmaf(v.x, a.y, fmaf(-v.y, a.x, wi));
          }
          wr += wr1;
          wi += wi1;
        }
#pragma unroll
        for (int o = QG / 2; o > 0; o >>= 1) {
          wr += __shfl_xor_sync(0xffffffffu, wr, o);
          wi += __shfl_xor_sync(0xffffffffu, wi, o);
        }
        float t2 = 0.f;
        if (c < n && !skipj) {
          const float br = beta * wr, bi = beta * wi;
          for (int i = j + ql; i < m; i += QG) {
            float2 a = ac[i];
            const float2 v = i == j ? v0 : vj[i];
            a.x -= br * v.x - bi * v.y;
            a.y -= br * v.y + bi * v.x;
            ac[i] = a;
            if (i > j) t2 = fmaf(a.x, a.x, fmaf(a.y, a.y, t2));
          }
        } else if (c < n) {
          for (int i = j + 1 + ql; i < m; i += QG) t2 = fmaf(ac[i].x, ac[i].x, fmaf(ac[i].y, ac[i].y, t2));
        }
        // only warp 0's first iteration holds the group of column j+1 (warp-uniform branch)
        if (c0 == j + 1 && warp == 0) {
#pragma unroll
          for (int o = QG / 2; o > 0; o >>= 1) t2 += __shfl_xor_sync(0xffffffffu, t2, o);
          __syncwarp();                            // row j+1 was written by another lane of the group
          if (qg == 0 && ql == 0) {
            s_xn2[(j + 1) & 1] = t2;
            s_x0[(j + 1) & 1] = ac[j + 1];
          }
        }
      }
      __syncthreads();
    }
    // ---- B = R^H in place (top n x n block, ld m); rows >= n and R's lower part (the reflectors) -> 0
    for (int x = tid; x < n * m; x += NT) {
      const int c = x / m, r = x % m;
      if (r > c) A[x] = make_float2(0.f, 0.f);
    }
    __syncthreads();
    for (int x = tid; x < n * n; x += NT) {
      const int c = x / n, r = x % n;               // R[r][c], r < c  ->  B[c][r] = conj(R[r][c])
      if (r < c) {
        const float2 v = A[(size_t)c * m + r];
        A[(size_t)r * m + c] = make_float2(v.x, -v.y);
        A[(size_t)c * m + r] = make_float2(0.f, 0.f);
      } else if (r == c) {
        const float2 d = s_rdiag[r];
        A[(size_t)r * m + r] = make_float2(d.x, -d.y);
      }
    }
    __syncthreads();
  }
  // ---- one-sided Jacobi on B's n columns of length n (ld m): registers, cached norms, schedule
  const float skip = norm2 * 3.5527137e-15f;
  const float tol = fmaxf(tol_min, 4.f * sqrtf((float)n) * 5.96046448e-8f);
  const float tol2 = tol * tol;
  const int gid = tid / GT, lgi = tid % GT;
  const int sh = gid & (32 / GT - 1);
  const bool active = gid < half;
  const bool full = (n == R * GT);
  int sweep = 0;
  bool converged = (n < 2);
  if constexpr (PK == 2) {
    // ---- block-recursive resident/visitor ordering (n = 4 * groups, a power of two): see
    // jacobi_block_recursive below. Two resident columns per lane group stay in registers while
    // the visitors stream through shared memory: one column load + one store per two rotations.
    (void)sched;
    jacobi_block_recursive<GT, R>(A, m, n, cn, skip, tol2, max_sweeps, sweep, converged);
    pair_planar(A, m, n);
    __syncthreads();
  } else {
    for (; sweep < max_sweeps && !converged; ++sweep) {
      for (int j = warp; j < n; j += nw) {
        float a = 0.f;
        for (int i = lane; i < n; i += 32) {
          const float2 v = A[(size_t)j * m + i];
          a = fmaf(v.x, v.x, fmaf(v.y, v.y, a));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) cn[j] = a;
      }
      __syncthreads();
      int any = 0;
      for (int rnd = 0; rnd < n - 1; ++rnd) {
        bool rot = false;
        // (a warp may hold active and idle groups: the shuffles run unconditionally)
        int p = 0, q = 1;
        float gr = 0.f, gi = 0.f;
        // PK: the columns fill the groups exactly (n = R GT, m even): 16-byte row pairs (PairRegs2)
        typename std::conditional<PK != 0, PairRegs2<GT, (R >= 2 ? R : 2)>, PairRegs<GT, R>>::type pr;
        if (active) {
          const uint32_t pq = sched[rnd * half + gid];
          p = pq & 0xFF;
          q = pq >> 8;
          if constexpr (PK != 0) {
            pr.load_full(A + (size_t)p * m, A + (size_t)q * m, lgi);
          } else {
            if (full) pr.load_full(A + (size_t)p * m, A + (size_t)q * m, lgi, sh);
            else pr.load(A + (size_t)p * m, A + (size_t)q * m, n, lgi, sh);
          }
          pr.cross(gr, gi);
        }
        group_sum2<GT>(gr, gi);
        if (active) {
          float2* ap = A + (size_t)p * m;
          float2* aq = A + (size_t)q * m;
          const float al = cn[p], be = cn[q];
          Rot Rt;
          float tg;
          if (jacobi_rot_fast(al, be, gr, gi, skip, tol2, Rt, tg)) {
            rot = true;
            if constexpr (PK != 0) {
              pr.rotate_store_full(ap, aq, lgi, Rt);
            } else {
              if (full) pr.rotate_store_full(ap, aq, lgi, sh, Rt);
              else pr.rotate_store(ap, aq, n, lgi, sh, Rt);
            }
            if (lgi == 0) {
              cn[p] = al - tg;
              cn[q] = be + tg;
            }
          }
        }
        any |= __syncthreads_or(rot);
      }
      converged = (any == 0);
    }
  }
  if (!converged && tid == 0) atomicCAS(&st->led.error, 0, -6 /* MPS_E_NOCONV */);
  if (tid == 0) gd.sweeps = sweep;
  // ---- V = B with unit columns (FP64 norms); V -> global (n x n, ld n)
  float2* gV = reinterpret_cast<float2*>(slab + gd.ws_V);
  for (int j = warp; j < n; j += nw) {
    float2* bj = A + (size_t)j * m;
    double a = 0.0;
    for (int i = lane; i < n; i += 32) a += (double)bj[i].x * bj[i].x + (double)bj[i].y * bj[i].y;
    a = warp_sum_d32(a);
    // a column at or below the rounding floor was never rotated (the Jacobi skips it), so its
    // direction is not orthogonal to the others: it carries no singular value (v_j = 0, sigma_j = 0)
    const float sc = a > (double)skip ? (float)(1.0 / sqrt(a)) : 0.f;
    for (int i = lane; i < n; i += 32) {
      const float2 v = make_float2(bj[i].x * sc, bj[i].y * sc);
      bj[i] = v;
      gV[(size_t)j * n + i] = v;
    }
  }
  // sigma_j^2 = |theta v_j|^2 / |v_j|^2 (FP64 products), the FP64-anchored polish and sort/tails run
  // in launch_spectrum_polish: the columns of V are orthonormal only to the Jacobi tolerance, which
  // lets a small sigma_j^2 pick up ~tol^2 sigma_l^2 from large ones; the polish removes exactly that
  (void)T;
  (void)s2;
  (void)six;
  (void)part;
}

template <int GT, int R, int PK>
void launch_qr_t(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem, int max_sweeps, uint8_t* slab,
                 DevState* st, cudaStream_t s) {
  static std::atomic<unsigned long long> attr_set{0};
  if (first_on_device(attr_set)) {
    cudaFuncSetAttribute(k_svd_qr<GT, R, PK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  }
  // Jacobi tolerance (relative |gamma| / sqrt(alpha beta)); EAMPS_QR_TOL overrides it for A/B runs
  static const float tol_min = getenv("EAMPS_QR_TOL") ? (float)atof(getenv("EAMPS_QR_TOL")) : 7.62939453e-6f;
  k_svd_qr<GT, R, PK><<<count, qr_threads<GT, R, PK>(), smem, s>>>(d_desc, d_list, slab, st, max_sweeps, tol_min);
}

}  // namespace

size_t svd_qr_smem(int m, int n) {
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  return (size_t)m * n * 8 + (size_t)QR_TILE * (n + 1) * 8 + (size_t)npow2 * 12 + 16 + QR_T * 8 +
         (size_t)(n - 1) * (n / 2) * 2 + 16 + (size_t)n * 4 + 64;
}

// QR path: m >= n, n <= 256, one pair per lane group with at most QR_T threads, rows per lane
// (n / GT) a power of two <= 16, the working set within one CTA's shared memory.
bool svd_qr_fits(int m, int n, int* gt_out, int* rpl_out) {
  // n < 64: the small kernel (theta and V in one CTA, one lane group per pair) is faster there
  if (m < n || n < 64 || n > 256 || (n & 1)) return false;
  int gt = 4;
  while (gt < 32 && (n / 2) * gt * 2 <= QR_T) gt <<= 1;   // widest group that still fits QR_T threads
  if ((n / 2) * gt > QR_T) return false;
  const int need = (n + gt - 1) / gt;
  int r = 1;
  while (r < need) r <<= 1;
  if (r > 16) return false;
  if (svd_qr_smem(m, n) > 220 * 1024) return false;
  *gt_out = gt;
  *rpl_out = r;
  return true;
}

// The block-recursive resident/visitor ordering (jacobi_block_recursive) applies to n = 64 and
// 128 with m even; EAMPS_QR_CIRCLE=1 keeps the circle method for A/B comparisons.
bool qr_block_order(int m, int n) {
  static const bool circle = getenv("EAMPS_QR_CIRCLE") != nullptr;
  return !circle && (n == 64 || n == 128) && m % 2 == 0;
}

void launch_svd_qr(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem, int max_sweeps, int gt, int rpl,
                   int packed, uint8_t* slab, DevState* st, cudaStream_t s) {
  if (count <= 0) return;
  if (packed == 2) {                                 // block-recursive ordering (qr_block_order)
    const int n = gt * rpl;
    static const bool g16 = getenv("EAMPS_QR_GT16") != nullptr;
    if (n == 128 && g16) return launch_qr_t<16, 8, 2>(d_desc, d_list, count, smem, max_sweeps, slab, st, s);
    if (n == 128) return launch_qr_t<8, 16, 2>(d_desc, d_list, count, smem, max_sweeps, slab, st, s);
    if (n == 64) return launch_qr_t<16, 4, 2>(d_desc, d_list, count, smem, max_sweeps, slab, st, s);
    return;
  }
#define EAMPS_QR(G, RR)                                                                              \
  if (gt == G && rpl == RR) {                                                                        \
    if (RR >= 2 && packed) return launch_qr_t<G, RR, 1>(d_desc, d_list, count, smem, max_sweeps, slab, st, s); \
    return launch_qr_t<G, RR, 0>(d_desc, d_list, count, smem, max_sweeps, slab, st, s);              \
  }
  EAMPS_QR(4, 16) EAMPS_QR(4, 8) EAMPS_QR(4, 4) EAMPS_QR(4, 2) EAMPS_QR(4, 1)
  EAMPS_QR(8, 16) EAMPS_QR(8, 8) EAMPS_QR(8, 4) EAMPS_QR(8, 2) EAMPS_QR(8, 1)
  EAMPS_QR(16, 16) EAMPS_QR(16, 8) EAMPS_QR(16, 4) EAMPS_QR(16, 2) EAMPS_QR(16, 1)
  EAMPS_QR(32, 8) EAMPS_QR(32, 4) EAMPS_QR(32, 2) EAMPS_QR(32, 1)
#undef EAMPS_QR
}

}  // namespace eamps
