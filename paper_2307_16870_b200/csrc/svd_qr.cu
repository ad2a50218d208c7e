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
#include <type_traits>

#include "jacobi_common.cuh"

namespace eamps {

namespace {

constexpr int QR_T = 512;          // threads per CTA
constexpr int QR_TILE = 32;        // Rayleigh row tile

template <int GT, int R, int PK>
__global__ void __launch_bounds__(QR_T) k_svd_qr(GateDesc* desc, const int32_t* __restrict__ list, uint8_t* slab,
                                                 DevState* st, int max_sweeps) {
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
  __shared__ float s_xn2, s_beta;
  __shared__ float2 s_x0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = QR_T / 32;
  const float2* __restrict__ gth = reinterpret_cast<const float2*>(slab + gd.ws_theta);
  float nrm = 0.f;
  for (int x = tid; x < m * n; x += QR_T) {
    const float2 v = gth[x];
    A[x] = v;
    nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, nrm));
  }
  build_circle_schedule(sched, n);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  if (lane == 0) s_wn[warp] = nrm;
  __syncthreads();
  float norm2 = 0.f;
  for (int w = 0; w < nw; ++w) norm2 += s_wn[w];
  // ---- Householder QR: column j's norm and leading entry come from the previous step
  if (warp == 0) {
    float a = 0.f;
    for (int i = lane; i < m; i += 32) a = fmaf(A[i].x, A[i].x, fmaf(A[i].y, A[i].y, a));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) {
      s_xn2 = a;
      s_x0 = A[0];
    }
  }
  __syncthreads();
  constexpr int QG = 8;                          // lanes per column in the update
  const int qg = tid / QG, ql = tid % QG, ngr = QR_T / QG;
  for (int j = 0; j < n; ++j) {
    // reflector H = I - beta v v^H with v = x - alpha e_1, alpha = -(x0/|x0|) |x|
    const float xn2 = s_xn2;
    const float2 x0 = s_x0;
    const float xn = sqrtf(xn2);
    const float ax0 = sqrtf(x0.x * x0.x + x0.y * x0.y);
    const float2 ph = ax0 > 0.f ? make_float2(x0.x / ax0, x0.y / ax0) : make_float2(1.f, 0.f);
    const float2 alpha = make_float2(-ph.x * xn, -ph.y * xn);
    const float2 v0 = make_float2(x0.x - alpha.x, x0.y - alpha.y);
    const float vn2 = xn2 - ax0 * ax0 + (v0.x * v0.x + v0.y * v0.y);
    const bool skipj = !(xn2 > 0.f) || !(vn2 > 0.f);
    const float beta = skipj ? 0.f : 2.f / vn2;
    float2* vj = A + (size_t)j * m;              // v lives in column j, rows j..m-1
    __syncthreads();                             // everyone has read s_xn2 / s_x0 / A[j][j]
    if (tid == 0) {
      s_rdiag[j] = skipj ? x0 : alpha;
      if (!skipj) vj[j] = v0;
    }
    __syncthreads();
    // columns c > j: w = v^H a_c ; a_c -= beta w v ; the group of column j+1 also returns its new
    // tail norm and leading entry for the next reflector
    for (int c0 = j + 1; c0 < n; c0 += ngr) {
      const int c = c0 + qg;
      float wr = 0.f, wi = 0.f;
      float2* ac = A + (size_t)c * m;
      if (c < n && !skipj) {
        for (int i = j + ql; i < m; i += QG) {
          const float2 v = vj[i], a = ac[i];
          wr = fmaf(v.x, a.x, fmaf(v.y, a.y, wr));     // Re conj(v) a
          wi = fmaf(v.x, a.y, fmaf(-v.y, a.x, wi));    // Im conj(v) a
        }
      }
#pragma unroll
      for (int o = QG / 2; o > 0; o >>= 1) {
        wr += __shfl_xor_sync(0xffffffffu, wr, o);
        wi += __shfl_xor_sync(0xffffffffu, wi, o);
      }
      float t2 = 0.f;
      if (c < n) {
        const float br = beta * wr, bi = beta * wi;
        for (int i = j + ql; i < m; i += QG) {
          float2 a = ac[i];
          if (!skipj) {
            const float2 v = vj[i];
            a.x -= br * v.x - bi * v.y;
            a.y -= br * v.y + bi * v.x;
            ac[i] = a;
          }
          if (c == j + 1 && i > j) t2 = fmaf(a.x, a.x, fmaf(a.y, a.y, t2));
        }
      }
      // (every lane takes part in the shuffle; only the group of column j+1 keeps the result)
#pragma unroll
      for (int o = QG / 2; o > 0; o >>= 1) t2 += __shfl_xor_sync(0xffffffffu, t2, o);
      if (c == j + 1 && ql == 0) {
        s_xn2 = t2;
        s_x0 = ac[j + 1];
      }
    }
    __syncthreads();
  }
  // ---- B = R^H in place (top n x n block, ld m); rows >= n and R's lower part (the reflectors) -> 0
  for (int x = tid; x < n * m; x += QR_T) {
    const int c = x / m, r = x % m;
    if (r > c) A[x] = make_float2(0.f, 0.f);
  }
  __syncthreads();
  for (int x = tid; x < n * n; x += QR_T) {
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
  // ---- one-sided Jacobi on B's n columns of length n (ld m): registers, cached norms, schedule
  const float skip = norm2 * 3.5527137e-15f;
  const float tol = fmaxf(7.62939453e-6f, 4.f * sqrtf((float)n) * 5.96046448e-8f);
  const float tol2 = tol * tol;
  const int gid = tid / GT, lgi = tid % GT;
  const int sh = gid & (32 / GT - 1);
  const bool active = gid < half;
  const bool full = (n == R * GT);
  int sweep = 0;
  bool converged = (n < 2);
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
  if (!converged && tid == 0) atomicCAS(&st->led.error, 0, -6 /* MPS_E_NOCONV */);
  if (tid == 0) gd.sweeps = sweep;
  // ---- V = B with unit columns (FP64 norms); V -> global (n x n, ld n)
  float2* gV = reinterpret_cast<float2*>(slab + gd.ws_V);
  for (int j = warp; j < n; j += nw) {
    float2* bj = A + (size_t)j * m;
    double a = 0.0;
    for (int i = lane; i < n; i += 32) a += (double)bj[i].x * bj[i].x + (double)bj[i].y * bj[i].y;
    a = warp_sum_d32(a);
    const float sc = a > 0.0 ? (float)(1.0 / sqrt(a)) : 0.f;
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
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_svd_qr<GT, R, PK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr_set = true;
  }
  k_svd_qr<GT, R, PK><<<count, QR_T, smem, s>>>(d_desc, d_list, slab, st, max_sweeps);
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

void launch_svd_qr(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem, int max_sweeps, int gt, int rpl,
                   int packed, uint8_t* slab, DevState* st, cudaStream_t s) {
  if (count <= 0) return;
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
