// jacobi_common.cuh -- pieces shared by the shared-memory Jacobi kernels (svd_small.cu,
// svd_medium.cu): the circle-method pairing, the 2x2 rotation, and the CTA epilogue
// (Rayleigh-quotient sigma^2 in FP64, V to global, bitonic sort, FP64 tails).
#pragma once
#include "eamps_internal.cuh"
#include "sort_tails.cuh"

namespace eamps {

// pair (p, q) of slot i in round rnd of the circle method over n (even) players
__device__ __forceinline__ void circle_pair_n(int i, int rnd, int n, int& p, int& q) {
  auto pos = [&](int j) { return j == 0 ? 0 : ((j - 1 + rnd) % (n - 1)) + 1; };
  p = pos(i);
  q = pos(n - 1 - i);
}

struct Rot {
  float c, s, er, ei;  // (a_p, a_q) <- (c a_p - s conj(e) a_q, s a_p + c conj(e) a_q)
};

// The 2x2 one-sided Jacobi rotation from alpha = |a_p|^2, beta = |a_q|^2, gamma = a_p^H a_q:
// e = gamma/|gamma|, zeta = (beta - alpha)/(2|gamma|), t = sgn(zeta)/(|zeta| + sqrt(1 + zeta^2)),
// c = 1/sqrt(1 + t^2), s = c t (SURVEY §8(c) algorithm item 3). Returns false (identity) when the
// pair is already orthogonal to tol or a column is below the rounding floor.
__device__ __forceinline__ bool jacobi_rot(float al, float be, float gr, float gi, float skip, float tol, Rot& R) {
  R.c = 1.f; R.s = 0.f; R.er = 1.f; R.ei = 0.f;
  if (fminf(al, be) <= skip) return false;
  const float g = sqrtf(gr * gr + gi * gi);
  if (!(g > tol * sqrtf(al) * sqrtf(be))) return false;
  R.er = gr / g;
  R.ei = gi / g;
  const float zeta = (be - al) / (2.f * g);
  const float az = fabsf(zeta);
  const float hyp = az > 1.f ? az * sqrtf(1.f + 1.f / (az * az)) : sqrtf(1.f + az * az);
  const float t = (zeta >= 0.f ? 1.f : -1.f) / (az + hyp);
  R.c = rsqrtf(1.f + t * t);
  R.s = R.c * t;
  return true;
}

// The same rotation with fast reciprocals (rsqrt / rcp.approx; sqrt(q) = q rsqrt(q)): e = gamma rsqrt(|gamma|^2), the
// criterion compared in squares; returns t |gamma| for the cached-norm update
// alpha' = alpha - t|gamma|, beta' = beta + t|gamma| (SURVEY §8(c) algorithm item 3, checked there
// in numpy). |e| and c^2 + s^2 are 1 to a few ulp.
__device__ __forceinline__ bool jacobi_rot_fast(float al, float be, float gr, float gi, float skip, float tol2, Rot& R,
                                                float& tg) {
  R.c = 1.f; R.s = 0.f; R.er = 1.f; R.ei = 0.f;
  tg = 0.f;
  const float g2 = fmaf(gr, gr, gi * gi);
  if (fminf(al, be) <= skip || !(g2 > tol2 * al * be)) return false;
  const float ig = rsqrtf(g2);
  R.er = gr * ig;
  R.ei = gi * ig;
  const float zeta = 0.5f * (be - al) * ig;
  const float az = fabsf(zeta);
  const float q = fmaf(az, az, 1.f);             // az <= sqrt(alpha / skip) / tol: no overflow
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(az + q * rsqrtf(q)));
  t = copysignf(t, zeta);
  R.c = rsqrtf(fmaf(t, t, 1.f));
  R.s = R.c * t;
  tg = t * (g2 * ig);
  return true;
}

// Packed FP32x2 arithmetic (Blackwell FFMA2 / FMUL2: one instruction for both halves of a complex
// number), used by the rotation -- the most frequent operation of every Jacobi kernel.
__device__ __forceinline__ uint64_t f2_pack(float2 a) { return *reinterpret_cast<uint64_t*>(&a); }
__device__ __forceinline__ float2 f2_unpack(uint64_t d) { return *reinterpret_cast<float2*>(&d); }
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)));
  return f2_unpack(d);
}
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_pack(a)), "l"(f2_pack(b)), "l"(f2_pack(c)));
  return f2_unpack(d);
}

// (x, y) <- (c x - s conj(e) y, s x + c conj(e) y):
//   conj(e) y = (er, er) * (y.re, y.im) + (ei, -ei) * (y.im, y.re)
__device__ __forceinline__ void apply_rot(float2& x, float2& y, const Rot& R) {
  const float2 ey = f2_fma(make_float2(R.ei, -R.ei), make_float2(y.y, y.x), f2_mul(make_float2(R.er, R.er), y));
  const float2 nx = f2_fma(make_float2(-R.s, -R.s), ey, f2_mul(make_float2(R.c, R.c), x));
  const float2 ny = f2_fma(make_float2(R.c, R.c), ey, f2_mul(make_float2(R.s, R.s), x));
  x = nx;
  y = ny;
}

// The rows of a column pair held in registers between the dot products and the rotation: lane
// lg of a GT-lane group owns rows lg, lg + GT, ..., lg + (R-1) GT (R = rows per lane, a compile-time
// bound; the caller guarantees m <= R GT). One shared-memory read and one write per element per
// round instead of two reads and one write.
template <int GT, int R>
struct PairRegs {
  float2 x[R], y[R];
  // row of register slot u for lane lg: lg + GT ((u + sh) mod R), sh = the group's index within its
  // warp, so the groups of a warp hit different shared-memory banks (2 wavefronts per float2 access)
  static __device__ __forceinline__ int row(int lg, int u, int sh) { return lg + GT * ((u + sh) & (R - 1)); }
  __device__ __forceinline__ void load(const float2* ap, const float2* aq, int m, int lg, int sh) {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int i = row(lg, u, sh);
      const bool ok = i < m;
      x[u] = ok ? ap[i] : make_float2(0.f, 0.f);
      y[u] = ok ? aq[i] : make_float2(0.f, 0.f);
    }
  }
  __device__ __forceinline__ void load_full(const float2* ap, const float2* aq, int lg, int sh) {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int i = row(lg, u, sh);
      x[u] = ap[i];
      y[u] = aq[i];
    }
  }
  __device__ __forceinline__ void cross(float& gr, float& gi) const {   // gamma = a_p^H a_q only
    // (a.re, a.re) (b.re, b.im) + (a.im, -a.im) (b.im, b.re), two packed accumulators
    float2 acc1 = make_float2(0.f, 0.f), acc2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const float2 a = x[u], b = y[u];
      acc1 = f2_fma(make_float2(a.x, a.x), b, acc1);
      acc2 = f2_fma(make_float2(a.y, -a.y), make_float2(b.y, b.x), acc2);
    }
    gr += acc1.x + acc2.x;
    gi += acc1.y + acc2.y;
  }
  __device__ __forceinline__ void dots(float& al, float& be, float& gr, float& gi) const {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const float2 a = x[u], b = y[u];
      al = fmaf(a.x, a.x, fmaf(a.y, a.y, al));
      be = fmaf(b.x, b.x, fmaf(b.y, b.y, be));
      gr = fmaf(a.x, b.x, fmaf(a.y, b.y, gr));    // Re conj(a) b
      gi = fmaf(a.x, b.y, fmaf(-a.y, b.x, gi));   // Im conj(a) b
    }
  }
  __device__ __forceinline__ void rotate_store(float2* ap, float2* aq, int m, int lg, int sh, const Rot& Rt) {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int i = row(lg, u, sh);
      if (i < m) {
        float2 a = x[u], b = y[u];
        apply_rot(a, b, Rt);
        ap[i] = a;
        aq[i] = b;
      }
    }
  }
  __device__ __forceinline__ void rotate_store_full(float2* ap, float2* aq, int lg, int sh, const Rot& Rt) {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int i = row(lg, u, sh);
      float2 a = x[u], b = y[u];
      apply_rot(a, b, Rt);
      ap[i] = a;
      aq[i] = b;
    }
  }
};

template <int GT>
__device__ __forceinline__ void group_sum2(float& a, float& b) {
#pragma unroll
  for (int o = GT / 2; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
}

// One column of B in a lane group's registers, PAIR-PLANAR: shared memory holds each column as
// float4 (Re b_2i, Re b_2i+1, Im b_2i, Im b_2i+1) (pair_planar below), lane lg owns row pairs
// i = lg + GT v, v < R / 2, and keeps re[v] = (Re b_2i, Re b_2i+1), im[v] = (Im b_2i, Im b_2i+1):
// every complex operation below is a packed FP32x2 instruction on two rows with broadcast scalar
// coefficients -- no (re, im) swaps or negations to build operand pairs (15% of the instructions
// with the interleaved layout, ncu).
template <int GT, int R>
struct ColRegs {
  float2 re[R / 2], im[R / 2];
  __device__ __forceinline__ void load(const float2* a, int lg) {
#pragma unroll
    for (int v = 0; v < R / 2; ++v) {
      const float4 t = *reinterpret_cast<const float4*>(a + 2 * (lg + GT * v));
      re[v] = make_float2(t.x, t.y);
      im[v] = make_float2(t.z, t.w);
    }
  }
  __device__ __forceinline__ void store(float2* a, int lg) const {
#pragma unroll
    for (int v = 0; v < R / 2; ++v)
      *reinterpret_cast<float4*>(a + 2 * (lg + GT * v)) = make_float4(re[v].x, re[v].y, im[v].x, im[v].y);
  }
};

// in-place layout change of B's n columns (ld m) between interleaved float2 rows and pair-planar
// float4 (Re 2i, Re 2i+1, Im 2i, Im 2i+1); the permutation is its own inverse
__device__ __forceinline__ void pair_planar(float2* A, int m, int n) {
  for (int x = threadIdx.x; x < n * (n / 2); x += blockDim.x) {
    float4* q = reinterpret_cast<float4*>(A + (size_t)(x / (n / 2)) * m) + x % (n / 2);
    const float4 t = *q;
    *q = make_float4(t.x, t.z, t.y, t.w);
  }
}

__device__ __forceinline__ float2 f2s(float a) { return make_float2(a, a); }

// gamma = x^H y of two pair-planar columns over the lane's rows (not yet reduced over the group)
template <int GT, int R>
__device__ __forceinline__ void cross_planar(const ColRegs<GT, R>& X, const ColRegs<GT, R>& Y, float& gr, float& gi) {
  float2 a1 = make_float2(0.f, 0.f), a2 = a1, a3 = a1, a4 = a1;
#pragma unroll
  for (int v = 0; v < R / 2; ++v) {
    a1 = f2_fma(X.re[v], Y.re[v], a1);     // Re conj(x) y = xr yr + xi yi
    a2 = f2_fma(X.im[v], Y.im[v], a2);
    a3 = f2_fma(X.re[v], Y.im[v], a3);     // Im conj(x) y = xr yi - xi yr
    a4 = f2_fma(X.im[v], Y.re[v], a4);
  }
  gr = (a1.x + a1.y) + (a2.x + a2.y);
  gi = (a3.x + a3.y) - (a4.x + a4.y);
}

// The rotation of a pair-planar column pair. With P + iQ = s e, U + iW = c e (e = gamma / |gamma|):
//   x' = c x - s conj(e) y:  Re x' = c Re x - P Re y - Q Im y,  Im x' = c Im x - P Im y + Q Re y
//   y' = s x + c conj(e) y:  Re y' = s Re x + U Re y + W Im y,  Im y' = s Im x + U Im y - W Re y
template <int GT, int R>
__device__ __forceinline__ void rot_planar(ColRegs<GT, R>& X, ColRegs<GT, R>& Y, const Rot& Rt) {
  const float P = Rt.s * Rt.er, Q = Rt.s * Rt.ei, U = Rt.c * Rt.er, W = Rt.c * Rt.ei;
  const float2 c2 = f2s(Rt.c), s2 = f2s(Rt.s), mP = f2s(-P), mQ = f2s(-Q), pQ = f2s(Q), U2 = f2s(U), W2 = f2s(W),
               mW = f2s(-W);
#pragma unroll
  for (int v = 0; v < R / 2; ++v) {
    const float2 xr = X.re[v], xi = X.im[v], yr = Y.re[v], yi = Y.im[v];
    X.re[v] = f2_fma(mQ, yi, f2_fma(mP, yr, f2_mul(c2, xr)));
    X.im[v] = f2_fma(pQ, yr, f2_fma(mP, yi, f2_mul(c2, xi)));
    Y.re[v] = f2_fma(W2, yi, f2_fma(U2, yr, f2_mul(s2, xr)));
    Y.im[v] = f2_fma(mW, yr, f2_fma(U2, yi, f2_mul(s2, xi)));
  }
}

// As PairRegs, but each register slot holds two consecutive rows loaded/stored as one 16-byte
// access: lane lg owns rows 2 (lg + GT v) and 2 (lg + GT v) + 1, v < R/2 (the caller guarantees
// rows == R GT, rows even). Half the shared-memory instructions of PairRegs; a warp's groups read
// 128 contiguous bytes each (the minimum number of wavefronts).
template <int GT, int R>
struct PairRegs2 {
  float2 x[R], y[R];
  __device__ __forceinline__ void load_full(const float2* ap, const float2* aq, int lg) {
#pragma unroll
    for (int v = 0; v < R / 2; ++v) {
      const int i = 2 * (lg + GT * v);
      const float4 a = *reinterpret_cast<const float4*>(ap + i);
      const float4 b = *reinterpret_cast<const float4*>(aq + i);
      x[2 * v] = make_float2(a.x, a.y);
      x[2 * v + 1] = make_float2(a.z, a.w);
      y[2 * v] = make_float2(b.x, b.y);
      y[2 * v + 1] = make_float2(b.z, b.w);
    }
  }
  __device__ __forceinline__ void cross(float& gr, float& gi) const {
    float2 acc1 = make_float2(0.f, 0.f), acc2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const float2 a = x[u], b = y[u];
      acc1 = f2_fma(make_float2(a.x, a.x), b, acc1);
      acc2 = f2_fma(make_float2(a.y, -a.y), make_float2(b.y, b.x), acc2);
    }
    gr += acc1.x + acc2.x;
    gi += acc1.y + acc2.y;
  }
  __device__ __forceinline__ void rotate_store_full(float2* ap, float2* aq, int lg, const Rot& Rt) {
#pragma unroll
    for (int v = 0; v < R / 2; ++v) {
      const int i = 2 * (lg + GT * v);
      float2 a0 = x[2 * v], b0 = y[2 * v], a1 = x[2 * v + 1], b1 = y[2 * v + 1];
      apply_rot(a0, b0, Rt);
      apply_rot(a1, b1, Rt);
      *reinterpret_cast<float4*>(ap + i) = make_float4(a0.x, a0.y, a1.x, a1.y);
      *reinterpret_cast<float4*>(aq + i) = make_float4(b0.x, b0.y, b1.x, b1.y);
    }
  }
};

// GT-lane xor-butterfly sum of the four pair statistics (bit-identical in every lane of the group)
template <int GT>
__device__ __forceinline__ void group_sum4(float& al, float& be, float& gr, float& gi) {
#pragma unroll
  for (int o = GT / 2; o > 0; o >>= 1) {
    al += __shfl_xor_sync(0xffffffffu, al, o);
    be += __shfl_xor_sync(0xffffffffu, be, o);
    gr += __shfl_xor_sync(0xffffffffu, gr, o);
    gi += __shfl_xor_sync(0xffffffffu, gi, o);
  }
}

// The circle-method schedule of one sweep, (p | q << 8) per (round, slot), in shared memory (n <= 256)
__device__ __forceinline__ void build_circle_schedule(uint16_t* sched, int n) {
  const int half = n / 2;
  for (int x = threadIdx.x; x < (n - 1) * half; x += blockDim.x) {
    const int rnd = x / half, slot = x % half;
    int p, q;
    circle_pair_n(slot, rnd, n, p, q);
    sched[x] = (uint16_t)(p | (q << 8));
  }
}

__device__ __forceinline__ double warp_sum_d32(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ inline void jacobi_finish(const GateDesc& gd, uint8_t* slab, const float2* V, double* s2, int32_t* six,
                                     double* part);

// Epilogue: A (m x n, ld m, shared) must hold the ORIGINAL theta, V (n x n, ld n, shared) the
// accumulated rotations. sigma_j^2 = ||theta v_j||^2 / ||v_j||^2 with FP64 products of the FP32
// inputs (second order in V's rounding); V -> global (ld n); sort (sigma^2,
// index) descending; tails T in FP64. `s2`/`six` are npow2-long shared scratch, `part` has
// blockDim.x doubles.
__device__ inline void jacobi_epilogue(const GateDesc& gd, uint8_t* slab, DevState* st, const float2* A,
                                       const float2* V, double* s2, int32_t* six, double* part) {
  const int m = gd.m, n = gd.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  for (int j = warp; j < n; j += nw) {
    const float2* vj = V + (size_t)j * n;
    double num = 0.0;
    for (int i = lane; i < m; i += 32) {
      double wr = 0.0, wi = 0.0;
      for (int k = 0; k < n; ++k) {
        float2 a = A[(size_t)k * m + i];
        float2 v = vj[k];
        wr = fma((double)a.x, (double)v.x, fma(-(double)a.y, (double)v.y, wr));
        wi = fma((double)a.x, (double)v.y, fma((double)a.y, (double)v.x, wi));
      }
      num += wr * wr + wi * wi;
    }
    double den = 0.0;
    for (int k = lane; k < n; k += 32) den += (double)vj[k].x * vj[k].x + (double)vj[k].y * vj[k].y;
    num = warp_sum_d32(num);
    den = warp_sum_d32(den);
    if (lane == 0) {
      double v = den > 0.0 ? num / den : 0.0;
      if (!isfinite(v)) atomicCAS(&st->led.error, 0, -7 /* MPS_E_NUMERIC */);
      s2[j] = v;
    }
  }
  __syncthreads();
  jacobi_finish(gd, slab, V, s2, six, part);
}

// Shared tail of the epilogues: s2[j] = sigma_j^2 (j < n) already in shared memory.
__device__ inline void jacobi_finish(const GateDesc& gd, uint8_t* slab, const float2* V, double* s2, int32_t* six,
                                     double* part) {
  const int n = gd.n, tid = threadIdx.x;
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  for (int j = tid; j < n; j += blockDim.x) six[j] = j;
  for (int j = n + tid; j < npow2; j += blockDim.x) { s2[j] = -1.0; six[j] = j; }
  float2* gV = reinterpret_cast<float2*>(slab + gd.ws_V);
  for (int x = tid; x < n * n; x += blockDim.x) gV[x] = V[x];
  __syncthreads();
  cta_sort_desc(s2, six, npow2);
  double* gS = reinterpret_cast<double*>(slab + gd.ws_sig2);
  int32_t* gP = reinterpret_cast<int32_t*>(slab + gd.ws_pi);
  for (int j = tid; j < n; j += blockDim.x) { gS[j] = s2[j]; gP[j] = six[j]; }
  cta_tails(s2, n, reinterpret_cast<double*>(slab + gd.ws_T), part);
}

}  // namespace eamps
