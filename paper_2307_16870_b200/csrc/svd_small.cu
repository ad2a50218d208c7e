// svd_small.cu -- step a2 + a3 for thetas whose working set fits one CTA's shared memory
// ("small" regime of K3 in SURVEY §2.4).
//
// One-sided (Hestenes) Jacobi on the COLUMNS of theta (m x n), accumulating V (n x n), so that
// theta V = X Sigma and V = Y (the Hastings update needs V). PAPER.md:65:
// "M = U Lambda V^dagger ... U is left-normalized, while V^dagger is right-normalized".
//   * parallel (tournament / circle-method) ordering: n/2 disjoint column pairs per round,
//     n-1 rounds per sweep; one warp per pair, lanes over rows, warp-shuffle reductions for
//     alpha = |a_p|^2, beta = |a_q|^2, gamma = a_p^H a_q (the north-star's "warp-shuffle
//     column-pair reductions");
//   * the 2x2 rotation: e = gamma/|gamma|, zeta = (beta-alpha)/(2|gamma|),
//     t = sgn(zeta)/(|zeta| + sqrt(1+zeta^2)), c = 1/sqrt(1+t^2), s = c t,
//     (a_p, a_q) <- (c a_p - s conj(e) a_q, s a_p + c conj(e) a_q), same on (v_p, v_q);
//   * stop when a sweep rotates nothing (|gamma| <= tol sqrt(alpha beta));
//   * sigma_j^2 = ||theta v_j||^2 / ||v_j||^2 (Rayleigh quotient, FP64 products of the FP32
//     inputs): second-order accurate in the FP32 rounding of V, it removes the ~eps*sqrt(n*S)
//     norm drift that FP32 rotations accumulate;
//   * then the CTA sorts sigma^2 (bitonic) and writes the FP64 tail sums T (sort_tails.cuh).
#include "eamps_internal.cuh"
#include "sort_tails.cuh"

namespace eamps {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// pair (p, q) of slot i in round rnd of the circle method over n (even) players
__device__ __forceinline__ void circle_pair(int i, int rnd, int n, int& p, int& q) {
  auto pos = [&](int j) { return j == 0 ? 0 : ((j - 1 + rnd) % (n - 1)) + 1; };
  p = pos(i);
  q = pos(n - 1 - i);
}

__global__ void __launch_bounds__(kThreads) k_svd_small(GateDesc* desc, const int32_t* __restrict__ list,
                                                        uint8_t* slab, DevState* st, int max_sweeps) {
  extern __shared__ __align__(16) uint8_t sm[];
  GateDesc& gd = desc[list[blockIdx.x]];
  const int m = gd.m, n = gd.n;  // n even (n = d * chi_r)
  float2* A = reinterpret_cast<float2*>(sm);      // m x n, ld m
  float2* V = A + (size_t)m * n;                  // n x n, ld n
  __shared__ int s_rot;
  __shared__ float s_norm2;
  __shared__ double s_part[kThreads];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float2* __restrict__ gth = reinterpret_cast<const float2*>(slab + gd.ws_theta);

  float nrm = 0.f;
  for (int x = tid; x < m * n; x += kThreads) {
    float2 v = gth[x];
    A[x] = v;
    nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, nrm));
  }
  for (int x = tid; x < n * n; x += kThreads) V[x] = make_float2((x / n) == (x % n) ? 1.f : 0.f, 0.f);
  nrm = warp_sum(nrm);
  __shared__ float s_wn[kWarps];
  if (lane == 0) s_wn[warp] = nrm;
  __syncthreads();
  if (tid == 0) {
    float t = 0.f;
    for (int w = 0; w < kWarps; ++w) t += s_wn[w];  // fixed order: deterministic
    s_norm2 = t;
  }
  __syncthreads();
  // rounding floor for a column (SURVEY §8(c) item 3 with eps = 2^-24 on the GPU)
  const float skip = s_norm2 * 3.5527137e-15f;  // (2^-24)^2 ||theta||_F^2
  const float tol = fmaxf(7.62939453e-6f, 4.f * sqrtf((float)m) * 5.96046448e-8f);  // max(2^-17, 4 sqrt(m) 2^-24)

  int sweep = 0;
  bool converged = (n < 2);
  for (; sweep < max_sweeps && !converged; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int rnd = 0; rnd < n - 1; ++rnd) {
      for (int slot = warp; slot < n / 2; slot += kWarps) {
        int p, q;
        circle_pair(slot, rnd, n, p, q);
        float2* ap = A + (size_t)p * m;
        float2* aq = A + (size_t)q * m;
        float al = 0.f, be = 0.f, gr = 0.f, gi = 0.f;
        for (int i = lane; i < m; i += 32) {
          float2 x = ap[i], y = aq[i];
          al = fmaf(x.x, x.x, fmaf(x.y, x.y, al));
          be = fmaf(y.x, y.x, fmaf(y.y, y.y, be));
          gr = fmaf(x.x, y.x, fmaf(x.y, y.y, gr));    // Re conj(x) y
          gi = fmaf(x.x, y.y, fmaf(-x.y, y.x, gi));   // Im conj(x) y
        }
        al = warp_sum(al); be = warp_sum(be); gr = warp_sum(gr); gi = warp_sum(gi);
        if (fminf(al, be) <= skip) continue;
        float g = sqrtf(gr * gr + gi * gi);
        if (!(g > tol * sqrtf(al) * sqrtf(be))) continue;
        float er = gr / g, ei = gi / g;
        float zeta = (be - al) / (2.f * g);
        float az = fabsf(zeta);
        float hyp = az > 1.f ? az * sqrtf(1.f + 1.f / (az * az)) : sqrtf(1.f + az * az);
        float t = (zeta >= 0.f ? 1.f : -1.f) / (az + hyp);
        float c = rsqrtf(1.f + t * t);
        float s = c * t;
        // x' = c x - s conj(e) y ; y' = s x + c conj(e) y
        for (int i = lane; i < m; i += 32) {
          float2 x = ap[i], y = aq[i];
          float2 ey = make_float2(er * y.x + ei * y.y, er * y.y - ei * y.x);
          ap[i] = make_float2(c * x.x - s * ey.x, c * x.y - s * ey.y);
          aq[i] = make_float2(s * x.x + c * ey.x, s * x.y + c * ey.y);
        }
        float2* vp = V + (size_t)p * n;
        float2* vq = V + (size_t)q * n;
        for (int i = lane; i < n; i += 32) {
          float2 x = vp[i], y = vq[i];
          float2 ey = make_float2(er * y.x + ei * y.y, er * y.y - ei * y.x);
          vp[i] = make_float2(c * x.x - s * ey.x, c * x.y - s * ey.y);
          vq[i] = make_float2(s * x.x + c * ey.x, s * x.y + c * ey.y);
        }
        if (lane == 0) s_rot = 1;
      }
      __syncthreads();
    }
    converged = (s_rot == 0);
    __syncthreads();
  }
  if (!converged && tid == 0) atomicCAS(&st->led.error, 0, -6 /* MPS_E_NOCONV */);

  // Rayleigh quotient sigma_j^2 = ||theta v_j||^2 / ||v_j||^2 with FP64 products of FP32 data.
  for (int x = tid; x < m * n; x += kThreads) A[x] = gth[x];   // reload the original theta
  __syncthreads();
  double* s2 = reinterpret_cast<double*>(V + (size_t)n * n);   // [npow2]
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  int32_t* six = reinterpret_cast<int32_t*>(s2 + npow2);
  for (int j = warp; j < n; j += kWarps) {
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
    num = warp_sum_d(num);
    den = warp_sum_d(den);
    if (lane == 0) {
      double v = den > 0.0 ? num / den : 0.0;
      if (!isfinite(v)) atomicCAS(&st->led.error, 0, -7 /* MPS_E_NUMERIC */);
      s2[j] = v;
      six[j] = j;
    }
  }
  for (int j = n + tid; j < npow2; j += kThreads) { s2[j] = -1.0; six[j] = j; }
  // V to global (column-major, ld = n_pad == n in the small regime)
  float2* gV = reinterpret_cast<float2*>(slab + gd.ws_V);
  for (int x = tid; x < n * n; x += kThreads) gV[x] = V[x];
  __syncthreads();
  cta_sort_desc(s2, six, npow2);
  double* gS = reinterpret_cast<double*>(slab + gd.ws_sig2);
  int32_t* gP = reinterpret_cast<int32_t*>(slab + gd.ws_pi);
  for (int j = tid; j < n; j += kThreads) { gS[j] = s2[j]; gP[j] = six[j]; }
  cta_tails(s2, n, reinterpret_cast<double*>(slab + gd.ws_T), s_part);
  if (tid == 0) gd.sweeps = sweep;
}

}  // namespace

size_t svd_small_smem(int m, int n) {
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  return (size_t)m * n * 8 + (size_t)n * n * 8 + (size_t)npow2 * 12 + 64;
}

bool svd_small_fits(int m, int n) { return svd_small_smem(m, n) <= 200 * 1024; }

void launch_svd_small(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem, int max_sweeps,
                      uint8_t* slab, DevState* st, cudaStream_t s) {
  if (count <= 0) return;
  // smem = max over the bucket of svd_small_smem(m, n); every gate in the list fits
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_svd_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 4096);
    attr_set = true;
  }
  k_svd_small<<<count, kThreads, smem, s>>>(d_desc, d_list, slab, st, max_sweeps);
}

}  // namespace eamps
