// svd_medium.cu -- step a2 + a3 when theta fits one CTA's shared memory but theta AND V do not
// (e.g. the config-2 chi = 64 thetas, 128 x 128 complex64 = 128 KB each).
//
// Two one-CTA-per-theta kernels instead of a cluster: the rotations are data-independent of V,
// so V can be built afterwards from a log of the rotations.
//   k_svd_theta : the one-sided Jacobi of svd_small.cu on theta alone (theta in shared memory);
//                 every round's rotation per column pair goes to a log in the workspace as
//                 (t = s/c, arg e): 8 B per pair-round, ~0.7 MB per theta for 11 sweeps at n = 128.
//                 V only has to be a unitary product of (nearly) the same rotations: the replay
//                 recomputing c, s, e from (t, arg e) to 1 ulp does not affect sigma or the update.
//   k_svd_vrep  : V = I R_1 R_2 ... R_T replayed from the log in shared memory (the same circle
//                 order, identity rotations skipped), then sigma_j^2 = ||theta v_j||^2/||v_j||^2
//                 with theta streamed from the workspace in row tiles (FP64 products), V to
//                 global, bitonic sort, FP64 tails (jacobi_finish).
// The flops are those of the small kernel; the only extra traffic is the log (written once, read
// once), a few percent of the update's time.
#include <algorithm>

#include "jacobi_common.cuh"

namespace eamps {

namespace {

template <int GT>
__global__ void __launch_bounds__(1024) k_svd_theta(GateDesc* desc, const int32_t* __restrict__ list, uint8_t* slab,
                                                    DevState* st, int max_sweeps) {
  extern __shared__ __align__(16) uint8_t sm[];
  GateDesc& gd = desc[list[blockIdx.x]];
  const int m = gd.m, n = gd.n;
  float2* A = reinterpret_cast<float2*>(sm);
  __shared__ float s_wn[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float2* __restrict__ gth = reinterpret_cast<const float2*>(slab + gd.ws_theta);
  float2* lg = reinterpret_cast<float2*>(slab + gd.ws_log);
  float nrm = 0.f;
  for (int x = tid; x < m * n; x += blockDim.x) {
    float2 v = gth[x];
    A[x] = v;
    nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, nrm));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  if (lane == 0) s_wn[warp] = nrm;
  __syncthreads();
  float norm2 = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) norm2 += s_wn[w];
  const float skip = norm2 * 3.5527137e-15f;
  const float tol = fmaxf(7.62939453e-6f, 4.f * sqrtf((float)m) * 5.96046448e-8f);
  const int groups = blockDim.x / GT, gid = tid / GT, lgi = tid % GT;
  const int cap = min(max_sweeps, gd.log_sweeps);
  int sweep = 0;
  bool converged = (n < 2);
  for (; sweep < cap && !converged; ++sweep) {
    int any = 0;
    for (int rnd = 0; rnd < n - 1; ++rnd) {
      bool rot = false;
      float2* lrow = lg + ((size_t)sweep * (n - 1) + rnd) * (n / 2);
      for (int base = 0; base < n / 2; base += groups) {
        const int slot = base + gid;
        const bool active = slot < n / 2;
        int p = 0, q = 1;
        if (active) circle_pair_n(slot, rnd, n, p, q);
        float2* ap = A + (size_t)p * m;
        float2* aq = A + (size_t)q * m;
        float al = 0.f, be = 0.f, gr = 0.f, gi = 0.f;
        if (active) {
          for (int i = lgi; i < m; i += GT) {
            float2 x = ap[i], y = aq[i];
            al = fmaf(x.x, x.x, fmaf(x.y, x.y, al));
            be = fmaf(y.x, y.x, fmaf(y.y, y.y, be));
            gr = fmaf(x.x, y.x, fmaf(x.y, y.y, gr));
            gi = fmaf(x.x, y.y, fmaf(-x.y, y.x, gi));
          }
        }
#pragma unroll
        for (int o = GT / 2; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          gr += __shfl_xor_sync(0xffffffffu, gr, o);
          gi += __shfl_xor_sync(0xffffffffu, gi, o);
        }
        Rot R;
        const bool doit = active && jacobi_rot(al, be, gr, gi, skip, tol, R);
        // log (t = s/c, phase of e): 8 B per pair-round; identity rotations are logged as t = 0
        if (active && lgi == 0) lrow[slot] = make_float2(doit ? R.s / R.c : 0.f, atan2f(R.ei, R.er));
        if (doit) {
          rot = true;
          for (int i = lgi; i < m; i += GT) {
            float2 x = ap[i], y = aq[i];
            apply_rot(x, y, R);
            ap[i] = x;
            aq[i] = y;
          }
        }
      }
      any |= __syncthreads_or(rot);
    }
    converged = (any == 0);
  }
  if (!converged && tid == 0) atomicCAS(&st->led.error, 0, -6 /* MPS_E_NOCONV */);
  if (tid == 0) gd.sweeps = sweep;
}

template <int GT>
__global__ void __launch_bounds__(1024) k_svd_vrep(GateDesc* desc, const int32_t* __restrict__ list, uint8_t* slab,
                                                   DevState* st, int tile_rows) {
  extern __shared__ __align__(16) uint8_t sm[];
  const GateDesc& gd = desc[list[blockIdx.x]];
  const int m = gd.m, n = gd.n, S = gd.sweeps;
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  float2* V = reinterpret_cast<float2*>(sm);                       // n x n
  const int ldt = n + 1;                                            // padded: conflict-free tile stores
  float2* T = V + (size_t)n * n;                                    // tile_rows x n (row-major tile of theta)
  double* s2 = reinterpret_cast<double*>(T + (size_t)tile_rows * ldt);
  int32_t* six = reinterpret_cast<int32_t*>(s2 + npow2);
  double* part = reinterpret_cast<double*>(six + npow2 + (npow2 & 1));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int x = tid; x < n * n; x += blockDim.x) V[x] = make_float2((x / n) == (x % n) ? 1.f : 0.f, 0.f);
  __syncthreads();
  const float2* lg = reinterpret_cast<const float2*>(slab + gd.ws_log);
  const int groups = blockDim.x / GT, gid = tid / GT, lgi = tid % GT;
  for (int sw = 0; sw < S; ++sw) {
    for (int rnd = 0; rnd < n - 1; ++rnd) {
      const float2* lrow = lg + ((size_t)sw * (n - 1) + rnd) * (n / 2);
      for (int slot = gid; slot < n / 2; slot += groups) {
        const float2 r = lrow[slot];
        if (r.x == 0.f) continue;  // identity rotation (uniform within the group)
        int p, q;
        circle_pair_n(slot, rnd, n, p, q);
        Rot R;
        R.c = rsqrtf(1.f + r.x * r.x);
        R.s = R.c * r.x;
        sincosf(r.y, &R.ei, &R.er);
        float2* vp = V + (size_t)p * n;
        float2* vq = V + (size_t)q * n;
        for (int i = lgi; i < n; i += GT) {
          float2 x = vp[i], y = vq[i];
          apply_rot(x, y, R);
          vp[i] = x;
          vq[i] = y;
        }
      }
      __syncthreads();
    }
  }
  // Rayleigh quotient with theta streamed in row tiles: num_j = sum_i |(theta V)_ij|^2 in FP64
  const float2* __restrict__ gth = reinterpret_cast<const float2*>(slab + gd.ws_theta);  // m x n, ld m
  for (int j = tid; j < n; j += blockDim.x) s2[j] = 0.0;
  __syncthreads();
  for (int r0 = 0; r0 < m; r0 += tile_rows) {
    const int tr = min(tile_rows, m - r0);
    for (int x = tid; x < tr * n; x += blockDim.x) {
      int i = x % tr, k = x / tr;  // coalesced along the rows of each theta column
      T[(size_t)i * ldt + k] = gth[(size_t)k * m + r0 + i];
    }
    __syncthreads();
    for (int j = warp; j < n; j += nw) {
      const float2* vj = V + (size_t)j * n;
      double num = 0.0;
      for (int i = lane; i < tr; i += 32) {
        const float2* ti = T + (size_t)i * ldt;
        double wr = 0.0, wi = 0.0;
        for (int k = 0; k < n; ++k) {
          float2 a = ti[k];
          float2 v = vj[k];
          wr = fma((double)a.x, (double)v.x, fma(-(double)a.y, (double)v.y, wr));
          wi = fma((double)a.x, (double)v.y, fma((double)a.y, (double)v.x, wi));
        }
        num += wr * wr + wi * wi;
      }
      num = warp_sum_d32(num);
      if (lane == 0) s2[j] += num;
    }
    __syncthreads();
  }
  for (int j = warp; j < n; j += nw) {
    const float2* vj = V + (size_t)j * n;
    double den = 0.0;
    for (int k = lane; k < n; k += 32) den += (double)vj[k].x * vj[k].x + (double)vj[k].y * vj[k].y;
    den = warp_sum_d32(den);
    if (lane == 0) {
      double v = den > 0.0 ? s2[j] / den : 0.0;
      if (!isfinite(v)) atomicCAS(&st->led.error, 0, -7);
      s2[j] = v;
    }
  }
  __syncthreads();
  jacobi_finish(gd, slab, V, s2, six, part);
}

}  // namespace

size_t svd_theta_smem(int m, int n) { return (size_t)m * n * 8 + 64; }

size_t svd_vrep_smem(int n, int tile_rows) {
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  return (size_t)n * n * 8 + (size_t)tile_rows * (n + 1) * 8 + (size_t)npow2 * 12 + 16 + 1024 * 8;
}

bool svd_medium_fits(int m, int n) { return svd_theta_smem(m, n) <= 210 * 1024 && svd_vrep_smem(n, 8) <= 210 * 1024; }

int vrep_tile_rows(int m, int n) {
  int t = 64;
  while (t > 8 && svd_vrep_smem(n, t) > 210 * 1024) t >>= 1;
  return std::min(t, m);
}

void launch_svd_medium(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem_theta, size_t smem_vrep,
                       int tile_rows, int max_sweeps, int gt, int threads, uint8_t* slab, DevState* st, cudaStream_t s) {
  if (count <= 0) return;
  static bool attr_set = false;
  if (!attr_set) {
#define EAMPS_ATTR(GTV)                                                                                  \
  cudaFuncSetAttribute(k_svd_theta<GTV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);      \
  cudaFuncSetAttribute(k_svd_vrep<GTV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    EAMPS_ATTR(4) EAMPS_ATTR(8) EAMPS_ATTR(16) EAMPS_ATTR(32)
#undef EAMPS_ATTR
    attr_set = true;
  }
  switch (gt) {
#define EAMPS_CASE(GTV)                                                                                   \
  case GTV:                                                                                               \
    k_svd_theta<GTV><<<count, threads, smem_theta, s>>>(d_desc, d_list, slab, st, max_sweeps);           \
    k_svd_vrep<GTV><<<count, threads, smem_vrep, s>>>(d_desc, d_list, slab, st, tile_rows);              \
    break;
    EAMPS_CASE(4) EAMPS_CASE(8) EAMPS_CASE(16)
    default:
      k_svd_theta<32><<<count, threads, smem_theta, s>>>(d_desc, d_list, slab, st, max_sweeps);
      k_svd_vrep<32><<<count, threads, smem_vrep, s>>>(d_desc, d_list, slab, st, tile_rows);
#undef EAMPS_CASE
  }
}

}  // namespace eamps
