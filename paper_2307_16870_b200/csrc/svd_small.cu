// svd_small.cu -- step a2 + a3 for thetas whose working set (theta AND V) fits one CTA's shared
// memory ("small" regime of K3 in SURVEY §2.4).
//
// One-sided (Hestenes) Jacobi on the COLUMNS of theta (m x n), accumulating V (n x n), so that
// theta V = X Sigma and V = Y (the Hastings update needs V). PAPER.md:65:
// "M = U Lambda V^dagger ... U is left-normalized, while V^dagger is right-normalized".
//   * parallel (tournament / circle-method) ordering: n/2 disjoint column pairs per round,
//     n-1 rounds per sweep; a group of GT lanes per pair (GT = 4..32 picked from m), rows split
//     over the group, xor-butterfly shuffle reductions of alpha = |a_p|^2, beta = |a_q|^2,
//     gamma = a_p^H a_q (bit-identical in every lane of the group, so the branch is uniform);
//   * the 2x2 rotation of jacobi_common.cuh; stop when a sweep rotates nothing
//     (|gamma| <= tol sqrt(alpha beta)); one __syncthreads_or per round;
//   * epilogue: Rayleigh-quotient sigma^2 (FP64 products), V to global, bitonic sort, FP64 tails.
#include "jacobi_common.cuh"

namespace eamps {

namespace {

// One round for all pairs. Returns (to the calling thread) whether it rotated something.
// R > 0: the pair's rows (m <= R GT) and V rows (n <= R GT) are register-resident across the dot
// products and the rotation; R = 0: the generic two-pass loop (tall or wide thetas).
template <int GT, int R>
__device__ __forceinline__ bool round_pairs(float2* A, int m, int n, float2* V, int rnd, float skip, float tol) {
  const int tid = threadIdx.x;
  const int groups = blockDim.x / GT, gid = tid / GT, lg = tid % GT;
  const int sh = gid & (32 / GT - 1);   // group index within the warp (bank spreading)
  bool rot = false;
  for (int base = 0; base < n / 2; base += groups) {
    const int slot = base + gid;
    const bool active = slot < n / 2;
    int p = 0, q = 1;
    if (active) circle_pair_n(slot, rnd, n, p, q);
    float2* ap = A + (size_t)p * m;
    float2* aq = A + (size_t)q * m;
    float al = 0.f, be = 0.f, gr = 0.f, gi = 0.f;
    if constexpr (R > 0) {
      PairRegs<GT, R> pr;
      if (active) {
        pr.load(ap, aq, m, lg, sh);
        pr.dots(al, be, gr, gi);
      }
      group_sum4<GT>(al, be, gr, gi);
      Rot Rt;
      if (active && jacobi_rot(al, be, gr, gi, skip, tol, Rt)) {
        rot = true;
        pr.rotate_store(ap, aq, m, lg, sh, Rt);
        PairRegs<GT, R> pv;
        float2* vp = V + (size_t)p * n;
        float2* vq = V + (size_t)q * n;
        pv.load(vp, vq, n, lg, sh);
        pv.rotate_store(vp, vq, n, lg, sh, Rt);
      }
    } else {
      if (active) {
        for (int i = lg; i < m; i += GT) {
          float2 x = ap[i], y = aq[i];
          al = fmaf(x.x, x.x, fmaf(x.y, x.y, al));
          be = fmaf(y.x, y.x, fmaf(y.y, y.y, be));
          gr = fmaf(x.x, y.x, fmaf(x.y, y.y, gr));    // Re conj(x) y
          gi = fmaf(x.x, y.y, fmaf(-x.y, y.x, gi));   // Im conj(x) y
        }
      }
      group_sum4<GT>(al, be, gr, gi);
      Rot Rt;
      if (active && jacobi_rot(al, be, gr, gi, skip, tol, Rt)) {
        rot = true;
        for (int i = lg; i < m; i += GT) {
          float2 x = ap[i], y = aq[i];
          apply_rot(x, y, Rt);
          ap[i] = x;
          aq[i] = y;
        }
        float2* vp = V + (size_t)p * n;
        float2* vq = V + (size_t)q * n;
        for (int i = lg; i < n; i += GT) {
          float2 x = vp[i], y = vq[i];
          apply_rot(x, y, Rt);
          vp[i] = x;
          vq[i] = y;
        }
      }
    }
  }
  return rot;
}

template <int GT, int R>
__global__ void __launch_bounds__(1024) k_svd_small(GateDesc* desc, const int32_t* __restrict__ list, uint8_t* slab,
                                                    DevState* st, int max_sweeps) {
  extern __shared__ __align__(16) uint8_t sm[];
  GateDesc& gd = desc[list[blockIdx.x]];
  const int m = gd.m, n = gd.n;  // n even (n = d * chi_r)
  float2* A = reinterpret_cast<float2*>(sm);      // m x n, ld m
  float2* V = A + (size_t)m * n;                  // n x n, ld n
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  double* s2 = reinterpret_cast<double*>(V + (size_t)n * n);
  int32_t* six = reinterpret_cast<int32_t*>(s2 + npow2);
  double* part = reinterpret_cast<double*>(six + npow2 + (npow2 & 1));  // blockDim.x doubles
  __shared__ float s_wn[32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float2* __restrict__ gth = reinterpret_cast<const float2*>(slab + gd.ws_theta);
  float nrm = 0.f;
  for (int x = tid; x < m * n; x += blockDim.x) {
    float2 v = gth[x];
    A[x] = v;
    nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, nrm));
  }
  for (int x = tid; x < n * n; x += blockDim.x) V[x] = make_float2((x / n) == (x % n) ? 1.f : 0.f, 0.f);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  if (lane == 0) s_wn[warp] = nrm;
  __syncthreads();
  float norm2 = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) norm2 += s_wn[w];  // fixed order: deterministic
  // rounding floor for a column (SURVEY §8(c) item 3 with eps = 2^-24 on the GPU)
  const float skip = norm2 * 3.5527137e-15f;  // (2^-24)^2 ||theta||_F^2
  const float tol = fmaxf(7.62939453e-6f, 4.f * sqrtf((float)m) * 5.96046448e-8f);  // max(2^-17, 4 sqrt(m) 2^-24)

  int sweep = 0;
  bool converged = (n < 2);
  const int half = n / 2, gid = tid / GT, lg = tid % GT;
  bool planar = false;
  if constexpr (R >= 2) planar = (m == R * GT && n == R * GT && (int)(blockDim.x / GT) >= half);
  if (planar) {
    // square theta whose rows fill the lane groups exactly (config 2 chi = 16: 32 x 32, 8-lane
    // groups, 4 rows per lane): theta and V PAIR-PLANAR (as the QR kernel, jacobi_common.cuh
    // ColRegs), so the gamma dot and both rotations are packed FFMA2 on two rows with broadcast
    // coefficients -- no operand-building MOVs of the interleaved layout, which made this kernel
    // issue-bound (IPC 3.0). Same circle schedule, criterion and cached norms as the path below.
    constexpr int RR = R >= 2 ? R : 2;
    uint16_t* sched = reinterpret_cast<uint16_t*>(part + blockDim.x);
    float* cn = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(sched + (n - 1) * half) + 15) & ~uintptr_t(15));
    build_circle_schedule(sched, n);
    __syncthreads();
    pair_planar(A, m, n);
    pair_planar(V, n, n);
    __syncthreads();
    const bool active = gid < half;
    const float tol2 = tol * tol;
    for (; sweep < max_sweeps && !converged; ++sweep) {
      for (int j = warp; j < n; j += (int)(blockDim.x >> 5)) {
        float a = 0.f;
        for (int i = lane; i < m; i += 32) a = fmaf(A[j * m + i].x, A[j * m + i].x, fmaf(A[j * m + i].y, A[j * m + i].y, a));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) cn[j] = a;
      }
      __syncthreads();
      int any = 0;
      for (int rnd = 0; rnd < n - 1; ++rnd) {
        bool rot = false;
        int p = 0, q = 1;
        float gr = 0.f, gi = 0.f;
        ColRegs<GT, RR> X, Y;
        if (active) {
          const uint32_t pq = sched[rnd * half + gid];
          p = pq & 0xFF;
          q = pq >> 8;
          X.load(A + p * m, lg);
          Y.load(A + q * m, lg);
          cross_planar(X, Y, gr, gi);
        }
        group_sum2<GT>(gr, gi);   // (all lanes: a warp may hold active and idle groups)
        if (active) {
          const float al = cn[p], be = cn[q];
          Rot Rt;
          float tg;
          if (jacobi_rot_fast(al, be, gr, gi, skip, tol2, Rt, tg)) {
            rot = true;
            rot_planar(X, Y, Rt);
            X.store(A + p * m, lg);
            Y.store(A + q * m, lg);
            ColRegs<GT, RR> P, Q;
            P.load(V + p * n, lg);
            Q.load(V + q * n, lg);
            rot_planar(P, Q, Rt);
            P.store(V + p * n, lg);
            Q.store(V + q * n, lg);
            if (lg == 0) {
              cn[p] = al - tg;
              cn[q] = be + tg;
            }
          }
        }
        any |= __syncthreads_or(rot);
      }
      converged = (any == 0);
    }
    pair_planar(V, n, n);   // back to interleaved rows for the epilogue (A is reloaded below)
    __syncthreads();
  } else if (R > 0 && n <= 256 && (int)(blockDim.x / GT) >= half) {
    // fast path (as the QR kernel): one pair per lane group, rows of theta and V in registers,
    // schedule from shared memory, cached column norms (exact at each sweep start), gamma-only dots
    constexpr int RR = R > 0 ? R : 1;
    uint16_t* sched = reinterpret_cast<uint16_t*>(part + blockDim.x);
    float* cn = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(sched + (n - 1) * half) + 15) & ~uintptr_t(15));
    build_circle_schedule(sched, n);
    const bool active = gid < half;
    const int sh = gid & (32 / GT - 1);
    const float tol2 = tol * tol;
    for (; sweep < max_sweeps && !converged; ++sweep) {
      for (int j = warp; j < n; j += (int)(blockDim.x >> 5)) {
        float a = 0.f;
        for (int i = lane; i < m; i += 32) a = fmaf(A[j * m + i].x, A[j * m + i].x, fmaf(A[j * m + i].y, A[j * m + i].y, a));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) cn[j] = a;
      }
      __syncthreads();
      int any = 0;
      for (int rnd = 0; rnd < n - 1; ++rnd) {
        bool rot = false;
        int p = 0, q = 1;
        float gr = 0.f, gi = 0.f;
        PairRegs<GT, RR> pr;
        if (active) {
          const uint32_t pq = sched[rnd * half + gid];
          p = pq & 0xFF;
          q = pq >> 8;
          pr.load(A + p * m, A + q * m, m, lg, sh);
          pr.cross(gr, gi);
        }
        group_sum2<GT>(gr, gi);   // (all lanes: a warp may hold active and idle groups)
        if (active) {
          const float al = cn[p], be = cn[q];
          Rot Rt;
          float tg;
          if (jacobi_rot_fast(al, be, gr, gi, skip, tol2, Rt, tg)) {
            rot = true;
            pr.rotate_store(A + p * m, A + q * m, m, lg, sh, Rt);
            PairRegs<GT, RR> pv;
            pv.load(V + p * n, V + q * n, n, lg, sh);
            pv.rotate_store(V + p * n, V + q * n, n, lg, sh, Rt);
            if (lg == 0) {
              cn[p] = al - tg;
              cn[q] = be + tg;
            }
          }
        }
        any |= __syncthreads_or(rot);
      }
      converged = (any == 0);
    }
  } else {
    for (; sweep < max_sweeps && !converged; ++sweep) {
      int any = 0;
      for (int rnd = 0; rnd < n - 1; ++rnd) any |= __syncthreads_or(round_pairs<GT, R>(A, m, n, V, rnd, skip, tol));
      converged = (any == 0);
    }
  }
  if (!converged && tid == 0) atomicCAS(&st->led.error, 0, -6 /* MPS_E_NOCONV */);
  for (int x = tid; x < m * n; x += blockDim.x) A[x] = gth[x];  // the original theta for the Rayleigh quotient
  __syncthreads();
  jacobi_epilogue(gd, slab, st, A, V, s2, six, part);
  if (tid == 0) gd.sweeps = sweep;
}

}  // namespace

size_t svd_small_smem(int m, int n) {
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  return (size_t)m * n * 8 + (size_t)n * n * 8 + (size_t)npow2 * 12 + 16 + 1024 * 8 +
         (n <= 256 ? (size_t)(n - 1) * (n / 2) * 2 + 16 + (size_t)n * 4 : 0);
}

bool svd_small_fits(int m, int n) { return svd_small_smem(m, n) <= 210 * 1024; }

int small_group(int m) {
  if (m <= 16) return 4;
  if (m <= 48) return 8;
  if (m <= 96) return 16;
  return 32;
}

template <int GT, int R>
static void launch_small_t(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem, int max_sweeps, int threads,
                           uint8_t* slab, DevState* st, cudaStream_t s) {
  static std::atomic<unsigned long long> attr_set{0};
  if (first_on_device(attr_set)) {
    cudaFuncSetAttribute(k_svd_small<GT, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  }
  k_svd_small<GT, R><<<count, threads, smem, s>>>(d_desc, d_list, slab, st, max_sweeps);
}

template <int GT>
static void launch_small_r(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem, int max_sweeps, int rpl,
                           int threads, uint8_t* slab, DevState* st, cudaStream_t s) {
  switch (rpl) {
    case 1: launch_small_t<GT, 1>(d_desc, d_list, count, smem, max_sweeps, threads, slab, st, s); break;
    case 2: launch_small_t<GT, 2>(d_desc, d_list, count, smem, max_sweeps, threads, slab, st, s); break;
    case 4: launch_small_t<GT, 4>(d_desc, d_list, count, smem, max_sweeps, threads, slab, st, s); break;
    case 8: launch_small_t<GT, 8>(d_desc, d_list, count, smem, max_sweeps, threads, slab, st, s); break;
    case 16: launch_small_t<GT, 16>(d_desc, d_list, count, smem, max_sweeps, threads, slab, st, s); break;
    default: launch_small_t<GT, 0>(d_desc, d_list, count, smem, max_sweeps, threads, slab, st, s); break;
  }
}

void launch_svd_small(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem, int max_sweeps, int gt, int rpl,
                      int threads, uint8_t* slab, DevState* st, cudaStream_t s) {
  if (count <= 0) return;
  switch (gt) {
    case 4: launch_small_r<4>(d_desc, d_list, count, smem, max_sweeps, rpl, threads, slab, st, s); break;
    case 8: launch_small_r<8>(d_desc, d_list, count, smem, max_sweeps, rpl, threads, slab, st, s); break;
    case 16: launch_small_r<16>(d_desc, d_list, count, smem, max_sweeps, rpl, threads, slab, st, s); break;
    default: launch_small_r<32>(d_desc, d_list, count, smem, max_sweeps, rpl, threads, slab, st, s); break;
  }
}

}  // namespace eamps
