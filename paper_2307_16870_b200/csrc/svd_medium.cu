// svd_medium.cu -- step a2 + a3 when theta fits one CTA's shared memory but theta AND V do not
// (e.g. the config-2 chi = 64 thetas, 128 x 128 complex64 = 128 KB each).
//
// Two one-CTA-per-theta kernels instead of a cluster: the rotations are data-independent of V,
// so V can be built afterwards from a log of the rotations.
//   k_svd_theta : the one-sided Jacobi of svd_small.cu on theta alone (theta in shared memory);
//                 every round's rotation per column pair goes to a log in the workspace exactly as
//                 applied, (c, s, Re e, Im e): 16 B per pair-round, ~1.5 MB per theta for 12
//                 sweeps at n = 128 (no transcendental on either side).
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

__device__ __forceinline__ void tc_cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void tc_cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void tc_cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void tc_cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// The circle-method schedule of one sweep, (p | q << 8) per (round, slot), built once per CTA in
// shared memory (n <= 256): no integer modulo on the per-round path.
__device__ __forceinline__ void build_schedule(uint16_t* sched, int n) {
  const int half = n / 2;
  for (int x = threadIdx.x; x < (n - 1) * half; x += blockDim.x) {
    const int rnd = x / half, slot = x % half;
    int p, q;
    circle_pair_n(slot, rnd, n, p, q);
    sched[x] = (uint16_t)(p | (q << 8));
  }
}

template <int GT, int R>
__global__ void __launch_bounds__(512) k_svd_theta(GateDesc* desc, const int32_t* __restrict__ list, uint8_t* slab,
                                                    DevState* st, int max_sweeps) {
  extern __shared__ __align__(16) uint8_t sm[];
  GateDesc& gd = desc[list[blockIdx.x]];
  const int m = gd.m, n = gd.n;
  float2* A = reinterpret_cast<float2*>(sm);
  uint16_t* sched = reinterpret_cast<uint16_t*>(A + (size_t)m * n);   // (n - 1) x n/2
  __shared__ float s_wn[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float2* __restrict__ gth = reinterpret_cast<const float2*>(slab + gd.ws_theta);
  float4* lg = reinterpret_cast<float4*>(slab + gd.ws_log);
  float nrm = 0.f;
  for (int x = tid; x < m * n; x += blockDim.x) {
    float2 v = gth[x];
    A[x] = v;
    nrm = fmaf(v.x, v.x, fmaf(v.y, v.y, nrm));
  }
  const bool use_sched = n <= 256 && R > 0 && blockDim.x / GT >= n / 2;   // (the fast path below)
  if (use_sched) build_schedule(sched, n);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
  if (lane == 0) s_wn[warp] = nrm;
  __syncthreads();
  float norm2 = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) norm2 += s_wn[w];
  const float skip = norm2 * 3.5527137e-15f;
  const float tol = fmaxf(7.62939453e-6f, 4.f * sqrtf((float)m) * 5.96046448e-8f);
  const int groups = blockDim.x / GT, gid = tid / GT, lgi = tid % GT;
  const int half = n / 2;
  const int cap = min(max_sweeps, gd.log_sweeps);
  int sweep = 0;
  bool converged = (n < 2);
  if (use_sched) {
    // fast path: one column pair per lane group (groups >= n/2, checked by the host), the pair's
    // rows in registers, schedule from shared memory, 32-bit log index, and cached column norms
    // (recomputed exactly at every sweep start, updated analytically after each rotation), so a
    // round only forms gamma = a_p^H a_q
    const bool active = gid < half;
    const bool full = (m == R * GT);   // (R > 0 here)
    const int sh = gid & (32 / GT - 1); // group index within the warp (bank spreading)
    float* cn = reinterpret_cast<float*>(                                 // n cached |a_j|^2
        (reinterpret_cast<uintptr_t>(sched + (n - 1) * half) + 15) & ~uintptr_t(15));
    const float tol2 = tol * tol;
    uint32_t li = (uint32_t)gid;      // log index = (sweep (n-1) + rnd) n/2 + slot
    for (; sweep < cap && !converged; ++sweep) {
      for (int j = warp; j < n; j += (int)(blockDim.x >> 5)) {   // exact norms at the sweep start
        float a = 0.f;
        for (int i = lane; i < m; i += 32) {
          const float2 v = A[j * m + i];
          a = fmaf(v.x, v.x, fmaf(v.y, v.y, a));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) cn[j] = a;
      }
      __syncthreads();
      int any = 0;
      for (int rnd = 0; rnd < n - 1; ++rnd, li += half) {
        bool rot = false;
        // (a warp may hold active and idle groups: the shuffles run unconditionally)
        constexpr int RR = R > 0 ? R : 1;
        PairRegs<GT, RR> pr;
        int p = 0, q = 1;
        float gr = 0.f, gi = 0.f;
        if (active) {
          const uint32_t pq = sched[rnd * half + gid];
          p = pq & 0xFF;
          q = pq >> 8;
          if (full) pr.load_full(A + p * m, A + q * m, lgi, sh);
          else pr.load(A + p * m, A + q * m, m, lgi, sh);
          pr.cross(gr, gi);
        }
        group_sum2<GT>(gr, gi);
        if (active) {
          float2* ap = A + p * m;
          float2* aq = A + q * m;
          const float al = cn[p], be = cn[q];
          Rot Rt;
          float tg;
          const bool doit = jacobi_rot_fast(al, be, gr, gi, skip, tol2, Rt, tg);
          if (lgi == 0) lg[li] = make_float4(Rt.c, Rt.s, Rt.er, Rt.ei);
          if (doit) {
            rot = true;
            if (full) pr.rotate_store_full(ap, aq, lgi, sh, Rt);
            else pr.rotate_store(ap, aq, m, lgi, sh, Rt);
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
  } else {
    for (; sweep < cap && !converged; ++sweep) {
      int any = 0;
      for (int rnd = 0; rnd < n - 1; ++rnd) {
        bool rot = false;
        float4* lrow = lg + ((size_t)sweep * (n - 1) + rnd) * half;
        for (int base = 0; base < half; base += groups) {
          const int slot = base + gid;
          const bool active = slot < half;
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
          group_sum4<GT>(al, be, gr, gi);
          Rot Rt;
          const bool doit = active && jacobi_rot(al, be, gr, gi, skip, tol, Rt);
          // log the applied rotation exactly (c, s, Re e, Im e); identity rotations have s = 0
          if (active && lgi == 0) lrow[slot] = make_float4(Rt.c, Rt.s, Rt.er, Rt.ei);
          if (doit) {
            rot = true;
            for (int i = lgi; i < m; i += GT) {
              float2 x = ap[i], y = aq[i];
              apply_rot(x, y, Rt);
              ap[i] = x;
              aq[i] = y;
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
}

template <int GT, int R>
__global__ void __launch_bounds__(512) k_svd_vrep(GateDesc* desc, const int32_t* __restrict__ list, uint8_t* slab,
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
  uint16_t* sched = reinterpret_cast<uint16_t*>(part + blockDim.x);   // (n - 1) x n/2 when n <= 256
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int x = tid; x < n * n; x += blockDim.x) V[x] = make_float2((x / n) == (x % n) ? 1.f : 0.f, 0.f);
  const bool use_sched = n <= 256;
  if (use_sched) build_schedule(sched, n);
  __syncthreads();
  const float4* lg = reinterpret_cast<const float4*>(slab + gd.ws_log);
  const int groups = blockDim.x / GT, gid = tid / GT, lgi = tid % GT;
  const int half = n / 2;
  // V = I R_1 R_2 ... replayed from the log. The log streams through shared memory in chunks of
  // LR rounds (cp.async, double-buffered in the space of the Rayleigh tile T), so the per-round
  // reads are shared-memory reads; the log is read once from HBM/L2.
  constexpr int LR = 8;
  const int total = S * (n - 1);
  const int nchunks = (total + LR - 1) / LR;
  float4* lbuf = reinterpret_cast<float4*>(T);                      // 2 x LR x n/2 float4
  const size_t lbuf_need = (size_t)2 * LR * half * sizeof(float4);
  const bool staged = lbuf_need <= (size_t)tile_rows * ldt * sizeof(float2);
  auto issue = [&](int c) {
    if (staged && c < nchunks) {
      const int t0 = c * LR, nt = min(LR, total - t0);
      float4* dst = lbuf + (size_t)(c & 1) * LR * half;
      const float4* src = lg + (size_t)t0 * half;
      for (int x = tid; x < nt * half; x += blockDim.x) tc_cp_async16(dst + x, src + x);
    }
    tc_cp_async_commit();
  };
  issue(0);
  const bool full = R > 0 && n == R * GT;
  const int sh = gid & (32 / GT - 1);
  for (int c = 0; c < nchunks; ++c) {
    issue(c + 1);
    tc_cp_async_wait1();
    __syncthreads();
    const float4* lrow0 = staged ? lbuf + (size_t)(c & 1) * LR * half : lg + (size_t)c * LR * half;
    const int t0 = c * LR, nt = min(LR, total - t0);
    for (int tt = 0; tt < nt; ++tt) {
      const int rnd = (t0 + tt) % (n - 1);
      const float4* lrow = lrow0 + (size_t)tt * half;
      for (int slot = gid; slot < half; slot += groups) {
        const float4 r = lrow[slot];
        if (r.y == 0.f) continue;  // identity rotation (uniform within the group)
        int p, q;
        if (use_sched) {
          const uint32_t pq = sched[rnd * half + slot];
          p = pq & 0xFF;
          q = pq >> 8;
        } else {
          circle_pair_n(slot, rnd, n, p, q);
        }
        Rot Rt;
        Rt.c = r.x;
        Rt.s = r.y;
        Rt.er = r.z;
        Rt.ei = r.w;
        float2* vp = V + (size_t)p * n;
        float2* vq = V + (size_t)q * n;
        if constexpr (R > 0) {
          PairRegs<GT, R> pv;
          if (full) {
            pv.load_full(vp, vq, lgi, sh);
            pv.rotate_store_full(vp, vq, lgi, sh, Rt);
          } else {
            pv.load(vp, vq, n, lgi, sh);
            pv.rotate_store(vp, vq, n, lgi, sh, Rt);
          }
        } else {
          for (int i = lgi; i < n; i += GT) {
            float2 x = vp[i], y = vq[i];
            apply_rot(x, y, Rt);
            vp[i] = x;
            vq[i] = y;
          }
        }
      }
      __syncthreads();
    }
  }
  tc_cp_async_wait0();
  __syncthreads();   // the log buffers (in T) are dead before the Rayleigh tiles overwrite them
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

size_t svd_theta_smem(int m, int n) { return (size_t)m * n * 8 + (size_t)(n - 1) * (n / 2) * 2 + 16 + (size_t)n * 4 + 64; }

size_t svd_vrep_smem(int n, int tile_rows) {
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  return (size_t)n * n * 8 + (size_t)tile_rows * (n + 1) * 8 + (size_t)npow2 * 12 + 16 + 1024 * 8 +
         (n <= 256 ? (size_t)(n - 1) * (n / 2) * 2 : 0);
}

bool svd_medium_fits(int m, int n) { return svd_theta_smem(m, n) <= 210 * 1024 && svd_vrep_smem(n, 8) <= 210 * 1024; }

int vrep_tile_rows(int m, int n) {
  int t = 64;
  while (t > 8 && svd_vrep_smem(n, t) > 210 * 1024) t >>= 1;
  return std::min(t, m);
}

template <int GT, int R>
static void launch_medium_t(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem_theta, size_t smem_vrep,
                            int tile_rows, int max_sweeps, int threads, uint8_t* slab, DevState* st, cudaStream_t s) {
  static std::atomic<unsigned long long> attr_set{0};
  if (first_on_device(attr_set)) {
    cudaFuncSetAttribute(k_svd_theta<GT, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k_svd_vrep<GT, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  }
  k_svd_theta<GT, R><<<count, threads, smem_theta, s>>>(d_desc, d_list, slab, st, max_sweeps);
  k_svd_vrep<GT, R><<<count, threads, smem_vrep, s>>>(d_desc, d_list, slab, st, tile_rows);
}

template <int GT>
static void launch_medium_r(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem_theta, size_t smem_vrep,
                            int tile_rows, int max_sweeps, int rpl, int threads, uint8_t* slab, DevState* st,
                            cudaStream_t s) {
  switch (rpl) {
    case 1: launch_medium_t<GT, 1>(d_desc, d_list, count, smem_theta, smem_vrep, tile_rows, max_sweeps, threads, slab, st, s); break;
    case 2: launch_medium_t<GT, 2>(d_desc, d_list, count, smem_theta, smem_vrep, tile_rows, max_sweeps, threads, slab, st, s); break;
    case 4: launch_medium_t<GT, 4>(d_desc, d_list, count, smem_theta, smem_vrep, tile_rows, max_sweeps, threads, slab, st, s); break;
    case 8: launch_medium_t<GT, 8>(d_desc, d_list, count, smem_theta, smem_vrep, tile_rows, max_sweeps, threads, slab, st, s); break;
    case 16: launch_medium_t<GT, 16>(d_desc, d_list, count, smem_theta, smem_vrep, tile_rows, max_sweeps, threads, slab, st, s); break;
    default: launch_medium_t<GT, 0>(d_desc, d_list, count, smem_theta, smem_vrep, tile_rows, max_sweeps, threads, slab, st, s); break;
  }
}

void launch_svd_medium(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem_theta, size_t smem_vrep,
                       int tile_rows, int max_sweeps, int gt, int rpl, int threads, uint8_t* slab, DevState* st,
                       cudaStream_t s) {
  if (count <= 0) return;
  switch (gt) {
    case 4: launch_medium_r<4>(d_desc, d_list, count, smem_theta, smem_vrep, tile_rows, max_sweeps, rpl, threads, slab, st, s); break;
    case 8: launch_medium_r<8>(d_desc, d_list, count, smem_theta, smem_vrep, tile_rows, max_sweeps, rpl, threads, slab, st, s); break;
    case 16: launch_medium_r<16>(d_desc, d_list, count, smem_theta, smem_vrep, tile_rows, max_sweeps, rpl, threads, slab, st, s); break;
    default: launch_medium_r<32>(d_desc, d_list, count, smem_theta, smem_vrep, tile_rows, max_sweeps, rpl, threads, slab, st, s); break;
  }
}

}  // namespace eamps
