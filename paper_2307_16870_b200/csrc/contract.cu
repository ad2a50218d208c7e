// contract.cu -- step a1: "Contracting both tensors neighbouring the bond"
// with the gate, plus the lambda_{i-1} row scale that turns the B-lambda pair into
// the Vidal centre:
//   C[(a,s'),(t',c)]      = sum_b B_i[a,s',b] B_{i+1}[b,t',c]          (GEMM, K = chi_m)
//   Theta'[(a,s),(t,c)]   = sum_{s',t'} U[s d + t, s' d + t'] C[(a,s'),(t',c)]   (epilogue)
//   theta                 = diag(lambda_{i-1} (x) 1_d) Theta'
// Both Theta' and theta are written column-major (ld = m) for the column-oriented Jacobi.
//
// One CTA computes a 64x64 tile of C covering TA = 64/d left indices a and TC = 64/d right
// indices c for ALL physical (s', t'), so the d^2 x d^2 gate mixing is local to the tile and
// fused into the epilogue (no extra pass over HBM). SIMT FP32: the contraction is 1-3% of the
// update's flops; the tensor-core path is reserved for the SVD rotations.
#include "eamps_internal.cuh"

namespace eamps {

namespace {

constexpr int KC = 16;

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

template <int D>
__global__ void __launch_bounds__(256) k_contract(const GateDesc* __restrict__ desc, const int32_t* __restrict__ prefix,
                                                  int G, uint8_t* slab, const DevState* st,
                                                  const float2* __restrict__ us) {
  constexpr int TA = 64 / D, TC = 64 / D;
  __shared__ float2 smem[64 * 65];  // As/Bs during the K loop, Cs in the epilogue
  __shared__ float2 Us[D * D * D * D];
  float2(*As)[65] = reinterpret_cast<float2(*)[65]>(smem);            // [KC][65]
  float2(*Bs)[65] = reinterpret_cast<float2(*)[65]>(smem + KC * 65);  // [KC][65]
  float2(*Cs)[65] = reinterpret_cast<float2(*)[65]>(smem);            // [64][65]

  const int tile = blockIdx.x;
  int lo = 0, hi = G - 1;
  while (lo < hi) {
    int md = (lo + hi + 1) >> 1;
    if (prefix[md] <= tile) lo = md; else hi = md - 1;
  }
  const GateDesc gd = desc[lo];
  const int local = tile - prefix[lo];
  const int ntc = (gd.r + TC - 1) / TC;
  const int a0 = (local / ntc) * TA, c0 = (local % ntc) * TC;
  const int l = gd.l, mid = gd.mid, r = gd.r, m = gd.m;

  const SiteEntry* sites = reinterpret_cast<const SiteEntry*>(slab + st->sites_off);
  const BondEntry* bonds = reinterpret_cast<const BondEntry*>(slab + st->bonds_off);
  const float2* __restrict__ Bi = reinterpret_cast<const float2*>(slab + sites[gd.site].off);
  const float2* __restrict__ Bj = reinterpret_cast<const float2*>(slab + sites[gd.site + 1].off);
  const float* __restrict__ lam = reinterpret_cast<const float*>(slab + bonds[gd.site].off);  // bond site-1
  float2* __restrict__ thp = reinterpret_cast<float2*>(slab + gd.ws_thetap);
  float2* __restrict__ th = reinterpret_cast<float2*>(slab + gd.ws_theta);

  const int tid = threadIdx.x;
  for (int x = tid; x < D * D * D * D; x += 256) Us[x] = us[(int64_t)gd.u_index * D * D * D * D + x];

  const int ty = tid >> 4, tx = tid & 15;
  // FP32 products accumulated per KC-chunk, chunk sums accumulated in FP64: the rounding of a
  // chi_m-long dot product drops from ~sqrt(chi_m) eps32 to ~sqrt(KC) eps32 (DESIGN "Precision")
  double2 dacc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) dacc[i][j] = make_double2(0.0, 0.0);

  for (int b0 = 0; b0 < mid; b0 += KC) {
    // A chunk: rows rho = (a_local, s') of B_i as (l d) x mid, columns b0..b0+KC (contiguous)
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      int e = tid + it * 256;          // 0..1023
      int kk = e & (KC - 1), rho = e >> 4;
      int a = a0 + rho / D, sp = rho % D, b = b0 + kk;
      float2 v = make_float2(0.f, 0.f);
      if (a < l && b < mid) v = Bi[((int64_t)a * D + sp) * mid + b];
      As[kk][rho] = v;
    }
    // B chunk: rows b, columns kappa = (t', c_local) of B_{i+1} as mid x (d r)
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      int e = tid + it * 256;
      int cc = e % TC, rest = e / TC;  // rest = t' + D * kk
      int tp = rest % D, kk = rest / D;
      int c = c0 + cc, b = b0 + kk;
      float2 v = make_float2(0.f, 0.f);
      if (c < r && b < mid) v = Bj[((int64_t)b * D + tp) * r + c];
      Bs[kk][tp * TC + cc] = v;
    }
    __syncthreads();
    float2 acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      float2 av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j].x = fmaf(av[i].x, bv[j].x, acc[i][j].x);
          acc[i][j].x = fmaf(-av[i].y, bv[j].y, acc[i][j].x);
          acc[i][j].y = fmaf(av[i].x, bv[j].y, acc[i][j].y);
          acc[i][j].y = fmaf(av[i].y, bv[j].x, acc[i][j].y);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) { dacc[i][j].x += acc[i][j].x; dacc[i][j].y += acc[i][j].y; }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) Cs[ty + 16 * i][tx + 16 * j] = make_float2((float)dacc[i][j].x, (float)dacc[i][j].y);
  __syncthreads();

  // epilogue: gate mixing over (s', t') and the lambda row scale; coalesced along a
  for (int p = tid; p < TA * TC; p += 256) {
    int al = p % TA, cl = p / TA;
    int a = a0 + al, c = c0 + cl;
    if (a >= l || c >= r) continue;
    float la = lam[a];
#pragma unroll
    for (int s = 0; s < D; ++s)
#pragma unroll
      for (int t = 0; t < D; ++t) {
        float2 o = make_float2(0.f, 0.f);
#pragma unroll
        for (int sp = 0; sp < D; ++sp)
#pragma unroll
          for (int tp = 0; tp < D; ++tp) {
            float2 u = Us[(s * D + t) * D * D + sp * D + tp];
            float2 cv = Cs[al * D + sp][tp * TC + cl];
            float2 pr = cmul(u, cv);
            o.x += pr.x;
            o.y += pr.y;
          }
        int64_t idx = (int64_t)(t * r + c) * m + (a * D + s);
        thp[idx] = o;
        th[idx] = make_float2(la * o.x, la * o.y);
      }
  }
}

}  // namespace

void launch_contract(const GateDesc* d_desc, const int32_t* d_tile_prefix, int G, int total_tiles, int d,
                     uint8_t* slab, const DevState* st, const float2* d_us, cudaStream_t s) {
  if (total_tiles <= 0) return;
  if (d == 2)
    k_contract<2><<<total_tiles, 256, 0, s>>>(d_desc, d_tile_prefix, G, slab, st, d_us);
  else
    k_contract<4><<<total_tiles, 256, 0, s>>>(d_desc, d_tile_prefix, G, slab, st, d_us);
}

}  // namespace eamps
