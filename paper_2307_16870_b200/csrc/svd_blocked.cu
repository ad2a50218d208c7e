// svd_blocked.cu -- step a2 + a3 for thetas that do not fit one CTA (K3 "large" regime,
// SURVEY §2.4 / §8(a) a2): blocked one-sided Jacobi with the working theta and V in HBM/L2.
//
// Columns are grouped in blocks of b = 16; a tournament (circle method) over the n_pad/16
// blocks pairs them, n_pad/32 disjoint block pairs per round, one CTA per block pair. A CTA
//   A. streams the 32-column panel P = [A_I A_J] through shared memory and forms its Gram
//      G = P^H P (FP32 products accumulated per 64-row chunk, chunks summed in FP64);
//   B. if some |g_pq| > tol sqrt(g_pp g_qq) (the one-sided Jacobi criterion, evaluated on the
//      freshly computed Gram), diagonalises G in FP64 with cyclic two-sided Jacobi, W = prod J,
//      using exactly the 2x2 rotation of the scalar method;
//   C. applies the block rotation P <- P W and [V_I V_J] <- [V_I V_J] W (streamed, FP32).
// A sweep = n_pad/16 - 1 rounds (one launch each); it converges when no CTA rotated. This is
// the same fixed point as the scalar method (all column pairs orthogonal to tol); the block
// rotation is the GEMM-shaped step that the tensor-core path will take over.
// Then sigma_j^2 = ||theta v_j||^2/||v_j||^2 (Rayleigh, FP64 accumulation) and sort + tails.
#include "eamps_internal.cuh"
#include "sort_tails.cuh"

namespace eamps {

namespace {

constexpr int BLK = 16;        // columns per block
constexpr int PW = 2 * BLK;    // panel width
constexpr int RC = 64;         // rows per streamed chunk

__device__ __forceinline__ void circle_pair(int i, int rnd, int n, int& p, int& q) {
  auto pos = [&](int j) { return j == 0 ? 0 : ((j - 1 + rnd) % (n - 1)) + 1; };
  p = pos(i);
  q = pos(n - 1 - i);
}

constexpr size_t kRoundSmem = sizeof(float2) * RC * (PW + 1) + 2 * sizeof(double2) * PW * (PW + 1) +
                              sizeof(float2) * PW * (PW + 1);

struct LargeCtl {               // per gate in the large list
  int32_t rot;                  // rotations this sweep (CTA-level)
  int32_t conv;                 // converged
};

__global__ void k_large_init(GateDesc* desc, const int32_t* list, uint8_t* slab) {
  GateDesc& gd = desc[list[blockIdx.y]];
  const int m = gd.m, n = gd.n, np = gd.n_pad;
  float2* th = reinterpret_cast<float2*>(slab + gd.ws_theta);
  float2* V = reinterpret_cast<float2*>(slab + gd.ws_V);
  const int64_t tot_pad = (int64_t)m * (np - n);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < (int64_t)np * np; x += (int64_t)gridDim.x * blockDim.x) {
    int64_t col = x / np, row = x % np;
    V[x] = make_float2(col == row ? 1.f : 0.f, 0.f);
    if (x < tot_pad) th[(int64_t)m * n + x] = make_float2(0.f, 0.f);  // padded zero columns
  }
}

// ||theta||_F^2 in FP64 (deterministic: fixed per-thread order + fixed tree)
__global__ void k_large_norm(GateDesc* desc, const int32_t* list, uint8_t* slab, double* norm2) {
  const GateDesc& gd = desc[list[blockIdx.x]];
  const float2* th = reinterpret_cast<const float2*>(slab + gd.ws_theta);
  const int64_t tot = (int64_t)gd.m * gd.n;
  double s = 0.0;
  for (int64_t x = threadIdx.x; x < tot; x += blockDim.x) s += (double)th[x].x * th[x].x + (double)th[x].y * th[x].y;
  __shared__ double part[256];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) part[threadIdx.x] += part[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) norm2[blockIdx.x] = part[0];
}

__global__ void __launch_bounds__(256) k_block_round(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                     int rnd, uint8_t* slab, LargeCtl* ctl, const double* norm2) {
  const int gi = blockIdx.y;
  if (ctl[gi].conv) return;
  const GateDesc gd = desc[list[gi]];
  const int nb = gd.n_pad / BLK;
  if ((int)blockIdx.x >= nb / 2 || rnd >= nb - 1) return;
  int I, J;
  circle_pair(blockIdx.x, rnd, nb, I, J);
  const int m = gd.m, np = gd.n_pad;
  float2* th = reinterpret_cast<float2*>(slab + gd.ws_theta);
  float2* V = reinterpret_cast<float2*>(slab + gd.ws_V);

  extern __shared__ __align__(16) uint8_t dsm[];
  float2(*Ps)[PW + 1] = reinterpret_cast<float2(*)[PW + 1]>(dsm);                                   // [RC]
  double2(*Gs)[PW + 1] = reinterpret_cast<double2(*)[PW + 1]>(dsm + sizeof(float2) * RC * (PW + 1));   // [PW]
  double2(*Ws)[PW + 1] = Gs + PW;                                                                      // [PW]
  float2(*Wf)[PW + 1] = reinterpret_cast<float2(*)[PW + 1]>(Ws + PW);                                 // [PW]
  __shared__ double rc[16][4];  // per pair: c, s, er, ei
  __shared__ int s_any, s_inner;

  const int tid = threadIdx.x;
  auto colof = [&](int x) { return x < BLK ? I * BLK + x : J * BLK + (x - BLK); };

  // ---- A. Gram of the panel
  const int gp = tid >> 3, gq = (tid & 7) * 4;
  double2 dacc[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) dacc[j] = make_double2(0.0, 0.0);
  for (int r0 = 0; r0 < m; r0 += RC) {
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      int i = tid & (RC - 1), c = (tid >> 6) + 4 * it;
      int row = r0 + i;
      Ps[i][c] = row < m ? th[(int64_t)colof(c) * m + row] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    float2 acc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j] = make_float2(0.f, 0.f);
    for (int i = 0; i < RC; ++i) {
      float2 x = Ps[i][gp];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 y = Ps[i][gq + j];
        acc[j].x = fmaf(x.x, y.x, fmaf(x.y, y.y, acc[j].x));   // conj(x) y
        acc[j].y = fmaf(x.x, y.y, fmaf(-x.y, y.x, acc[j].y));
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) { dacc[j].x += acc[j].x; dacc[j].y += acc[j].y; }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) Gs[gp][gq + j] = dacc[j];
  for (int x = tid; x < PW * PW; x += 256) {
    int a = x / PW, b = x % PW;
    Ws[a][b] = make_double2(a == b ? 1.0 : 0.0, 0.0);
  }
  if (tid == 0) s_any = 0;
  __syncthreads();

  // ---- B. is the panel already orthogonal? (the scalar criterion on the fresh Gram)
  const double skip = norm2[gi] * 3.552713678800501e-15;                    // (2^-24)^2 ||theta||^2
  const double tol = fmax(7.62939453125e-6, 4.0 * sqrt((double)m) * 5.960464477539063e-8);
  for (int x = tid; x < PW * PW; x += 256) {
    int p = x / PW, q = x % PW;
    if (p < q) {
      double al = Gs[p][p].x, be = Gs[q][q].x;
      double g = sqrt(Gs[p][q].x * Gs[p][q].x + Gs[p][q].y * Gs[p][q].y);
      if (fmin(al, be) > skip && g > tol * sqrt(al * be)) s_any = 1;
    }
  }
  __syncthreads();
  if (!s_any) return;
  if (tid == 0) atomicAdd(&ctl[gi].rot, 1);

  // inner FP64 Hermitian Jacobi on G, accumulating W
  const int grp = tid >> 4, t16 = tid & 15;
  for (int isw = 0; isw < 3; ++isw) {  // partial diagonalisation: the outer sweeps re-check fresh Grams
    if (tid == 0) s_inner = 0;
    __syncthreads();
    for (int rr = 0; rr < PW - 1; ++rr) {
      int p, q;
      circle_pair(grp, rr, PW, p, q);
      if (t16 == 0) {
        double al = Gs[p][p].x, be = Gs[q][q].x;
        double2 gm = Gs[p][q];
        double g = sqrt(gm.x * gm.x + gm.y * gm.y);
        double c = 1.0, s = 0.0, er = 1.0, ei = 0.0;
        if (fmin(al, be) > skip && g > 1e-12 * sqrt(al * be)) {
          er = gm.x / g; ei = gm.y / g;
          double zeta = (be - al) / (2.0 * g);
          double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
          c = 1.0 / sqrt(1.0 + t * t);
          s = c * t;
          s_inner = 1;
        }
        rc[grp][0] = c; rc[grp][1] = s; rc[grp][2] = er; rc[grp][3] = ei;
      }
      __syncthreads();
      {
        double c = rc[grp][0], s = rc[grp][1], er = rc[grp][2], ei = rc[grp][3];
        if (s != 0.0) {
          // columns: x' = c x - s conj(e) y ; y' = s x + c conj(e) y   (G J and W J)
          for (int x = t16; x < PW; x += 16) {
            double2 a = Gs[x][p], b = Gs[x][q];
            double2 eb = make_double2(er * b.x + ei * b.y, er * b.y - ei * b.x);
            Gs[x][p] = make_double2(c * a.x - s * eb.x, c * a.y - s * eb.y);
            Gs[x][q] = make_double2(s * a.x + c * eb.x, s * a.y + c * eb.y);
            a = Ws[x][p]; b = Ws[x][q];
            eb = make_double2(er * b.x + ei * b.y, er * b.y - ei * b.x);
            Ws[x][p] = make_double2(c * a.x - s * eb.x, c * a.y - s * eb.y);
            Ws[x][q] = make_double2(s * a.x + c * eb.x, s * a.y + c * eb.y);
          }
        }
      }
      __syncthreads();
      {
        double c = rc[grp][0], s = rc[grp][1], er = rc[grp][2], ei = rc[grp][3];
        if (s != 0.0) {
          // rows (J^H G): x' = c x - s e y ; y' = s x + c e y
          for (int x = t16; x < PW; x += 16) {
            double2 a = Gs[p][x], b = Gs[q][x];
            double2 eb = make_double2(er * b.x - ei * b.y, er * b.y + ei * b.x);
            Gs[p][x] = make_double2(c * a.x - s * eb.x, c * a.y - s * eb.y);
            Gs[q][x] = make_double2(s * a.x + c * eb.x, s * a.y + c * eb.y);
          }
        }
      }
      __syncthreads();
    }
    const bool again = s_inner != 0;
    __syncthreads();  // every thread has read s_inner before thread 0 resets it
    if (!again) break;
  }
  for (int x = tid; x < PW * PW; x += 256) {
    int a = x / PW, b = x % PW;
    Wf[a][b] = make_float2((float)Ws[a][b].x, (float)Ws[a][b].y);
  }
  __syncthreads();

  // ---- C. block rotation of theta and V panels: P <- P W
  const int oi = tid & (RC - 1), oj = (tid >> 6) * 8;
  for (int pass = 0; pass < 2; ++pass) {
    float2* M = pass == 0 ? th : V;
    const int rows = pass == 0 ? m : np;
    const int ld = pass == 0 ? m : np;
    for (int r0 = 0; r0 < rows; r0 += RC) {
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        int i = tid & (RC - 1), c = (tid >> 6) + 4 * it;
        int row = r0 + i;
        Ps[i][c] = row < rows ? M[(int64_t)colof(c) * ld + row] : make_float2(0.f, 0.f);
      }
      __syncthreads();
      float2 out[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) out[j] = make_float2(0.f, 0.f);
      for (int c = 0; c < PW; ++c) {
        float2 x = Ps[oi][c];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float2 w = Wf[c][oj + j];
          out[j].x = fmaf(x.x, w.x, fmaf(-x.y, w.y, out[j].x));
          out[j].y = fmaf(x.x, w.y, fmaf(x.y, w.x, out[j].y));
        }
      }
      int row = r0 + oi;
      if (row < rows) {
#pragma unroll
        for (int j = 0; j < 8; ++j) M[(int64_t)colof(oj + j) * ld + row] = out[j];
      }
      __syncthreads();
    }
  }
}

__global__ void k_block_check(GateDesc* desc, const int32_t* list, int count, LargeCtl* ctl, int32_t* unconv,
                              int final_sweep) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int g = threadIdx.x; g < count; g += blockDim.x) {
    if (ctl[g].conv) continue;
    GateDesc& gd = desc[list[g]];
    gd.sweeps += 1;
    if (ctl[g].rot == 0) ctl[g].conv = 1;
    else atomicAdd(&cnt, 1);
    ctl[g].rot = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) *unconv = cnt;
  (void)final_sweep;
}

// sigma_j^2 = ||theta v_j||^2 / ||v_j||^2 with theta = lambda (x) Theta' (the FP32 theta the
// Jacobi started from), FP64 accumulation. One CTA per (32-column block, gate).
__global__ void __launch_bounds__(256) k_rayleigh(const GateDesc* __restrict__ desc, const int32_t* list, uint8_t* slab,
                                                  const DevState* st) {
  const GateDesc gd = desc[list[blockIdx.y]];
  const int j0 = blockIdx.x * 32;
  if (j0 >= gd.n) return;
  const int m = gd.m, n = gd.n, np = gd.n_pad, dd = st->d;
  const BondEntry* bonds = reinterpret_cast<const BondEntry*>(slab + st->bonds_off);
  const float* lam = reinterpret_cast<const float*>(slab + bonds[gd.site].off);
  const float2* thp = reinterpret_cast<const float2*>(slab + gd.ws_thetap);
  const float2* V = reinterpret_cast<const float2*>(slab + gd.ws_V);
  __shared__ float2 As[16][RC + 1];
  __shared__ float2 Bs[16][33];
  __shared__ double red[4][RC];
  const int tid = threadIdx.x;
  const int oi = tid & (RC - 1), oj = (tid >> 6) * 8;   // 64 rows x (4 groups x 8 columns)
  double num[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) num[j] = 0.0;
  for (int r0 = 0; r0 < m; r0 += RC) {
    double2 w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) w[j] = make_double2(0.0, 0.0);
    for (int k0 = 0; k0 < n; k0 += 16) {
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        int e = tid + it * 256;  // 1024 = 16 k x 64 rows
        int i = e & (RC - 1), kk = e >> 6;
        int row = r0 + i, k = k0 + kk;
        float2 v = make_float2(0.f, 0.f);
        if (row < m && k < n) {
          float2 tp = thp[(int64_t)k * m + row];
          float la = lam[row / dd];
          v = make_float2(la * tp.x, la * tp.y);
        }
        As[kk][i] = v;
      }
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        int e = tid + it * 256;  // 512 = 32 j x 16 k
        int kk = e & 15, jj = e >> 4;
        int k = k0 + kk, j = j0 + jj;
        Bs[kk][jj] = (k < n && j < n) ? V[(int64_t)j * np + k] : make_float2(0.f, 0.f);
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        float2 a = As[kk][oi];
        double ax = a.x, ay = a.y;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float2 b = Bs[kk][oj + j];
          w[j].x = fma(ax, (double)b.x, fma(-ay, (double)b.y, w[j].x));
          w[j].y = fma(ax, (double)b.y, fma(ay, (double)b.x, w[j].y));
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) num[j] += w[j].x * w[j].x + w[j].y * w[j].y;
  }
  // reduce num over the 64 row-threads of each column group (fixed order -> deterministic)
  __shared__ double colsum[32];
  const int grp = tid >> 6;
  for (int jj = 0; jj < 8; ++jj) {
    red[grp][oi] = num[jj];
    __syncthreads();
    if (oi == 0) {
      double sum = 0.0;
      for (int i = 0; i < RC; ++i) sum += red[grp][i];
      colsum[oj + jj] = sum;
    }
    __syncthreads();
  }
  if (tid < 32) {
    int j = j0 + tid;
    if (j < n) {
      double den = 0.0;
      const float2* vj = V + (int64_t)j * np;
      for (int k = 0; k < n; ++k) den += (double)vj[k].x * vj[k].x + (double)vj[k].y * vj[k].y;
      double v = den > 0.0 ? colsum[tid] / den : 0.0;
      reinterpret_cast<double*>(slab + gd.ws_sig2)[j] = v;
    }
  }
}

__global__ void k_sort_tails_large(GateDesc* desc, const int32_t* list, uint8_t* slab, DevState* st) {
  extern __shared__ __align__(16) uint8_t sm[];
  const GateDesc gd = desc[list[blockIdx.x]];
  const int n = gd.n;
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  double* keys = reinterpret_cast<double*>(sm);
  int32_t* idx = reinterpret_cast<int32_t*>(keys + npow2);
  double* part = reinterpret_cast<double*>(idx + npow2 + (npow2 & 1));
  double* gS = reinterpret_cast<double*>(slab + gd.ws_sig2);
  for (int j = threadIdx.x; j < npow2; j += blockDim.x) {
    double v = j < n ? gS[j] : -1.0;
    if (j < n && !isfinite(v)) atomicCAS(&st->led.error, 0, -7);
    keys[j] = v;
    idx[j] = j;
  }
  __syncthreads();
  cta_sort_desc(keys, idx, npow2);
  int32_t* gP = reinterpret_cast<int32_t*>(slab + gd.ws_pi);
  for (int j = threadIdx.x; j < n; j += blockDim.x) { gS[j] = keys[j]; gP[j] = idx[j]; }
  cta_tails(keys, n, reinterpret_cast<double*>(slab + gd.ws_T), part);
}

}  // namespace

int run_svd_blocked(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* d_list, const int32_t* h_list, int count,
                    int max_sweeps, uint8_t* slab, DevState* st, int32_t* d_scratch, int32_t* h_pinned_flag,
                    cudaStream_t s, int* error_out) {
  *error_out = 0;
  if (count <= 0) return 0;
  int launches = 0;
  int max_np = 0, max_n = 0;
  for (int g = 0; g < count; ++g) {
    max_np = max(max_np, h_desc[h_list[g]].n_pad);
    max_n = max(max_n, h_desc[h_list[g]].n);
  }
  // scratch layout: ctl[count] | norm2[count] (8-aligned) | unconv
  LargeCtl* ctl = reinterpret_cast<LargeCtl*>(d_scratch);
  double* norm2 = reinterpret_cast<double*>(d_scratch + 2 * ((count + 1) & ~1));
  int32_t* unconv = reinterpret_cast<int32_t*>(norm2 + count);
  cudaMemsetAsync(ctl, 0, sizeof(LargeCtl) * count, s);
  k_large_init<<<dim3(256, count), 256, 0, s>>>(d_desc, d_list, slab);
  k_large_norm<<<count, 256, 0, s>>>(d_desc, d_list, slab, norm2);
  launches += 2;
  const int nb_max = max_np / BLK;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_block_round, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRoundSmem);
    attr = true;
  }
  int sweep = 0;
  bool done = false;
  for (; sweep < max_sweeps && !done; ++sweep) {
    for (int rnd = 0; rnd < nb_max - 1; ++rnd) {
      // gates with fewer blocks simply have fewer rounds: rounds >= nb-1 are skipped by them
      k_block_round<<<dim3(nb_max / 2, count), 256, kRoundSmem, s>>>(d_desc, d_list, rnd, slab, ctl, norm2);
      ++launches;
    }
    k_block_check<<<1, 256, 0, s>>>(d_desc, d_list, count, ctl, unconv, 0);
    ++launches;
    cudaMemcpyAsync(h_pinned_flag, unconv, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    done = (*h_pinned_flag == 0);
  }
  if (!done) *error_out = -6;
  k_rayleigh<<<dim3((max_n + 31) / 32, count), 256, 0, s>>>(d_desc, d_list, slab, st);
  int npow2 = 1;
  while (npow2 < max_n) npow2 <<= 1;
  size_t smem = (size_t)npow2 * 12 + 16 + 1024 * 8;
  cudaFuncSetAttribute(k_sort_tails_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_sort_tails_large<<<count, 1024, smem, s>>>(d_desc, d_list, slab, st);
  launches += 2;
  return launches;
}

}  // namespace eamps
