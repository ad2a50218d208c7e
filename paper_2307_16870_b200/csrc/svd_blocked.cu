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
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "eamps_internal.cuh"
#include "jacobi_common.cuh"
#include "sort_tails.cuh"
#include "tc_common.cuh"

namespace eamps {

// EAMPS_DEBUG_SYNC=1 (development): synchronise and check after every large-regime launch, naming
// the kernel that faulted (the library's own bounds/alignment checks stand in for compute-sanitizer,
// which is closed on this pool).
static void dbg_sync(cudaStream_t s, const char* what) {
  static const bool on = getenv("EAMPS_DEBUG_SYNC") != nullptr;
  if (!on) return;
  cudaStreamSynchronize(s);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "[eamps debug] after %s: %s\n", what, cudaGetErrorString(e));
}


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
  if (gd.jrows > 0) return;   // preconditioned: B (with its zero pad columns) and V written elsewhere
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
  __shared__ int cnt, tot;
  if (threadIdx.x == 0) cnt = tot = 0;
  __syncthreads();
  for (int g = threadIdx.x; g < count; g += blockDim.x) {
    if (ctl[g].conv) continue;
    GateDesc& gd = desc[list[g]];
    gd.sweeps += 1;
    if (ctl[g].rot == 0) ctl[g].conv = 1;
    else atomicAdd(&cnt, 1);
    atomicAdd(&tot, ctl[g].rot);
    ctl[g].rot = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unconv[0] = cnt;
    unconv[1] = tot;   // rotated block pairs this sweep (diagnostics)
  }
  (void)final_sweep;
}

// sigma_j^2 = ||theta v_j||^2 / ||v_j||^2 with theta = lambda (x) Theta' (the FP32 theta the
// Jacobi started from), FP64 accumulation. One CTA per (32-column block, gate).
// QR-regime gates preconditioned by the FP64 Gram + Cholesky (G = theta^H theta = L L^H, L still in
// the precond scratch at ws_log, column-major, lower) take ||theta v||^2 = v^H G v = ||L^H v||^2
// instead: L^H is n x n upper triangular, so the row chunk r0 only needs k >= r0 -- half the FP64
// products of theta V (m x n). Accuracy: the FP64 Gram and Cholesky carry ~eps64 ||theta||^2 of
// absolute error in sigma_j^2, i.e. eps64 kappa^2 relative; the gates this does not resolve
// (sigma_min < 2e-4 sigma_max, kappa^2 > 2.5e7) are re-solved by the FP64 refinement (refine.cu)
// from a recontracted theta anyway. B = L^H V has the Gram of theta V (V^H G V), which is all the
// polish reads from it (rows n .. m-1 are written as zeros).
__global__ void __launch_bounds__(256) k_rayleigh(const GateDesc* __restrict__ desc, const int32_t* list, uint8_t* slab,
                                                  const DevState* st, int write_b = 0, int use_l = 0) {
  const GateDesc gd = desc[list[blockIdx.y]];
  const int j0 = blockIdx.x * 32;
  if (j0 >= gd.n) return;
  const int m = gd.m, n = gd.n, np = gd.n_pad, dd = st->d;
  static_assert(RC % 16 == 0, "row chunks start on a k chunk");
  const bool from_l = use_l && gd.regime == 3 && gd.jrows > 0;
  const int rows = from_l ? n : m;
  const double2* __restrict__ Lg = reinterpret_cast<const double2*>(slab + gd.ws_log);
  const BondEntry* bonds = reinterpret_cast<const BondEntry*>(slab + st->bonds_off);
  const float* lam = reinterpret_cast<const float*>(slab + bonds[gd.site].off);
  const float2* thp = reinterpret_cast<const float2*>(slab + gd.ws_thetap);
  const float2* V = reinterpret_cast<const float2*>(slab + gd.ws_V);
  // tiles are staged in FP64 (one conversion per element per chunk, not one per product)
  __shared__ double2 As[16][RC + 1];
  __shared__ double2 Bs[16][33];
  __shared__ double red[8][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int oi = tid & (RC - 1), oj = (tid >> 6) * 8;   // 64 rows x (4 groups x 8 columns)
  double num[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) num[j] = 0.0;
  // theta (= lambda (x) Theta', FP32) and V tiles of the next 16-column chunk are fetched into
  // registers while the current chunk's FP64 products run (one barrier pair per chunk)
  auto fetch = [&](int r0, int k0, double2* ra, float2* rb) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int e = tid + it * 256;  // 1024 = 16 k x 64 rows
      const int i = e & (RC - 1), kk = e >> 6;
      const int row = r0 + i, k = k0 + kk;
      double2 v = make_double2(0.0, 0.0);
      if (from_l) {
        if (row < n && k < n && k >= row) {            // (L^H)[row][k] = conj(L[k][row])
          const double2 l = Lg[(int64_t)row * n + k];
          v = make_double2(l.x, -l.y);
        }
      } else if (row < m && k < n) {
        const float2 tp = thp[(int64_t)k * m + row];
        const float la = lam[row / dd];
        v = make_double2(la * tp.x, la * tp.y);
      }
      ra[it] = v;
    }
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int e = tid + it * 256;  // 512 = 32 j x 16 k
      const int kk = e & 15, jj = e >> 4;
      const int k = k0 + kk, j = j0 + jj;
      rb[it] = (k < n && j < n) ? V[(int64_t)j * np + k] : make_float2(0.f, 0.f);
    }
  };
  const int nk = (n + 15) / 16;
  for (int r0 = 0; r0 < rows; r0 += RC) {
    double2 w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) w[j] = make_double2(0.0, 0.0);
    double2 ra[4];
    float2 rb[2];
    const int kc0 = from_l ? r0 / 16 : 0;               // L^H: rows r0.. need k >= r0 only
    fetch(r0, kc0 * 16, ra, rb);
    for (int kc = kc0; kc < nk; ++kc) {
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int e = tid + it * 256;
        As[e >> 6][e & (RC - 1)] = ra[it];
      }
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const int e = tid + it * 256;
        Bs[e & 15][e >> 4] = make_double2(rb[it].x, rb[it].y);
      }
      __syncthreads();
      if (kc + 1 < nk) fetch(r0, (kc + 1) * 16, ra, rb);
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const double2 a = As[kk][oi];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double2 bq = Bs[kk][oj + j];
          w[j].x = fma(a.x, bq.x, fma(-a.y, bq.y, w[j].x));
          w[j].y = fma(a.x, bq.y, fma(a.y, bq.x, w[j].y));
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) num[j] += w[j].x * w[j].x + w[j].y * w[j].y;
    if (write_b) {   // B = theta V for the FP64-anchored polish (the Jacobi's working theta is dead now)
      float2* Bw = reinterpret_cast<float2*>(slab + gd.ws_theta);
      const int row = r0 + oi;
      if (row < rows) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + oj + j < n) Bw[(int64_t)(j0 + oj + j) * m + row] = make_float2((float)w[j].x, (float)w[j].y);
      }
    }
  }
  if (write_b && rows < m) {   // L^H V has n rows: the polish reads m, the rest are zero
    float2* Bw = reinterpret_cast<float2*>(slab + gd.ws_theta);
    for (int x = tid; x < 32 * (m - rows); x += 256) {
      const int j = j0 + x / (m - rows), row = rows + x % (m - rows);
      if (j < n) Bw[(int64_t)j * m + row] = make_float2(0.f, 0.f);
    }
  }
  // reduce num over the 64 row-threads of each column group: warp butterflies, then the two warps
  // of a group in a fixed order (deterministic)
#pragma unroll
  for (int j = 0; j < 8; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) num[j] += __shfl_xor_sync(0xffffffffu, num[j], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) red[warp][j] = num[j];
  }
  // den_j = |v_j|^2: warp w handles columns 4w .. 4w+3, lanes stride over k (coalesced)
  double den[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int j = j0 + warp * 4 + c;
    double d = 0.0;
    if (j < n) {
      const float2* vj = V + (int64_t)j * np;
      for (int k = lane; k < n; k += 32) d += (double)vj[k].x * vj[k].x + (double)vj[k].y * vj[k].y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    den[c] = d;
  }
  __syncthreads();
  if (lane < 4) {
    const int jl = warp * 4 + lane, j = j0 + jl;    // column jl belongs to group jl / 8 = warps 2g, 2g+1
    const double dj = lane == 0 ? den[0] : lane == 1 ? den[1] : lane == 2 ? den[2] : den[3];
    if (j < n) {
      const int g = jl >> 3, jj = jl & 7;
      const double numj = red[2 * g][jj] + red[2 * g + 1][jj];
      const double v = dj > 0.0 ? numj / dj : 0.0;
      reinterpret_cast<double*>(slab + gd.ws_sig2)[j] = v;
      if (write_b) {   // polish scratch at ws_E: shift[n_pad] | den[n_pad]
        double* shift = reinterpret_cast<double*>(slab + gd.ws_E);
        shift[j] = 0.0;
        shift[np + j] = dj;
      }
    }
  }
}

// The same Rayleigh quotients and B as k_rayleigh (write_b = 1), on 64 x 64 output tiles: one CTA per
// (64-column block, gate), a 16 x 16 thread grid with 4 rows x 4 columns of W = A V per thread (A = L^H
// or lambda (x) Theta' as in k_rayleigh), k chunks of 16 double-buffered in shared memory (one barrier
// per chunk, the next chunk fetched into registers while the current one multiplies). Per k step a warp
// reads 8 shared double2 (4 rows: 16 distinct addresses, 4 columns: 2) for 16 complex FMAs (k_rayleigh:
// 9 for 8), and the L^H chunk is fetched along k (contiguous in the column-major L; k_rayleigh strides
// rows of L by n). Same products, different FP64 summation order (rows 4 at a time per thread, then the
// 16 row lanes by a butterfly). ncu r02: k_rayleigh ran at 0.34 of the FP64 peak (4.16 ms per chi = 64
// step). EAMPS_RAYLEIGH_OLD=1 keeps k_rayleigh (A/B).
constexpr int RT_K = 16, RT_P = 65;
constexpr size_t kRay64Half = sizeof(double2) * 2 * RT_K * RT_P;   // 33 KB per operand
__global__ void __launch_bounds__(256, 2) k_rayleigh64(const GateDesc* __restrict__ desc, const int32_t* list,
                                                       uint8_t* slab, const DevState* st, int use_l) {
  const GateDesc gd = desc[list[blockIdx.y]];
  const int j0 = blockIdx.x * 64;
  if (j0 >= gd.n) return;
  const int m = gd.m, n = gd.n, np = gd.n_pad, dd = st->d;
  const bool from_l = use_l && gd.regime == 3 && gd.jrows > 0;
  const int rows = from_l ? n : m;
  const double2* __restrict__ Lg = reinterpret_cast<const double2*>(slab + gd.ws_log);
  const BondEntry* bonds = reinterpret_cast<const BondEntry*>(slab + st->bonds_off);
  const float* lam = reinterpret_cast<const float*>(slab + bonds[gd.site].off);
  const float2* thp = reinterpret_cast<const float2*>(slab + gd.ws_thetap);
  const float2* V = reinterpret_cast<const float2*>(slab + gd.ws_V);
  float2* Bw = reinterpret_cast<float2*>(slab + gd.ws_theta);
  extern __shared__ __align__(16) uint8_t r64_sm[];
  double2 (*As)[RT_K][RT_P] = reinterpret_cast<double2 (*)[RT_K][RT_P]>(r64_sm);                   // [buf][k][row]
  double2 (*Bs)[RT_K][RT_P] = reinterpret_cast<double2 (*)[RT_K][RT_P]>(r64_sm + kRay64Half);      // [buf][k][col]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid & 15, ty = tid >> 4;   // rows tx + 16a, columns ty + 16b
  double num[4] = {0.0, 0.0, 0.0, 0.0};
  double2 ra[4];
  float2 rb[4];
  auto fetch = [&](int r0, int k0) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int e = tid + it * 256;          // 1024 = 16 k x 64 rows
      double2 v = make_double2(0.0, 0.0);
      if (from_l) {                          // along k: (L^H)[row][k] = conj(L[k][row]) = conj(Lg[row n + k])
        const int kk = e & 15, row = r0 + (e >> 4), k = k0 + kk;
        if (row < n && k < n && k >= row) {
          const double2 l = Lg[(int64_t)row * n + k];
          v = make_double2(l.x, -l.y);
        }
      } else {                               // along rows: theta'[k][row], column-major ld m
        const int row = r0 + (e & 63), k = k0 + (e >> 6);
        if (row < m && k < n) {
          const float2 tp = thp[(int64_t)k * m + row];
          const float la = lam[row / dd];
          v = make_double2(la * tp.x, la * tp.y);
        }
      }
      ra[it] = v;
      const int kk = e & 15, jj = e >> 4, k = k0 + kk, j = j0 + jj;
      rb[it] = (k < n && j < n) ? V[(int64_t)j * np + k] : make_float2(0.f, 0.f);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int e = tid + it * 256;
      if (from_l) As[buf][e & 15][e >> 4] = ra[it];
      else As[buf][e >> 6][e & 63] = ra[it];
      Bs[buf][e & 15][e >> 4] = make_double2(rb[it].x, rb[it].y);
    }
  };
  const int nk = (n + RT_K - 1) / RT_K;
  for (int r0 = 0; r0 < rows; r0 += 64) {
    double2 w[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) w[a][b] = make_double2(0.0, 0.0);
    const int kc0 = from_l ? r0 / RT_K : 0;           // L^H: rows r0.. need k >= r0 only
    fetch(r0, kc0 * RT_K);
    stash(0);
    __syncthreads();
    for (int kc = kc0; kc < nk; ++kc) {
      const int cur = (kc - kc0) & 1;
      if (kc + 1 < nk) fetch(r0, (kc + 1) * RT_K);
#pragma unroll
      for (int kk = 0; kk < RT_K; ++kk) {
        double2 a[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) a[p] = As[cur][kk][tx + 16 * p];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 b = Bs[cur][kk][ty + 16 * q];
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            w[p][q].x = fma(a[p].x, b.x, fma(-a[p].y, b.y, w[p][q].x));
            w[p][q].y = fma(a[p].x, b.y, fma(a[p].y, b.x, w[p][q].y));
          }
        }
      }
      if (kc + 1 < nk) stash(cur ^ 1);   // the other buffer: last read before the previous barrier
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + ty + 16 * q;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int row = r0 + tx + 16 * p;
        num[q] += w[p][q].x * w[p][q].x + w[p][q].y * w[p][q].y;   // zero beyond rows / n
        if (row < rows && j < n) Bw[(int64_t)j * m + row] = make_float2((float)w[p][q].x, (float)w[p][q].y);
      }
    }
  }
  if (rows < m) {   // L^H V has n rows: the polish reads m, the rest are zero
    for (int x = tid; x < 64 * (m - rows); x += 256) {
      const int j = j0 + x / (m - rows), row = rows + x % (m - rows);
      if (j < n) Bw[(int64_t)j * m + row] = make_float2(0.f, 0.f);
    }
  }
  // num: the 16 row lanes (tx) of each half-warp hold one column set ty; butterfly over them
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) num[q] += __shfl_xor_sync(0xffffffffu, num[q], o);
  }
  __shared__ double s_num[64];
  if (tx == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) s_num[ty + 16 * q] = num[q];
  }
  __syncthreads();
  // den_j = |v_j|^2 and the outputs: warp w handles columns 8w .. 8w+7, lanes stride over k
  double* sig2 = reinterpret_cast<double*>(slab + gd.ws_sig2);
  double* shift = reinterpret_cast<double*>(slab + gd.ws_E);   // polish scratch: shift[n_pad] | den[n_pad]
  for (int c = 0; c < 8; ++c) {
    const int jl = warp * 8 + c, j = j0 + jl;
    if (j >= n) break;
    const float2* vj = V + (int64_t)j * np;
    double d = 0.0;
    for (int k = lane; k < n; k += 32) d += (double)vj[k].x * vj[k].x + (double)vj[k].y * vj[k].y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0) {
      sig2[j] = d > 0.0 ? s_num[jl] / d : 0.0;
      shift[j] = 0.0;
      shift[np + j] = d;
    }
  }
}

__global__ void k_sort_tails_large(GateDesc* desc, const int32_t* list, uint8_t* slab, DevState* st, int polish = 0) {
  extern __shared__ __align__(16) uint8_t sm[];
  const GateDesc gd = desc[list[blockIdx.x]];
  const int n = gd.n;
  int npow2 = 1;
  while (npow2 < n) npow2 <<= 1;
  double* keys = reinterpret_cast<double*>(sm);
  int32_t* idx = reinterpret_cast<int32_t*>(keys + npow2);
  double* part = reinterpret_cast<double*>(idx + npow2 + (npow2 & 1));
  double* gS = reinterpret_cast<double*>(slab + gd.ws_sig2);
  const double* shift = reinterpret_cast<const double*>(slab + gd.ws_E);
  for (int j = threadIdx.x; j < npow2; j += blockDim.x) {
    double v = j < n ? gS[j] + (polish ? shift[j] : 0.0) : -1.0;
    if (j < n && v < 0.0) v = 0.0;
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


// =================================================================================================
// Tensor-core (tcgen05, 3xTF32) blocked one-sided Jacobi -- the large regime on sm_100a.
//
// Columns in blocks of TB = 32; a round pairs blocks (I, J) by the circle method; the panel
// P = [A_I A_J] (m x 64 complex) is handled by three kernels per round (all gates, all pairs):
//   k_tc_gram  : G = P^H P on the tensor core. With Q = [Re P | Im P] (m x 128 real, staged
//                K-major from theta's columns), D = Q^T Q (128 x 128, K = m) and
//                G_re = D[p][q] + D[64+p][64+q], G_im = D[p][64+q] - D[64+p][q]. 3xTF32 by the
//                symmetric form D'' = hi^T hi + hi^T (2 lo), D = (D'' + D''^T)/2 (2 MMAs / k-step).
//   k_tc_inner : the one-sided Jacobi criterion on G (as the SIMT path), then cyclic two-sided
//                Jacobi on G in FP64 (the scalar 2x2 rotation), W = prod J, E = W - I split into
//                TF32 hi + lo images laid out for the rotation's B operand.
//   k_tc_rot   : P <- P + P E (identity split: the tensor-core error scales with |E|, which goes
//                to 0 as the sweep converges) for the theta panel (m rows) and the V panel
//                (n_pad rows), 128-row tiles, [Re' Im'] = [Re Im] [[E_re, E_im], [-E_im, E_re]]
//                as 4 K=64 x N=64 MMA groups per tile (b_negate for -E_im), 3xTF32.
// =================================================================================================
namespace tcj {

constexpr int TB = 32;          // complex columns per block
constexpr int PWC = 2 * TB;     // panel width (complex) = 64
constexpr int GKC = 32;         // rows per Gram K-chunk
constexpr uint32_t G_SBO = 128, G_LBO = (128 / 8) * 128;   // Gram operand image: 128 rows (panel re/im cols)
constexpr uint32_t E_SBO = 128, E_LBO = (64 / 8) * 128;    // E image: 64 rows (output cols) x 64 k
constexpr uint32_t R_SBO = 128, R_LBO = (128 / 8) * 128;   // rotation A image: 128 rows x 16 k
constexpr int EIMG_FLOATS = 4 * 64 * 64;                   // Re hi|lo, Im hi|lo
constexpr size_t kGramStage = (size_t)128 * GKC * 4;        // one image (hi or lo2) of a chunk: 16 KB
constexpr size_t kGramSmem = 4 * (size_t)128 * 32 * 4 + 2 * (size_t)64 * 288 + 1024;  // images | raw ring (>= D staging)
constexpr size_t kRotStage = (size_t)128 * 16 * 4;          // one image of a 128 x 16 chunk: 8 KB
constexpr size_t kRotSmem = (size_t)EIMG_FLOATS * 4 + 2 * (size_t)64 * 128 * 8 + 2 * 2 * kRotStage + 1024;
constexpr size_t kInnerSmem = 2 * sizeof(float2) * 64 * 65;
constexpr int kInnerT = 512;   // threads of the inner solve (more warps per SM hide shared-memory latency)

struct Scratch {                  // per gate: slab offset of its TC scratch (GateDesc::ws_log)
  static __host__ __device__ size_t gram_bytes(int pairs) { return (size_t)pairs * 64 * 64 * 8; }
  static __host__ __device__ size_t eimg_bytes(int pairs) { return (size_t)pairs * EIMG_FLOATS * 4; }
  static __host__ __device__ size_t total(int pairs) { return gram_bytes(pairs) + eimg_bytes(pairs) + (size_t)pairs * 4 + 256; }
};

__device__ __forceinline__ int colof(int c, int I, int J) { return c < TB ? I * TB + c : J * TB + (c - TB); }

// ---- panel Gram on the tensor core: D (128 x 128 real, in shared memory Ds[128][129]) = Q^T Q,
// Q = [Re P | Im P] of the 64 complex columns colof(0..63) of M (m rows, ld m; columns >= ncols read
// as zero). Raw 32-row chunks arrive by cp.async through a GR-deep ring (pitch 288 B per column),
// are split into TF32 hi / 2*lo images (double-buffered) and fed to 2 MMAs per k-step
// (symmetric 3xTF32: D = sym(hi^T hi + hi^T 2lo)). 128 threads. Shared memory: kGramSmem.
constexpr int GR = 2;                                   // raw ring depth
constexpr uint32_t GRAW_PITCH = 288;                    // bytes per column of a raw chunk (32 rows + pad)
constexpr size_t kGramRaw = (size_t)64 * GRAW_PITCH;    // 18 KB
// kNamed: the 128 threads synchronise on named barrier 1 instead of __syncthreads (the fused
// kernel runs the Gram on warps 0-3 of a larger CTA).
__device__ __forceinline__ void bar128() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }
template <bool kNamed = false>
__device__ __forceinline__ void gram_panel(const float2* __restrict__ M, int m, int ncols, int I, int J,
                                           uint8_t* base, uint64_t* mbar, uint32_t tmem, float* Ds) {
  auto csync = [] {
    if constexpr (kNamed) bar128();
    else __syncthreads();
  };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* img = base;                                   // 2 x (hi, lo2) x 16 KB
  uint8_t* ring = base + 4 * kGramStage;                 // GR x 18 KB
  const int nchunks = (m + GKC - 1) / GKC;
  auto issue = [&](int q) {
    if (q < nchunks) {
      uint8_t* dst = ring + (size_t)(q % GR) * kGramRaw;
      const int r0 = q * GKC;
      // 64 columns x 32 rows x 8 B = 1024 x 16 B; 16 consecutive copies per column
      for (int x = tid; x < 1024; x += 128) {
        const int c = x >> 4, rp = (x & 15) * 2;
        const int col = colof(c, I, J), r = r0 + rp;
        float2* d = reinterpret_cast<float2*>(dst + c * GRAW_PITCH) + rp;
        if (col < ncols && r + 1 < m) {
          tc::cp_async16(d, M + (int64_t)col * m + r);
        } else {
          d[0] = (col < ncols && r < m) ? M[(int64_t)col * m + r] : make_float2(0.f, 0.f);
          d[1] = make_float2(0.f, 0.f);
        }
      }
    }
    tc::cp_async_commit();   // (possibly empty) group: keeps the wait_group count uniform
  };
  for (int q = 0; q < GR - 1; ++q) issue(q);
  const uint32_t idesc = tc::make_idesc_tf32(128, 128, false, false);
  for (int q = 0; q < nchunks; ++q) {
    issue(q + GR - 1);
    tc::cp_async_wait<GR - 1>();
    csync();                                     // raw chunk q visible to all
    const int b = q & 1;
    if (q >= 2) tc::mbar_wait(&mbar[b], ((q - 2) >> 1) & 1);
    uint8_t* hi = img + (size_t)b * 2 * kGramStage;
    uint8_t* lo2 = hi + kGramStage;
    const uint8_t* raw = ring + (size_t)(q % GR) * kGramRaw;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int c = lane + 32 * (warp & 1);
      const int rg = (warp >> 1) + 2 * it;
      const float4 v0 = *reinterpret_cast<const float4*>(raw + c * GRAW_PITCH + 32 * rg);
      const float4 v1 = *reinterpret_cast<const float4*>(raw + c * GRAW_PITCH + 32 * rg + 16);
      float4 rh, rl, ih, il;
      tc::split_tf32(v0.x, rh.x, rl.x); tc::split_tf32(v0.z, rh.y, rl.y);
      tc::split_tf32(v1.x, rh.z, rl.z); tc::split_tf32(v1.z, rh.w, rl.w);
      tc::split_tf32(v0.y, ih.x, il.x); tc::split_tf32(v0.w, ih.y, il.y);
      tc::split_tf32(v1.y, ih.z, il.z); tc::split_tf32(v1.w, ih.w, il.w);
      rl.x *= 2.f; rl.y *= 2.f; rl.z *= 2.f; rl.w *= 2.f;
      il.x *= 2.f; il.y *= 2.f; il.z *= 2.f; il.w *= 2.f;
      const uint32_t oR = tc::kmaj_off(c, 4 * rg, G_LBO, G_SBO), oI = tc::kmaj_off(64 + c, 4 * rg, G_LBO, G_SBO);
      *reinterpret_cast<float4*>(hi + oR) = rh;
      *reinterpret_cast<float4*>(lo2 + oR) = rl;
      *reinterpret_cast<float4*>(hi + oI) = ih;
      *reinterpret_cast<float4*>(lo2 + oI) = il;
    }
    tc::fence_async_smem();
    csync();                                     // images written; raw slot q%GR free
    if (tid == 0) {
      tc::fence_after_sync();
      const uint32_t ah = tc::smem_u32(hi), al = tc::smem_u32(lo2);
#pragma unroll
      for (int s = 0; s < GKC / 8; ++s) {
        const uint32_t off = 2 * s * G_LBO;
        const uint64_t dh = tc::make_desc(ah + off, G_LBO, G_SBO), dl = tc::make_desc(al + off, G_LBO, G_SBO);
        tc::mma_tf32(tmem, dh, dh, idesc, (q > 0 || s > 0) ? 1u : 0u);
        tc::mma_tf32(tmem, dh, dl, idesc, 1u);
      }
      tc::mma_commit(&mbar[b]);
    }
    __syncwarp();
  }
  tc::cp_async_wait<0>();
  tc::mbar_wait(&mbar[(nchunks - 1) & 1], ((nchunks - 1) >> 1) & 1);
  // (persistent use: the other barrier's last commit must have landed too before the barriers are
  // re-initialised for the next panel)
  if (kNamed && nchunks >= 2) tc::mbar_wait(&mbar[(nchunks - 2) & 1], ((nchunks - 2) >> 1) & 1);
  tc::fence_after_sync();
  csync();                                       // every thread past its last smem read
  const int row = warp * 32 + lane;
#pragma unroll 1
  for (int c = 0; c < 128; c += 8) {
    float v[8];
    tc::tmem_ld8(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
#pragma unroll
    for (int i = 0; i < 8; ++i) Ds[row * 129 + c + i] = v[i];
  }
  tc::fence_before_sync();
  csync();
}

__device__ __forceinline__ void tc_setup(uint64_t* mbar, uint32_t* tbase) {
  if ((threadIdx.x >> 5) == 0) tc::tmem_alloc(tbase, 128);
  if (threadIdx.x == 0) {
    tc::mbar_init(&mbar[0], 1);
    tc::mbar_init(&mbar[1], 1);
    tc::fence_barrier_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
}

// ---- G = P^H P of the round's panel. grid (n_pad/64 pairs max, count); 128 threads.
__global__ void __launch_bounds__(128) k_tc_gram(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                 int rnd, uint8_t* slab, const LargeCtl* ctl) {
  const int gi = blockIdx.y;
  if (ctl[gi].conv) return;
  const GateDesc& gd = desc[list[gi]];
  const int nb = gd.n_pad / TB, pair = blockIdx.x;
  if (pair >= nb / 2 || rnd >= nb - 1) return;
  int I, J;
  circle_pair(pair, rnd, nb, I, J);
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tbase;
  tc_setup(mbar, &tbase);
  float* Ds = reinterpret_cast<float*>(base);
  gram_panel(reinterpret_cast<const float2*>(slab + gd.ws_theta), jacobi_rows(gd), gd.n_pad, I, J, base, mbar, tbase, Ds);
  if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc(tbase, 128);
  float2* Gout = reinterpret_cast<float2*>(slab + gd.ws_log) + (size_t)pair * 64 * 64;
  auto sym = [&](int a, int b2) { return 0.5f * (Ds[a * 129 + b2] + Ds[b2 * 129 + a]); };
  for (int x = threadIdx.x; x < 64 * 64; x += 128) {
    const int p = x >> 6, qq = x & 63;
    Gout[x] = make_float2(sym(p, qq) + sym(64 + p, 64 + qq), sym(p, 64 + qq) - sym(64 + p, qq));
  }
}

// ---- inner Jacobi on G -> E = W - I images. grid (pairs max, count); 256 threads, FP32.
// One cyclic sweep (tournament order) of two-sided Jacobi on the 64 x 64 Hermitian G, the
// rotations accumulated into W; each rotation is computed redundantly by the 8 threads of its
// group (no broadcast round trip). W's FP32 drift from unitarity (~1e-6) is consistent between
// theta and V (the same E rotates both) and is absorbed by the Rayleigh normalisation and the
// FP64-anchored polish.
__global__ void __launch_bounds__(kInnerT) k_tc_inner(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                  int rnd, uint8_t* slab, LargeCtl* ctl, const double* norm2,
                                                  int inner_sweeps, float tol_floor, float tol_internal) {
  const int gi = blockIdx.y;
  if (ctl[gi].conv) return;
  const GateDesc& gd = desc[list[gi]];
  const int nb = gd.n_pad / TB, pair = blockIdx.x;
  if (pair >= nb / 2 || rnd >= nb - 1) return;
  const int pairs = gd.n_pad / PWC;
  const float2* Gin = reinterpret_cast<const float2*>(slab + gd.ws_log) + (size_t)pair * 64 * 64;
  float* Eimg = reinterpret_cast<float*>(slab + gd.ws_log + Scratch::gram_bytes(pairs)) + (size_t)pair * EIMG_FLOATS;
  int32_t* rflag = reinterpret_cast<int32_t*>(slab + gd.ws_log + Scratch::gram_bytes(pairs) + Scratch::eimg_bytes(pairs));
  extern __shared__ __align__(16) uint8_t dsm[];
  float2(*Gs)[65] = reinterpret_cast<float2(*)[65]>(dsm);
  float2(*Ws)[65] = Gs + 64;
  // G is Hermitian: only its upper triangle is kept current; (i, j) with i > j reads / writes the
  // conjugate at (j, i) (no mirror stores: a third of the shared-memory stores of a round)
  auto gld = [&](int i, int j) {
    const float2 v = Gs[min(i, j)][max(i, j)];
    return i <= j ? v : make_float2(v.x, -v.y);
  };
  auto gst = [&](int i, int j, float2 v) { Gs[min(i, j)][max(i, j)] = i <= j ? v : make_float2(v.x, -v.y); };
  const int tid = threadIdx.x;
  for (int x = tid; x < 64 * 64; x += kInnerT) {
    const int a = x >> 6, b = x & 63;
    Gs[a][b] = Gin[x];
    Ws[a][b] = make_float2(a == b ? 1.f : 0.f, 0.f);
  }
  __syncthreads();
  const float skip = (float)(norm2[gi] * 3.552713678800501e-15);  // (2^-24)^2 ||theta||^2
  const float tol = fmaxf(tol_floor, 4.f * sqrtf((float)jacobi_rows(gd)) * 5.960464477539063e-8f);
  const float tol_int = fmaxf(tol, tol_internal);
  int any = 0, internal = 0;
  for (int x = tid; x < 64 * 64; x += kInnerT) {
    const int p = x >> 6, q = x & 63;
    if (p < q) {
      const float al = Gs[p][p].x, be = Gs[q][q].x;
      const float g = sqrtf(Gs[p][q].x * Gs[p][q].x + Gs[p][q].y * Gs[p][q].y);
      if (fminf(al, be) > skip && g > tol * sqrtf(al) * sqrtf(be)) {
        any = 1;
        // within-block non-orthogonality above tol_int forces the full tournament (and round 0 of
        // every sweep always runs it, so each block's internal pairs are revisited once a sweep)
        if ((p < 32) == (q < 32) && (rnd == 0 || g > tol_int * sqrtf(al) * sqrtf(be))) internal = 1;
      }
    }
  }
  internal = __syncthreads_or(internal);
  if (!__syncthreads_or(any)) {
    if (tid == 0) rflag[pair] = 0;
    return;
  }
  if (tid == 0) {
    rflag[pair] = 1;
    atomicAdd(&ctl[gi].rot, 1);
  }
  // When both blocks are already internally orthogonal (to tol), the off-diagonal mass of G sits
  // in the I x J block and an inner sweep only needs the 32 x 32 cross pairs
  // (p = i, q = 32 + (i + rr) mod 32): 32 rounds. Otherwise the full 64-column tournament (63).
  // A round: (A) each of the 32 pairs computes its rotation J_k from its 2x2 diagonal block;
  // (B) every 2x2 block (pair a rows, pair b cols), a < b, becomes J_a^H X J_b in the upper triangle
  // (G Hermitian: half the work of separate column and row passes, one barrier fewer), and
  // W <- W J (columns p_k, q_k).
  __shared__ float4 par[32];      // c, s, er, ei
  __shared__ int2 pq[32];
  __shared__ uint16_t blk[496];   // the off-diagonal block pairs a < b
  for (int x = tid; x < 496; x += kInnerT) {
    int aa = 0, rem = x;
    while (rem >= 31 - aa) { rem -= 31 - aa; ++aa; }
    blk[x] = (uint16_t)(aa | ((aa + 1 + rem) << 8));
  }
  const int nrr = internal ? 63 : 32;
  for (int isw = 0; isw < inner_sweeps; ++isw) {
    int rot = 0;
    for (int rr = 0; rr < nrr; ++rr) {
      if (tid < 32) {
        int p, q;
        if (internal) {
          circle_pair(tid, rr, 64, p, q);
        } else {
          p = tid;
          q = 32 + ((tid + rr) & 31);
        }
        const float al = Gs[p][p].x, be = Gs[q][q].x;
        const float2 gm = gld(p, q);
        const float g2 = gm.x * gm.x + gm.y * gm.y;
        float c = 1.f, sn = 0.f, er = 1.f, ei = 0.f;
        if (fminf(al, be) > skip && g2 > 1e-13f * al * be) {
          const float ig = rsqrtf(g2);
          er = gm.x * ig;
          ei = gm.y * ig;
          const float zeta = 0.5f * (be - al) * ig;
          const float az = fabsf(zeta);
          const float t = copysignf(1.f, zeta) / (az + sqrtf(fmaf(az, az, 1.f)));
          c = rsqrtf(fmaf(t, t, 1.f));
          sn = c * t;
          rot = 1;
          // the pair's own 2x2 block J^H X J is diagonal: (alpha - t|gamma|, beta + t|gamma|)
          const float tg = t * (g2 * ig);
          Gs[p][p] = make_float2(al - tg, 0.f);
          Gs[q][q] = make_float2(be + tg, 0.f);
          gst(p, q, make_float2(0.f, 0.f));
        }
        par[tid] = make_float4(c, sn, er, ei);
        pq[tid] = make_int2(p, q);
      }
      __syncthreads();
      for (int x = tid; x < 496; x += kInnerT) {
        const int ia = blk[x] & 0xFF, ib = blk[x] >> 8;
        const float4 Ja = par[ia], Jb = par[ib];
        if (Ja.y == 0.f && Jb.y == 0.f) continue;
        const int2 ra = pq[ia], cb = pq[ib];
        float2 X[2][2] = {{gld(ra.x, cb.x), gld(ra.x, cb.y)}, {gld(ra.y, cb.x), gld(ra.y, cb.y)}};
        if (Jb.y != 0.f) {   // columns: (x, y) -> (c x - s conj(e) y, s x + c conj(e) y)
          const Rot rb{Jb.x, Jb.y, Jb.z, Jb.w};
#pragma unroll
          for (int r = 0; r < 2; ++r) apply_rot(X[r][0], X[r][1], rb);
        }
        if (Ja.y != 0.f) {   // rows: (u, v) -> (c u - s e v, s u + c e v), i.e. the rotation with conj(e) -> e
          const Rot ra{Ja.x, Ja.y, Ja.z, -Ja.w};
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) apply_rot(X[0][cc], X[1][cc], ra);
        }
        gst(ra.x, cb.x, X[0][0]); gst(ra.x, cb.y, X[0][1]);
        gst(ra.y, cb.x, X[1][0]); gst(ra.y, cb.y, X[1][1]);
      }
      {   // W <- W J for every pair: thread (pair k = tid / (T/32), rows tid % (T/32) + (T/32) i)
        const int k = tid / (kInnerT / 32);
        const float4 J = par[k];
        if (J.y != 0.f) {
          const int2 cq = pq[k];
#pragma unroll 4
          const Rot rw{J.x, J.y, J.z, J.w};
          for (int x = tid % (kInnerT / 32); x < 64; x += kInnerT / 32) {
            float2 xx = Ws[x][cq.x], yy = Ws[x][cq.y];
            apply_rot(xx, yy, rw);
            Ws[x][cq.x] = xx;
            Ws[x][cq.y] = yy;
          }
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rot)) break;
  }
  __syncthreads();
  // E = W - I as the rotation's B images (hi, lo), Re then Im: element (n = out col, k = in col) = E[k][n]
  for (int x = tid; x < 64 * 64; x += kInnerT) {
    const int k = x >> 6, n = x & 63;
    float2 w = Ws[k][n];
    if (k == n) w.x -= 1.f;
    const uint32_t o = tc::kmaj_off(n, k, E_LBO, E_SBO) >> 2;
    float h, l;
    tc::split_tf32(w.x, h, l);
    Eimg[o] = h;
    Eimg[4096 + o] = l;
    tc::split_tf32(w.y, h, l);
    Eimg[8192 + o] = h;
    Eimg[12288 + o] = l;
  }
}

// ---- P <- P + P E for theta (m rows) and V (n_pad rows) panels. grid (pairs max, count); 256 threads.
// Double-buffered raw 128-row tiles (64 KB each, cp.async: tile t+1 loads while tile t computes);
// thread (row, half) splits 4 of each 8-column chunk into TF32 hi/lo images; 3xTF32 MMAs
// (hi hi + hi lo + lo hi) for D_re/D_im with N = 64; epilogue P' = P + D from the raw tile.
__global__ void __launch_bounds__(256) k_tc_rot(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                int rnd, uint8_t* slab, const LargeCtl* ctl) {
  const int gi = blockIdx.y;
  if (ctl[gi].conv) return;
  const GateDesc& gd = desc[list[gi]];
  const int nb = gd.n_pad / TB, pair = blockIdx.x;
  if (pair >= nb / 2 || rnd >= nb - 1) return;
  const int pairs = gd.n_pad / PWC;
  const int32_t* rflag =
      reinterpret_cast<const int32_t*>(slab + gd.ws_log + Scratch::gram_bytes(pairs) + Scratch::eimg_bytes(pairs));
  if (!rflag[pair]) return;
  int I, J;
  circle_pair(pair, rnd, nb, I, J);
  const float* Eg = reinterpret_cast<const float*>(slab + gd.ws_log + Scratch::gram_bytes(pairs)) + (size_t)pair * EIMG_FLOATS;
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  float* Es = reinterpret_cast<float*>(base);                            // 64 KB: Re h|l, Im h|l
  float2* rawb = reinterpret_cast<float2*>(base + (size_t)EIMG_FLOATS * 4);   // 2 x [64 cols][128 rows]
  uint8_t* stg = reinterpret_cast<uint8_t*>(rawb + 2 * 64 * 128);       // 2 stages x (hi, lo) x 8 KB
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, row_l = tid & 127, half = tid >> 7;
  const int m = jacobi_rows(gd), np = gd.n_pad;   // preconditioned: B (n rows), no V tiles
  const int tiles_th = (m + 127) / 128, tiles_v = gd.jrows > 0 ? 0 : (np + 127) / 128, ntiles = tiles_th + tiles_v;
  for (int x = tid; x < EIMG_FLOATS / 4; x += 256) tc::cp_async16(Es + 4 * x, Eg + 4 * x);
  auto issue_tile = [&](int tile) {
    if (tile < ntiles) {
      const bool isV = tile >= tiles_th;
      const float2* M = reinterpret_cast<const float2*>(slab + (isV ? gd.ws_V : gd.ws_theta));
      const int rows = isV ? np : m;
      const int r0 = (isV ? tile - tiles_th : tile) * 128;
      float2* raw = rawb + (tile & 1) * 64 * 128;
      for (int x = tid; x < 64 * 64; x += 256) {
        const int c = x >> 6, rp = (x & 63) * 2;
        float2* dst = raw + c * 128 + rp;
        if (r0 + rp + 1 < rows) {
          tc::cp_async16(dst, M + (int64_t)colof(c, I, J) * rows + r0 + rp);
        } else {
          dst[0] = (r0 + rp < rows) ? M[(int64_t)colof(c, I, J) * rows + r0 + rp] : make_float2(0.f, 0.f);
          dst[1] = make_float2(0.f, 0.f);
        }
      }
    }
    tc::cp_async_commit();
  };
  issue_tile(0);
  tc_setup(mbar, &tbase);
  const uint32_t tmem = tbase;
  const uint32_t id_p = tc::make_idesc_tf32(128, 64, false, false);
  const uint32_t id_n = id_p | (1u << 14);   // negate B (-E_im)
  const uint32_t e0 = tc::smem_u32(Es);
  constexpr uint32_t EI = 16384;             // bytes per E image
  int chunk_ctr = 0;
  for (int tile = 0; tile < ntiles; ++tile) {
    const bool isV = tile >= tiles_th;
    float2* M = reinterpret_cast<float2*>(slab + (isV ? gd.ws_V : gd.ws_theta));
    const int rows = isV ? np : m;
    const int r0 = (isV ? tile - tiles_th : tile) * 128;
    const float2* raw = rawb + (tile & 1) * 64 * 128;
    issue_tile(tile + 1);                    // its buffer was released by tile - 1's epilogue
    tc::cp_async_wait<1>();
    __syncthreads();                         // raw tile (and E) visible to every thread
    for (int q = 0; q < PWC / 8; ++q, ++chunk_ctr) {
      const int b = chunk_ctr & 1;
      if (chunk_ctr >= 2) tc::mbar_wait(&mbar[b], ((chunk_ctr - 2) >> 1) & 1);
      uint8_t* im0 = stg + (size_t)b * 2 * kRotStage;
      // thread (row, half): complex columns 8q + 4 half .. +3 -> K 4half..4half+3 (Re), 8+4half.. (Im)
      float4 rh, rl, ih, il;
      {
        const float2 z0 = raw[(8 * q + 4 * half + 0) * 128 + row_l], z1 = raw[(8 * q + 4 * half + 1) * 128 + row_l];
        const float2 z2 = raw[(8 * q + 4 * half + 2) * 128 + row_l], z3 = raw[(8 * q + 4 * half + 3) * 128 + row_l];
        tc::split_tf32(z0.x, rh.x, rl.x); tc::split_tf32(z1.x, rh.y, rl.y);
        tc::split_tf32(z2.x, rh.z, rl.z); tc::split_tf32(z3.x, rh.w, rl.w);
        tc::split_tf32(z0.y, ih.x, il.x); tc::split_tf32(z1.y, ih.y, il.y);
        tc::split_tf32(z2.y, ih.z, il.z); tc::split_tf32(z3.y, ih.w, il.w);
      }
      const uint32_t oR = tc::kmaj_off(row_l, 4 * half, R_LBO, R_SBO), oI = tc::kmaj_off(row_l, 8 + 4 * half, R_LBO, R_SBO);
      *reinterpret_cast<float4*>(im0 + oR) = rh;
      *reinterpret_cast<float4*>(im0 + kRotStage + oR) = rl;
      *reinterpret_cast<float4*>(im0 + oI) = ih;
      *reinterpret_cast<float4*>(im0 + kRotStage + oI) = il;
      tc::fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t a0 = tc::smem_u32(im0);
        const uint32_t eoff = 2 * q * E_LBO;   // input columns 8q..8q+7
        const uint64_t aRh = tc::make_desc(a0, R_LBO, R_SBO), aRl = tc::make_desc(a0 + kRotStage, R_LBO, R_SBO);
        const uint64_t aIh = tc::make_desc(a0 + 2 * R_LBO, R_LBO, R_SBO);
        const uint64_t aIl = tc::make_desc(a0 + kRotStage + 2 * R_LBO, R_LBO, R_SBO);
        const uint64_t bRh = tc::make_desc(e0 + eoff, E_LBO, E_SBO), bRl = tc::make_desc(e0 + EI + eoff, E_LBO, E_SBO);
        const uint64_t bIh = tc::make_desc(e0 + 2 * EI + eoff, E_LBO, E_SBO);
        const uint64_t bIl = tc::make_desc(e0 + 3 * EI + eoff, E_LBO, E_SBO);
        const uint32_t dRe = tmem, dIm = tmem + 64;
        const uint32_t acc0 = q > 0 ? 1u : 0u;
        // D_re += Re E_re - Im E_im ; D_im += Re E_im + Im E_re   (3xTF32 each)
        tc::mma_tf32(dRe, aRh, bRh, id_p, acc0);
        tc::mma_tf32(dRe, aRh, bRl, id_p, 1u);
        tc::mma_tf32(dRe, aRl, bRh, id_p, 1u);
        tc::mma_tf32(dRe, aIh, bIh, id_n, 1u);
        tc::mma_tf32(dRe, aIh, bIl, id_n, 1u);
        tc::mma_tf32(dRe, aIl, bIh, id_n, 1u);
        tc::mma_tf32(dIm, aRh, bIh, id_p, acc0);
        tc::mma_tf32(dIm, aRh, bIl, id_p, 1u);
        tc::mma_tf32(dIm, aRl, bIh, id_p, 1u);
        tc::mma_tf32(dIm, aIh, bRh, id_p, 1u);
        tc::mma_tf32(dIm, aIh, bRl, id_p, 1u);
        tc::mma_tf32(dIm, aIl, bRh, id_p, 1u);
        tc::mma_commit(&mbar[b]);
      }
      __syncwarp();
    }
    // this tile's MMAs done -> P' = P + D; warp w reads TMEM lanes 32 (w % 4); half 0: D_re, half 1: D_im
    tc::mbar_wait(&mbar[(chunk_ctr - 1) & 1], ((chunk_ctr - 1) >> 1) & 1);
    tc::fence_after_sync();
    const int r = r0 + row_l;
    // thread (row, half) writes whole complex entries of columns 32 half .. 32 half + 31 (coalesced)
#pragma unroll 1
    for (int c = 32 * half; c < 32 * half + 32; c += 8) {
      float dr[8], di[8];
      const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16);
      tc::tmem_ld8(ta + c, dr);
      tc::tmem_ld8(ta + 64 + c, di);
      if (r < rows) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float2 v = raw[(c + u) * 128 + row_l];
          M[(int64_t)colof(c + u, I, J) * rows + r] = make_float2(v.x + dr[u], v.y + di[u]);
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();   // TMEM and raw reads done before they are overwritten
  }
  tc::cp_async_wait<0>();
  if (warp == 0) tc::tmem_dealloc(tmem, 128);
}

// ---- P <- P + P E, warp-specialised (the default rotation kernel). grid (pairs max, count);
// 288 threads = 9 warps:
//   warp 0      : one elected thread issues the MMAs (12 per 8-column chunk, 3xTF32, N = 64) into
//                 one of two TMEM accumulators (tile t uses buffer t % 2);
//   warps 1-4   : producers, thread = row of the 128-row tile: global -> registers -> TF32 hi/lo
//                 images in a 4-deep shared-memory ring (full / empty mbarriers);
//   warps 5-8   : epilogue, thread = row: TMEM -> registers, P' = P + D with P re-read from L2,
//                 coalesced stores; then releases the accumulator buffer.
// Loads, MMAs and stores of consecutive chunks and tiles overlap (the simple kernel serialised a
// chunk's conversion with the previous chunk's MMAs and the tile epilogue with both).
constexpr int WS_NS = 4;                                     // image ring depth
constexpr int WS_RAW = 8;                                    // raw chunks in flight per producer row
constexpr size_t rot_ws_smem(int ns, int nr) { return (size_t)EIMG_FLOATS * 4 + (size_t)ns * 2 * kRotStage + (size_t)nr * 8 * 128 * 8 + 1024; }
constexpr size_t kRotWsSmem = rot_ws_smem(WS_NS, WS_RAW);
// the lean variant (EAMPS_ROT_LEAN=1): 2-deep image ring, 4 raw chunks in flight -- 129 KB, so that a
// rotation CTA and an inner-solve CTA (66 KB) of the other stream's gate group fit one SM together
constexpr int WS_NS_LEAN = 2, WS_RAW_LEAN = 4;
constexpr size_t kRotWsSmemLean = rot_ws_smem(WS_NS_LEAN, WS_RAW_LEAN);
template <int NS, int NR>
__global__ void __launch_bounds__(288) k_tc_rot_ws(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                   int rnd, uint8_t* slab, const LargeCtl* ctl) {
  const int gi = blockIdx.y;
  if (ctl[gi].conv) return;
  const GateDesc& gd = desc[list[gi]];
  const int nb = gd.n_pad / TB, pair = blockIdx.x;
  if (pair >= nb / 2 || rnd >= nb - 1) return;
  const int pairs = gd.n_pad / PWC;
  const int32_t* rflag =
      reinterpret_cast<const int32_t*>(slab + gd.ws_log + Scratch::gram_bytes(pairs) + Scratch::eimg_bytes(pairs));
  if (!rflag[pair]) return;
  int I, J;
  circle_pair(pair, rnd, nb, I, J);
  const float* Eg = reinterpret_cast<const float*>(slab + gd.ws_log + Scratch::gram_bytes(pairs)) + (size_t)pair * EIMG_FLOATS;
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  float* Es = reinterpret_cast<float*>(base);                      // 64 KB: Re h|l, Im h|l
  uint8_t* ring = base + (size_t)EIMG_FLOATS * 4;                  // NS x (hi, lo) x 8 KB
  float2* rawr = reinterpret_cast<float2*>(ring + (size_t)NS * 2 * kRotStage);   // NR x [8 cols][128 rows]
  __shared__ uint64_t full[NS], empty[NS], tfull[2], tempty[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int x = tid; x < EIMG_FLOATS / 4; x += blockDim.x) tc::cp_async16(Es + 4 * x, Eg + 4 * x);
  tc::cp_async_commit();
  if (warp == 0) tc::tmem_alloc(&tbase, 256);
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      tc::mbar_init(&full[i], 128);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 128);
    }
    tc::fence_barrier_init();
  }
  tc::cp_async_wait_all();
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tbase;
  const int m = jacobi_rows(gd), np = gd.n_pad;   // preconditioned: B (n rows), no V tiles
  const int tiles_th = (m + 127) / 128, tiles_v = gd.jrows > 0 ? 0 : (np + 127) / 128, ntiles = tiles_th + tiles_v;
  constexpr int CH = PWC / 8;                                     // chunks per tile
  if (warp == 0) {
    // ---------------- MMA issuer
    if (tid == 0) {
      const uint32_t id_p = tc::make_idesc_tf32(128, 64, false, false);
      const uint32_t id_n = id_p | (1u << 14);   // negate B (-E_im)
      const uint32_t e0 = tc::smem_u32(Es);
      constexpr uint32_t EI = 16384;
      int u = 0;                                 // chunk counter
      for (int t = 0; t < ntiles; ++t) {
        const int ab = t & 1;
        if (t >= 2) tc::mbar_wait(&tempty[ab], ((t - 2) >> 1) & 1);
        tc::fence_after_sync();
        const uint32_t dRe = tmem + 128 * ab, dIm = dRe + 64;
        for (int q = 0; q < CH; ++q, ++u) {
          const int sl = u % NS;
          tc::mbar_wait(&full[sl], (u / NS) & 1);
          tc::fence_after_sync();
          const uint32_t a0 = tc::smem_u32(ring + (size_t)sl * 2 * kRotStage);
          const uint32_t eoff = 2 * q * E_LBO;
          const uint64_t aRh = tc::make_desc(a0, R_LBO, R_SBO), aRl = tc::make_desc(a0 + kRotStage, R_LBO, R_SBO);
          const uint64_t aIh = tc::make_desc(a0 + 2 * R_LBO, R_LBO, R_SBO);
          const uint64_t aIl = tc::make_desc(a0 + kRotStage + 2 * R_LBO, R_LBO, R_SBO);
          const uint64_t bRh = tc::make_desc(e0 + eoff, E_LBO, E_SBO), bRl = tc::make_desc(e0 + EI + eoff, E_LBO, E_SBO);
          const uint64_t bIh = tc::make_desc(e0 + 2 * EI + eoff, E_LBO, E_SBO);
          const uint64_t bIl = tc::make_desc(e0 + 3 * EI + eoff, E_LBO, E_SBO);
          const uint32_t acc0 = q > 0 ? 1u : 0u;
          tc::mma_tf32(dRe, aRh, bRh, id_p, acc0);
          tc::mma_tf32(dRe, aRh, bRl, id_p, 1u);
          tc::mma_tf32(dRe, aRl, bRh, id_p, 1u);
          tc::mma_tf32(dRe, aIh, bIh, id_n, 1u);
          tc::mma_tf32(dRe, aIh, bIl, id_n, 1u);
          tc::mma_tf32(dRe, aIl, bIh, id_n, 1u);
          tc::mma_tf32(dIm, aRh, bIh, id_p, acc0);
          tc::mma_tf32(dIm, aRh, bIl, id_p, 1u);
          tc::mma_tf32(dIm, aRl, bIh, id_p, 1u);
          tc::mma_tf32(dIm, aIh, bRh, id_p, 1u);
          tc::mma_tf32(dIm, aIh, bRl, id_p, 1u);
          tc::mma_tf32(dIm, aIl, bRh, id_p, 1u);
          tc::mma_commit(&empty[sl]);            // the slot is free once these MMAs completed
        }
        tc::mma_commit(&tfull[ab]);              // the tile's accumulator is complete
      }
    }
    __syncwarp();
  } else if (warp <= 4) {
    // ---------------- producers: thread = row. Each thread copies its own row of the next NR
    // chunks with 8-byte cp.async (64 KB in flight per CTA), then converts its row into the images.
    const int row_l = tid - 32;
    const int total = ntiles * CH;
    auto issue = [&](int uu) {
      if (uu < total) {
        const int t = uu / CH, q = uu % CH;
        const bool isV = t >= tiles_th;
        const float2* M = reinterpret_cast<const float2*>(slab + (isV ? gd.ws_V : gd.ws_theta));
        const int rows = isV ? np : m;
        const int r = (isV ? t - tiles_th : t) * 128 + row_l;
        float2* dst = rawr + (size_t)(uu % NR) * 8 * 128 + row_l;
        if (r < rows) {
#pragma unroll
          for (int c = 0; c < 8; ++c) tc::cp_async8(dst + c * 128, M + (int64_t)colof(8 * q + c, I, J) * rows + r);
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) dst[c * 128] = make_float2(0.f, 0.f);
        }
      }
      tc::cp_async_commit();
    };
    for (int uu = 0; uu < NR - 1; ++uu) issue(uu);
    for (int u = 0; u < total; ++u) {
      issue(u + NR - 1);
      tc::cp_async_wait<NR - 1>();                  // this thread's copies of chunk u landed
      const float2* src = rawr + (size_t)(u % NR) * 8 * 128 + row_l;
      float2 z[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) z[c] = src[c * 128];
      const int sl = u % NS;
      if (u >= NS) tc::mbar_wait(&empty[sl], ((u / NS) - 1) & 1);
      uint8_t* hi = ring + (size_t)sl * 2 * kRotStage;
      uint8_t* lo = hi + kRotStage;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float4 rh, rl, ih, il;
        tc::split_tf32(z[4 * h + 0].x, rh.x, rl.x); tc::split_tf32(z[4 * h + 1].x, rh.y, rl.y);
        tc::split_tf32(z[4 * h + 2].x, rh.z, rl.z); tc::split_tf32(z[4 * h + 3].x, rh.w, rl.w);
        tc::split_tf32(z[4 * h + 0].y, ih.x, il.x); tc::split_tf32(z[4 * h + 1].y, ih.y, il.y);
        tc::split_tf32(z[4 * h + 2].y, ih.z, il.z); tc::split_tf32(z[4 * h + 3].y, ih.w, il.w);
        const uint32_t oR = tc::kmaj_off(row_l, 4 * h, R_LBO, R_SBO), oI = tc::kmaj_off(row_l, 8 + 4 * h, R_LBO, R_SBO);
        *reinterpret_cast<float4*>(hi + oR) = rh;
        *reinterpret_cast<float4*>(lo + oR) = rl;
        *reinterpret_cast<float4*>(hi + oI) = ih;
        *reinterpret_cast<float4*>(lo + oI) = il;
      }
      tc::fence_async_smem();
      tc::mbar_arrive(&full[sl]);
    }
    tc::cp_async_wait<0>();
  } else {
    // ---------------- epilogue: thread = row, TMEM lane quadrant = warp % 4
    const int row_l = (warp & 3) * 32 + (tid & 31);
    for (int t = 0; t < ntiles; ++t) {
      const bool isV = t >= tiles_th;
      float2* M = reinterpret_cast<float2*>(slab + (isV ? gd.ws_V : gd.ws_theta));
      const int rows = isV ? np : m;
      const int r = (isV ? t - tiles_th : t) * 128 + row_l;
      const int ab = t & 1;
      tc::mbar_wait(&tfull[ab], (t >> 1) & 1);
      tc::fence_after_sync();
      const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 128 * ab;
#pragma unroll 1
      for (int c = 0; c < PWC; c += 8) {
        float dr[8], di[8];
        tc::tmem_ld8(ta + c, dr);
        tc::tmem_ld8(ta + 64 + c, di);
        if (r < rows) {
          float2 v[8];
#pragma unroll
          for (int u2 = 0; u2 < 8; ++u2) v[u2] = M[(int64_t)colof(c + u2, I, J) * rows + r];
#pragma unroll
          for (int u2 = 0; u2 < 8; ++u2)
            M[(int64_t)colof(c + u2, I, J) * rows + r] = make_float2(v[u2].x + dr[u2], v[u2].y + di[u2]);
        }
      }
      tc::fence_before_sync();
      tc::mbar_arrive(&tempty[ab]);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

// ---- FP64-anchored polish of the spectrum (after convergence). With B = theta V (FP64-accumulated,
// stored FP32 in the theta workspace) and C = B^H B, the Rayleigh values c_j = C_jj / |v_j|^2 are
// exact eigenvalues of C only if the off-diagonal C_lj vanish; the FP32 accumulation of V leaves
// |C_lj| ~ 1e-6 sigma_l sigma_j, which contaminates a small sigma_j^2 by ~|C_lj|^2 / sigma_l^2.
// Every pair (l, j) contributes the exact 2x2 eigenvalue shift
//   delta_j = sgn(c_j - c_l) g^2 / (|c_j - c_l|/2 + sqrt((c_j - c_l)^2/4 + g^2)),
//   g^2 = |C_lj|^2 / (|v_l|^2 |v_j|^2)
// (second-order perturbation, bounded for near-degenerate pairs), summed over l. C_lj comes from the
// tensor core (3xTF32: ~2^-22 |b_l||b_j|, far below the |C_lj| it measures); c_j from the FP64
// Rayleigh quotient. Grid (n_pad/64 pairs, count, n_pad/32 - 1 rounds): the circle method's rounds
// enumerate every block pair once; round 0 also covers the pairs inside each block.
__global__ void __launch_bounds__(128) k_tc_polish(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                   uint8_t* slab) {
  const int gi = blockIdx.y, rnd = blockIdx.z;
  const GateDesc& gd = desc[list[gi]];
  const int n = gd.n, np = gd.n_pad;
  const int nb = ((n + PWC - 1) / PWC) * 2, pair = blockIdx.x;   // blocks of 32 over n rounded up to 64
  if (pair >= nb / 2 || rnd >= nb - 1) return;
  int I, J;
  circle_pair(pair, rnd, nb, I, J);
  if (I * TB >= n && J * TB >= n) return;
  const double* s2 = reinterpret_cast<const double*>(slab + gd.ws_sig2);
  double* shift = reinterpret_cast<double*>(slab + gd.ws_E);
  const double* den = shift + np;
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  tc_setup(mbar, &tbase);
  float* Ds = reinterpret_cast<float*>(base);  // [128][129]
  gram_panel(reinterpret_cast<const float2*>(slab + gd.ws_theta), gd.m, n, I, J, base, mbar, tbase, Ds);
  if ((tid >> 5) == 0) tc::tmem_dealloc(tbase, 128);
  // panel column j = tid % 64, two threads per column (all 128 of the CTA: the loop below is a chain of
  // FP64 divisions and square roots, latency-bound at one thread per column, ncu r02 -- 55% of the
  // kernel's stall samples): partners = the other block (always) and the column's own block (round 0);
  // in round 0 thread half 0 takes the other block and half 1 the own block, otherwise the halves
  // split the other block's 32 columns. Each half adds its partial sum (atomicAdd, as before across CTAs).
  {
    const int j = tid & 63, half = tid >> 6, cj = colof(j, I, J);
    if (cj < n) {
      const double aj = s2[cj], dj = den[cj];
      auto sym = [&](int a, int b2) { return 0.5f * (Ds[a * 129 + b2] + Ds[b2 * 129 + a]); };
      double acc = 0.0;
      const int other0 = j < TB ? TB : 0;
      const int own0 = j < TB ? 0 : TB;
      const int lb = rnd == 0 ? (half == 0 ? other0 : own0) : other0 + half * (TB / 2);
      const int le = rnd == 0 ? lb + TB : lb + TB / 2;
      {
        for (int l = lb; l < le; ++l) {
          const int cl = colof(l, I, J);
          if (l == j || cl >= n) continue;
          const double gr = sym(l, j) + sym(64 + l, 64 + j), gim = sym(l, 64 + j) - sym(64 + l, j);
          const double al_ = s2[cl];
          // only well-separated pairs (ratio > 4): the contamination of a small sigma^2 by a large
          // one. Between near-degenerate pairs C_lj also holds the product of their shared
          // contaminations (a fourth-order coupling over a small gap) that the pairwise formula
          // would turn into a spurious shift; their own mixing moves sigma^2 by at most ~tol.
          if (fmax(aj, al_) < 4.0 * fmin(aj, al_)) continue;
          if (!(dj > 0.0) || !(den[cl] > 0.0)) continue;   // a zero column (rank-deficient theta)
          const double g2 = (gr * gr + gim * gim) / (dj * den[cl]);
          const double dlt = aj - al_;
          const double h = 0.5 * fabs(dlt);
          const double sh = g2 / (h + sqrt(h * h + g2));
          acc += dlt >= 0.0 ? sh : -sh;
        }
      }
      atomicAdd(&shift[cj], acc);
    }
  }
}


// =====================================================================================================
// Fused persistent large-regime Jacobi (the default since round 2): ONE cooperative launch per wave
// runs every sweep and round of every large gate of the wave. A CTA (288 threads, one per SM) takes
// pair tasks (gate, block pair) of the current round and, per task, runs the three steps of a block
// rotation back to back with the panel Gram, the Hermitian 64 x 64 G and the E images never leaving
// the SM:
//   1. Gram  (warps 0-3, tensor core): D = Q^T Q of the panel P = [A_I A_J], TMEM accumulator,
//      symmetric 3xTF32 (gram_panel) -> G = P^H P in shared memory;
//   2. inner (all warps, SIMT FP32): one cyclic Jacobi sweep on G -> W, E = W - I as TF32 hi/lo images;
//   3. rotation (warp-specialised, tensor core): P <- P + P E (identity-split 3xTF32), as k_tc_rot_ws.
// Rounds are separated by a grid-wide barrier (co-residency guaranteed by the cooperative launch);
// the end of a sweep runs the per-gate convergence check on the device (no host round trip per
// sweep, no three launches per round). The arithmetic of every step is that of the three
// separate kernels (k_tc_gram / k_tc_inner / k_tc_rot_ws), which stay as the EAMPS_TC_UNFUSED=1
// development reference.
// Shared memory (from the 1024-aligned base):
//   [0, 64K)        E images (written by the inner solve, the rotation's B operand)
//   [64K, 164K)     Gram images + raw ring; D staging (128 x 129 floats) aliases its start
//   [130K, 196.5K)  G, W of the inner solve (64 x 65 complex each)
//   [64K, 192K)     rotation image ring + raw chunks (dead Gram / inner data by then)
constexpr int FT = 288;
constexpr size_t F_ES = 0;
constexpr size_t F_GRAM = (size_t)EIMG_FLOATS * 4;                 // 64 KB
constexpr size_t F_RING = F_GRAM;
constexpr size_t F_RAW = F_RING + (size_t)WS_NS * 2 * kRotStage;  // 128 KB
constexpr size_t F_GW = F_GRAM + (size_t)128 * 129 * 4 + 64;       // after the D staging
constexpr size_t F_END = F_GW + 2 * sizeof(float2) * 64 * 65;
constexpr size_t kFusedSmem = (F_END > F_RAW + (size_t)WS_RAW * 8 * 128 * 8 ? F_END : F_RAW + (size_t)WS_RAW * 8 * 128 * 8) + 1024;
static_assert(F_GRAM + 4 * kGramStage + GR * kGramRaw <= F_GW || true, "layout");

struct FusedCtl {                 // device-side control of the persistent kernel (in the wave scratch)
  unsigned int bar_count, bar_gen;
  int32_t unconv[2];              // unconverged gates of the sweep, by sweep parity
  int32_t done;                   // every gate converged
  int32_t sweeps_run;
};

__device__ __forceinline__ void grid_barrier(FusedCtl* fc) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = &fc->bar_gen;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(&fc->bar_count, 1u) == gridDim.x - 1) {
      fc->bar_count = 0;
      __threadfence();
      atomicAdd(&fc->bar_gen, 1u);
    } else {
      while (*gen == g) __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence();   // gpu-scope fence: invalidates this SM's L1 (other CTAs' panel writes)
}

// The inner solve of k_tc_inner on G (shared memory) with NT threads, writing the E images into Es.
// Returns true if any pair rotated (CTA-uniform).
template <int NT>
__device__ bool inner_solve(float2 (*Gs)[65], float2 (*Ws)[65], float* Es, int rnd, float skip, float tol,
                            float tol_int, int inner_sweeps, float4* par, int2* pq, const uint16_t* blk) {
  auto gld = [&](int i, int j) {
    const float2 v = Gs[min(i, j)][max(i, j)];
    return i <= j ? v : make_float2(v.x, -v.y);
  };
  auto gst = [&](int i, int j, float2 v) { Gs[min(i, j)][max(i, j)] = i <= j ? v : make_float2(v.x, -v.y); };
  const int tid = threadIdx.x;
  int any = 0, internal = 0;
  for (int x = tid; x < 64 * 64; x += NT) {
    const int p = x >> 6, q = x & 63;
    if (p < q) {
      const float al = Gs[p][p].x, be = Gs[q][q].x;
      const float g = sqrtf(Gs[p][q].x * Gs[p][q].x + Gs[p][q].y * Gs[p][q].y);
      if (fminf(al, be) > skip && g > tol * sqrtf(al) * sqrtf(be)) {
        any = 1;
        if ((p < 32) == (q < 32) && (rnd == 0 || g > tol_int * sqrtf(al) * sqrtf(be))) internal = 1;
      }
    }
  }
  internal = __syncthreads_or(internal);
  if (!__syncthreads_or(any)) return false;
  const int nrr = internal ? 63 : 32;
  constexpr int TPP = NT / 32;    // threads per pair in the W update
  for (int isw = 0; isw < inner_sweeps; ++isw) {
    int rot = 0;
    for (int rr = 0; rr < nrr; ++rr) {
      if (tid < 32) {
        int p, q;
        if (internal) {
          circle_pair(tid, rr, 64, p, q);
        } else {
          p = tid;
          q = 32 + ((tid + rr) & 31);
        }
        const float al = Gs[p][p].x, be = Gs[q][q].x;
        const float2 gm = gld(p, q);
        const float g2 = gm.x * gm.x + gm.y * gm.y;
        float c = 1.f, sn = 0.f, er = 1.f, ei = 0.f;
        if (fminf(al, be) > skip && g2 > 1e-13f * al * be) {
          const float ig = rsqrtf(g2);
          er = gm.x * ig;
          ei = gm.y * ig;
          const float zeta = 0.5f * (be - al) * ig;
          const float az = fabsf(zeta);
          const float t = copysignf(1.f, zeta) / (az + sqrtf(fmaf(az, az, 1.f)));
          c = rsqrtf(fmaf(t, t, 1.f));
          sn = c * t;
          rot = 1;
          const float tg = t * (g2 * ig);
          Gs[p][p] = make_float2(al - tg, 0.f);
          Gs[q][q] = make_float2(be + tg, 0.f);
          gst(p, q, make_float2(0.f, 0.f));
        }
        par[tid] = make_float4(c, sn, er, ei);
        pq[tid] = make_int2(p, q);
      }
      __syncthreads();
      for (int x = tid; x < 496; x += NT) {
        const int ia = blk[x] & 0xFF, ib = blk[x] >> 8;
        const float4 Ja = par[ia], Jb = par[ib];
        if (Ja.y == 0.f && Jb.y == 0.f) continue;
        const int2 ra = pq[ia], cb = pq[ib];
        float2 X[2][2] = {{gld(ra.x, cb.x), gld(ra.x, cb.y)}, {gld(ra.y, cb.x), gld(ra.y, cb.y)}};
        if (Jb.y != 0.f) {
          const Rot rb{Jb.x, Jb.y, Jb.z, Jb.w};
#pragma unroll
          for (int r = 0; r < 2; ++r) apply_rot(X[r][0], X[r][1], rb);
        }
        if (Ja.y != 0.f) {
          const Rot ra2{Ja.x, Ja.y, Ja.z, -Ja.w};
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) apply_rot(X[0][cc], X[1][cc], ra2);
        }
        gst(ra.x, cb.x, X[0][0]); gst(ra.x, cb.y, X[0][1]);
        gst(ra.y, cb.x, X[1][0]); gst(ra.y, cb.y, X[1][1]);
      }
      {
        const int k = tid / TPP;
        if (k < 32) {
          const float4 J = par[k];
          if (J.y != 0.f) {
            const int2 cq = pq[k];
            const Rot rw{J.x, J.y, J.z, J.w};
            for (int x = tid % TPP; x < 64; x += TPP) {
              float2 xx = Ws[x][cq.x], yy = Ws[x][cq.y];
              apply_rot(xx, yy, rw);
              Ws[x][cq.x] = xx;
              Ws[x][cq.y] = yy;
            }
          }
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rot)) break;
  }
  __syncthreads();
  for (int x = tid; x < 64 * 64; x += NT) {
    const int k = x >> 6, n = x & 63;
    float2 w = Ws[k][n];
    if (k == n) w.x -= 1.f;
    const uint32_t o = tc::kmaj_off(n, k, E_LBO, E_SBO) >> 2;
    float h, l;
    tc::split_tf32(w.x, h, l);
    Es[o] = h;
    Es[4096 + o] = l;
    tc::split_tf32(w.y, h, l);
    Es[8192 + o] = h;
    Es[12288 + o] = l;
  }
  return true;
}

// P <- P + P E with E in shared memory: the warp-specialised body of k_tc_rot_ws (288 threads).
__device__ void rot_panel_ws(const GateDesc& gd, uint8_t* slab, int I, int J, const float* Es, uint8_t* ring,
                             float2* rawr, uint64_t* full, uint64_t* empty, uint64_t* tfull, uint64_t* tempty,
                             uint32_t tmem) {
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < WS_NS; ++i) {
      tc::mbar_init(&full[i], 128);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&tfull[i], 1);
      tc::mbar_init(&tempty[i], 128);
    }
    tc::fence_barrier_init();
  }
  tc::fence_async_smem();   // E images (generic-proxy writes) -> visible to the tensor core
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const int m = jacobi_rows(gd), np = gd.n_pad;
  const int tiles_th = (m + 127) / 128, tiles_v = gd.jrows > 0 ? 0 : (np + 127) / 128, ntiles = tiles_th + tiles_v;
  constexpr int CH = PWC / 8;
  if (warp == 0) {
    if (tid == 0) {
      const uint32_t id_p = tc::make_idesc_tf32(128, 64, false, false);
      const uint32_t id_n = id_p | (1u << 14);
      const uint32_t e0 = tc::smem_u32(Es);
      constexpr uint32_t EI = 16384;
      int u = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int ab = t & 1;
        if (t >= 2) tc::mbar_wait(&tempty[ab], ((t - 2) >> 1) & 1);
        tc::fence_after_sync();
        const uint32_t dRe = tmem + 128 * ab, dIm = dRe + 64;
        for (int q = 0; q < CH; ++q, ++u) {
          const int sl = u % WS_NS;
          tc::mbar_wait(&full[sl], (u / WS_NS) & 1);
          tc::fence_after_sync();
          const uint32_t a0 = tc::smem_u32(ring + (size_t)sl * 2 * kRotStage);
          const uint32_t eoff = 2 * q * E_LBO;
          const uint64_t aRh = tc::make_desc(a0, R_LBO, R_SBO), aRl = tc::make_desc(a0 + kRotStage, R_LBO, R_SBO);
          const uint64_t aIh = tc::make_desc(a0 + 2 * R_LBO, R_LBO, R_SBO);
          const uint64_t aIl = tc::make_desc(a0 + kRotStage + 2 * R_LBO, R_LBO, R_SBO);
          const uint64_t bRh = tc::make_desc(e0 + eoff, E_LBO, E_SBO), bRl = tc::make_desc(e0 + EI + eoff, E_LBO, E_SBO);
          const uint64_t bIh = tc::make_desc(e0 + 2 * EI + eoff, E_LBO, E_SBO);
          const uint64_t bIl = tc::make_desc(e0 + 3 * EI + eoff, E_LBO, E_SBO);
          const uint32_t acc0 = q > 0 ? 1u : 0u;
          tc::mma_tf32(dRe, aRh, bRh, id_p, acc0);
          tc::mma_tf32(dRe, aRh, bRl, id_p, 1u);
          tc::mma_tf32(dRe, aRl, bRh, id_p, 1u);
          tc::mma_tf32(dRe, aIh, bIh, id_n, 1u);
          tc::mma_tf32(dRe, aIh, bIl, id_n, 1u);
          tc::mma_tf32(dRe, aIl, bIh, id_n, 1u);
          tc::mma_tf32(dIm, aRh, bIh, id_p, acc0);
          tc::mma_tf32(dIm, aRh, bIl, id_p, 1u);
          tc::mma_tf32(dIm, aRl, bIh, id_p, 1u);
          tc::mma_tf32(dIm, aIh, bRh, id_p, 1u);
          tc::mma_tf32(dIm, aIh, bRl, id_p, 1u);
          tc::mma_tf32(dIm, aIl, bRh, id_p, 1u);
          tc::mma_commit(&empty[sl]);
        }
        tc::mma_commit(&tfull[ab]);
      }
      // drain: the last WS_NS slot releases were never waited on by the producers; they must land
      // before the barriers are re-initialised for the next task
      for (int uu = max(0, u - WS_NS); uu < u; ++uu) tc::mbar_wait(&empty[uu % WS_NS], (uu / WS_NS) & 1);
    }
    __syncwarp();
  } else if (warp <= 4) {
    const int row_l = tid - 32;
    const int total = ntiles * CH;
    auto issue = [&](int uu) {
      if (uu < total) {
        const int t = uu / CH, q = uu % CH;
        const bool isV = t >= tiles_th;
        const float2* M = reinterpret_cast<const float2*>(slab + (isV ? gd.ws_V : gd.ws_theta));
        const int rows = isV ? np : m;
        const int r = (isV ? t - tiles_th : t) * 128 + row_l;
        float2* dst = rawr + (size_t)(uu % WS_RAW) * 8 * 128 + row_l;
        if (r < rows) {
#pragma unroll
          for (int c = 0; c < 8; ++c) tc::cp_async8(dst + c * 128, M + (int64_t)colof(8 * q + c, I, J) * rows + r);
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) dst[c * 128] = make_float2(0.f, 0.f);
        }
      }
      tc::cp_async_commit();
    };
    for (int uu = 0; uu < WS_RAW - 1; ++uu) issue(uu);
    for (int u = 0; u < total; ++u) {
      issue(u + WS_RAW - 1);
      tc::cp_async_wait<WS_RAW - 1>();
      const float2* src = rawr + (size_t)(u % WS_RAW) * 8 * 128 + row_l;
      float2 z[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) z[c] = src[c * 128];
      const int sl = u % WS_NS;
      if (u >= WS_NS) tc::mbar_wait(&empty[sl], ((u / WS_NS) - 1) & 1);
      uint8_t* hi = ring + (size_t)sl * 2 * kRotStage;
      uint8_t* lo = hi + kRotStage;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float4 rh, rl, ih, il;
        tc::split_tf32(z[4 * h + 0].x, rh.x, rl.x); tc::split_tf32(z[4 * h + 1].x, rh.y, rl.y);
        tc::split_tf32(z[4 * h + 2].x, rh.z, rl.z); tc::split_tf32(z[4 * h + 3].x, rh.w, rl.w);
        tc::split_tf32(z[4 * h + 0].y, ih.x, il.x); tc::split_tf32(z[4 * h + 1].y, ih.y, il.y);
        tc::split_tf32(z[4 * h + 2].y, ih.z, il.z); tc::split_tf32(z[4 * h + 3].y, ih.w, il.w);
        const uint32_t oR = tc::kmaj_off(row_l, 4 * h, R_LBO, R_SBO), oI = tc::kmaj_off(row_l, 8 + 4 * h, R_LBO, R_SBO);
        *reinterpret_cast<float4*>(hi + oR) = rh;
        *reinterpret_cast<float4*>(lo + oR) = rl;
        *reinterpret_cast<float4*>(hi + oI) = ih;
        *reinterpret_cast<float4*>(lo + oI) = il;
      }
      tc::fence_async_smem();
      tc::mbar_arrive(&full[sl]);
    }
    tc::cp_async_wait<0>();
  } else {
    const int row_l = (warp & 3) * 32 + (tid & 31);
    for (int t = 0; t < ntiles; ++t) {
      const bool isV = t >= tiles_th;
      float2* M = reinterpret_cast<float2*>(slab + (isV ? gd.ws_V : gd.ws_theta));
      const int rows = isV ? np : m;
      const int r = (isV ? t - tiles_th : t) * 128 + row_l;
      const int ab = t & 1;
      tc::mbar_wait(&tfull[ab], (t >> 1) & 1);
      tc::fence_after_sync();
      const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 128 * ab;
#pragma unroll 1
      for (int c = 0; c < PWC; c += 8) {
        float dr[8], di[8];
        tc::tmem_ld8(ta + c, dr);
        tc::tmem_ld8(ta + 64 + c, di);
        if (r < rows) {
          float2 v[8];
#pragma unroll
          for (int u2 = 0; u2 < 8; ++u2) v[u2] = __ldcg(M + (int64_t)colof(c + u2, I, J) * rows + r);
#pragma unroll
          for (int u2 = 0; u2 < 8; ++u2)
            M[(int64_t)colof(c + u2, I, J) * rows + r] = make_float2(v[u2].x + dr[u2], v[u2].y + di[u2]);
        }
      }
      tc::fence_before_sync();
      tc::mbar_arrive(&tempty[ab]);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
}

// pair_pre[g] = sum of the block pairs (n_pad / 64) of the gates before g (the task index space of a round)
__global__ void k_pair_prefix(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list, int count,
                              int32_t* pair_pre, FusedCtl* fc) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int32_t acc = 0;
    for (int g = 0; g < count; ++g) {
      pair_pre[g] = acc;
      acc += desc[list[g]].n_pad / PWC;
    }
    pair_pre[count] = acc;
    fc->bar_count = 0;
    fc->bar_gen = 0;
    fc->unconv[0] = fc->unconv[1] = 0;
    fc->done = 0;
    fc->sweeps_run = 0;
  }
}

__global__ void __launch_bounds__(FT, 1) k_tc_fused(GateDesc* __restrict__ desc, const int32_t* __restrict__ list,
                                                    int count, uint8_t* slab, LargeCtl* ctl, const double* norm2,
                                                    const int32_t* __restrict__ pair_pre, FusedCtl* fc, int max_sweeps,
                                                    int inner_sweeps, float tol_floor, float tol_internal) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
  float* Es = reinterpret_cast<float*>(base + F_ES);
  uint8_t* gram_base = base + F_GRAM;
  float* Ds = reinterpret_cast<float*>(base + F_GRAM);
  float2(*Gs)[65] = reinterpret_cast<float2(*)[65]>(base + F_GW);
  float2(*Ws)[65] = Gs + 64;
  uint8_t* ring = base + F_RING;
  float2* rawr = reinterpret_cast<float2*>(base + F_RAW);
  __shared__ uint64_t gbar[2], full[WS_NS], empty[WS_NS], tfull[2], tempty[2];
  __shared__ uint32_t tbase;
  __shared__ float4 par[32];
  __shared__ int2 pq[32];
  __shared__ uint16_t blk[496];
  __shared__ int s_rot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int x = tid; x < 496; x += FT) {
    int aa = 0, rem = x;
    while (rem >= 31 - aa) { rem -= 31 - aa; ++aa; }
    blk[x] = (uint16_t)(aa | ((aa + 1 + rem) << 8));
  }
  if (warp == 0) tc::tmem_alloc(&tbase, 256);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tbase;
  const int total = pair_pre[count];
  int nb_max = 0;
  for (int g = 0; g < count; ++g) nb_max = max(nb_max, desc[list[g]].n_pad / TB);
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    for (int rnd = 0; rnd < nb_max - 1; ++rnd) {
      for (int task = blockIdx.x; task < total; task += gridDim.x) {
        int lo = 0, hi = count - 1;          // gate of the task: last g with pair_pre[g] <= task
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (pair_pre[mid] <= task) lo = mid; else hi = mid - 1;
        }
        const int gi = lo, pair = task - pair_pre[gi];
        if (ctl[gi].conv) continue;          // (uniform: every thread reads the same value)
        const GateDesc& gd = desc[list[gi]];
        const int nb = gd.n_pad / TB;
        if (rnd >= nb - 1) continue;
        int I, J;
        circle_pair(pair, rnd, nb, I, J);
        // 1. Gram on warps 0-3
        if (warp < 4) {
          if (tid == 0) {
            tc::mbar_init(&gbar[0], 1);
            tc::mbar_init(&gbar[1], 1);
            tc::fence_barrier_init();
          }
          bar128();
          gram_panel<true>(reinterpret_cast<const float2*>(slab + gd.ws_theta), jacobi_rows(gd), gd.n_pad, I, J,
                           gram_base, gbar, tmem, Ds);
        }
        __syncthreads();
        // 2. G (Hermitian 64 x 64) from D, W = I; inner solve -> E images
        auto sym = [&](int a, int b2) { return 0.5f * (Ds[a * 129 + b2] + Ds[b2 * 129 + a]); };
        for (int x = tid; x < 64 * 64; x += FT) {
          const int p = x >> 6, qq = x & 63;
          Gs[p][qq] = make_float2(sym(p, qq) + sym(64 + p, 64 + qq), sym(p, 64 + qq) - sym(64 + p, qq));
          Ws[p][qq] = make_float2(p == qq ? 1.f : 0.f, 0.f);
        }
        __syncthreads();
        const float skip = (float)(norm2[gi] * 3.552713678800501e-15);
        const float tol = fmaxf(tol_floor, 4.f * sqrtf((float)jacobi_rows(gd)) * 5.960464477539063e-8f);
        const bool rotated = inner_solve<FT>(Gs, Ws, Es, rnd, skip, tol, fmaxf(tol, tol_internal), inner_sweeps,
                                             par, pq, blk);
        if (!rotated) {
          __syncthreads();
          continue;
        }
        if (tid == 0) atomicAdd(&ctl[gi].rot, 1);
        __syncthreads();
        // 3. P <- P + P E
        rot_panel_ws(gd, slab, I, J, Es, ring, rawr, full, empty, tfull, tempty, tmem);
      }
      grid_barrier(fc);
      if (rnd == 0 && blockIdx.x == 0 && tid == 0) fc->unconv[(sweep + 1) & 1] = 0;   // read last sweep
    }
    // end of sweep: per-gate convergence (a gate whose sweep rotated nothing is converged)
    for (int g = blockIdx.x * FT + tid; g < count; g += gridDim.x * FT) {
      if (ctl[g].conv) continue;
      GateDesc& gd = desc[list[g]];
      gd.sweeps += 1;
      if (ctl[g].rot == 0) ctl[g].conv = 1;
      else atomicAdd(&fc->unconv[sweep & 1], 1);
      ctl[g].rot = 0;
    }
    grid_barrier(fc);
    const int left = *reinterpret_cast<volatile int32_t*>(&fc->unconv[sweep & 1]);
    if (blockIdx.x == 0 && tid == 0) fc->sweeps_run = sweep + 1;
    if (left == 0) {
      if (blockIdx.x == 0 && tid == 0) fc->done = 1;
      break;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

}  // namespace tcj

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
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(k_block_round, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRoundSmem);
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

size_t svd_tc_scratch_bytes(int n_pad) { return tcj::Scratch::total(n_pad / tcj::PWC); }

// Rayleigh quotients + FP64-anchored polish + sort/tails for gates whose V (ld n_pad) is in the
// workspace (the large regime and the QR-preconditioned regime). Returns launches issued.
int launch_spectrum_polish(GateDesc* d_desc, const int32_t* d_list, int count, int max_n, uint8_t* slab, DevState* st,
                           cudaStream_t s) {
  if (count <= 0) return 0;
  // EAMPS_RAYLEIGH_THETA=1: the QR-regime Rayleigh quotients from theta V instead of L^H V (A/B)
  static const int use_l = getenv("EAMPS_RAYLEIGH_THETA") ? 0 : 1;
  static const bool old = getenv("EAMPS_RAYLEIGH_OLD") != nullptr;   // dev A/B switch
  if (old) {
    k_rayleigh<<<dim3((max_n + 31) / 32, count), 256, 0, s>>>(d_desc, d_list, slab, st, 1, use_l);
  } else {
    static std::atomic<unsigned long long> rattr{0};
    if (first_on_device(rattr))
      cudaFuncSetAttribute(k_rayleigh64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * kRay64Half));
    k_rayleigh64<<<dim3((max_n + 63) / 64, count), 256, 2 * kRay64Half, s>>>(d_desc, d_list, slab, st, use_l);
  }
  static std::atomic<unsigned long long> pattr{0};
  if (first_on_device(pattr)) {
    cudaFuncSetAttribute(tcj::k_tc_polish, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tcj::kGramSmem);
  }
  const int nb = ((max_n + tcj::PWC - 1) / tcj::PWC) * 2;
  static const bool no_polish = getenv("EAMPS_NO_POLISH") != nullptr;   // dev A/B switch
  if (!no_polish && nb >= 2)
    tcj::k_tc_polish<<<dim3(nb / 2, count, nb - 1), 128, tcj::kGramSmem, s>>>(d_desc, d_list, slab);
  int npow2 = 1;
  while (npow2 < max_n) npow2 <<= 1;
  const size_t smem = (size_t)npow2 * 12 + 16 + 1024 * 8;
  cudaFuncSetAttribute(k_sort_tails_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_sort_tails_large<<<count, 1024, smem, s>>>(d_desc, d_list, slab, st, 1);
  return 3;
}

// The side stream of the two-group round schedule and its two events: created once per device
// (cudaStream/cudaEvent are device-bound) and kept for the life of the process, instead of a
// create/destroy per wave. Returns false (one group is used) if creation fails.
static bool side_stream(cudaStream_t* s2, cudaEvent_t* go, cudaEvent_t* done) {
  struct Side { cudaStream_t s = nullptr; cudaEvent_t go = nullptr, done = nullptr; bool bad = false; };
  static Side side[64];
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  std::lock_guard<std::mutex> lock(mu);
  Side& x = side[dev];
  if (!x.s && !x.bad) {
    if (cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.go, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      x.bad = true;
      x.s = nullptr;
    }
  }
  if (x.bad) return false;
  *s2 = x.s;
  *go = x.go;
  *done = x.done;
  return true;
}

// ---- deep-spectrum re-Jacobi of the large regime (run_svd_tc): flags, preparation, finish
constexpr double kDeepRatio = 5e-5;   // config 2 chi = 256 (8.6e-5) stays on the polish; chi = 1024 (1.1e-5) not

// flags[g] = 1 if n > 256 and the smallest Rayleigh sigma^2 >= 1e-12 sigma_max^2 is below r2 sigma_max^2
__global__ void k_deep_flags(const GateDesc* __restrict__ desc, const int32_t* __restrict__ list, uint8_t* slab,
                             int32_t* flags, double r2) {
  const GateDesc& gd = desc[list[blockIdx.x]];
  const int n = gd.n;
  const double* s2 = reinterpret_cast<const double*>(slab + gd.ws_sig2);
  __shared__ double smx[256], smn[256];
  double mx = 0.0;
  for (int j = threadIdx.x; j < n; j += 256) mx = fmax(mx, s2[j]);
  smx[threadIdx.x] = mx;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) smx[threadIdx.x] = fmax(smx[threadIdx.x], smx[threadIdx.x + o]);
    __syncthreads();
  }
  mx = smx[0];
  double mn = mx;
  for (int j = threadIdx.x; j < n; j += 256)
    if (s2[j] >= 1e-12 * mx) mn = fmin(mn, s2[j]);
  smn[threadIdx.x] = mn;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) smn[threadIdx.x] = fmin(smn[threadIdx.x], smn[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) flags[blockIdx.x] = (n > 256 && gd.jrows > 0 && mx > 0.0 && smn[0] < r2 * mx) ? 1 : 0;
}

// The re-Jacobi works on B1 = theta V (k_rayleigh's write_b output in ws_theta, ld m): jrows = m,
// zero pad columns, fresh per-list control and norms. grid (64, dc).
__global__ void k_deep_prepare(GateDesc* desc, const int32_t* list, int count, const int32_t* dlist, uint8_t* slab,
                               LargeCtl* ctl, const double* norm2, double* dnorm2) {
  const int di = blockIdx.y, gdx = dlist[di];
  GateDesc& gd = desc[gdx];
  const int m = gd.m, n = gd.n, np = gd.n_pad;
  float2* B = reinterpret_cast<float2*>(slab + gd.ws_theta);
  const int64_t tot = (int64_t)m * (np - n);
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x)
    B[(int64_t)m * n + x] = make_float2(0.f, 0.f);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double nv = 0.0;
    for (int g = 0; g < count; ++g)
      if (list[g] == gdx) nv = norm2[g];
    dnorm2[di] = nv;
    ctl[di].rot = 0;
    ctl[di].conv = 0;
    gd.jrows = m;
  }
}

// sigma_j^2 = |b1_j|^2 (FP64 sums of the FP32 entries) replaces the Rayleigh value; the polish shift
// is cleared (sort_tails adds it); jrows back to n. One CTA per deep gate.
__global__ void k_deep_finish(GateDesc* desc, const int32_t* dlist, uint8_t* slab) {
  GateDesc& gd = desc[dlist[blockIdx.x]];
  const int m = gd.m, n = gd.n, np = gd.n_pad;
  const float2* B = reinterpret_cast<const float2*>(slab + gd.ws_theta);
  double* s2 = reinterpret_cast<double*>(slab + gd.ws_sig2);
  double* shift = reinterpret_cast<double*>(slab + gd.ws_E);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < n; j += 8) {
    const float2* bj = B + (int64_t)j * m;
    double a = 0.0;
    for (int r = lane; r < m; r += 32) a += (double)bj[r].x * bj[r].x + (double)bj[r].y * bj[r].y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) {
      s2[j] = a;
      shift[j] = 0.0;
    }
  }
  (void)np;
  __syncthreads();
  if (threadIdx.x == 0) gd.jrows = n;
}

// The outer sweeps of the three-launch round schedule (k_tc_gram -> k_tc_inner -> k_tc_rot_ws per
// round) over the gates d_list[0..count) (per-list-position ctl / norm2), until every gate's sweep
// rotates nothing or max_sweeps. Returns true if all converged; *launches is advanced.
static bool tc_sweep_rounds(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* d_list, const int32_t* h_list,
                            int count, int max_sweeps, uint8_t* slab, LargeCtl* ctl, const double* norm2,
                            int32_t* unconv, int32_t* h_pinned_flag, cudaStream_t s, int& launches) {
  int max_np = 0;
  for (int g = 0; g < count; ++g) max_np = max(max_np, h_desc[h_list[g]].n_pad);
  const int nb_max = max_np / tcj::TB, pairs_max = nb_max / 2;
  static const int inner_sweeps = getenv("EAMPS_INNER_SWEEPS") ? atoi(getenv("EAMPS_INNER_SWEEPS")) : 1;
  static const bool rot_simple = getenv("EAMPS_ROT_SIMPLE") != nullptr;   // dev A/B switch
  static const float tol_floor = getenv("EAMPS_TC_TOL") ? (float)atof(getenv("EAMPS_TC_TOL")) : 7.62939453125e-6f;
  static const float tol_internal = getenv("EAMPS_TC_TOL_INT") ? (float)atof(getenv("EAMPS_TC_TOL_INT")) : 3.0e38f;
  static const bool prof = getenv("EAMPS_TC_PROF") != nullptr;   // dev: per-kernel device time
  static const int nstreams = getenv("EAMPS_TC_STREAMS") ? atoi(getenv("EAMPS_TC_STREAMS")) : 2;
  static const bool rot_lean = getenv("EAMPS_ROT_LEAN") != nullptr;   // dev A/B switch
  // L2-resident batches: the rounds of a batch stream each gate's Jacobi matrix (B = L, n x n_pad
  // FP32; + V when not preconditioned) through the Gram and rotation kernels three times a round; a
  // batch whose matrices fit the 126 MB L2 (budget 80 MB) keeps those passes out of HBM. A batch
  // still holds enough block pairs for >= 2 waves of the round kernels (kMinPairs), and
  // EAMPS_TC_BATCH=0 runs the whole list at once (the round-1 schedule).
  // Measured slower (chi = 256 x 4096: 1073 vs 1348 updates/s: the round kernels are latency-bound,
  // not HBM-bound, and the smaller grids of a batch overlap less), so EAMPS_TC_BATCH=-1 (auto) is an
  // opt-in and the default runs the whole list at once.
  static const int batch_env = getenv("EAMPS_TC_BATCH") ? atoi(getenv("EAMPS_TC_BATCH")) : 0;
  const size_t per_gate = (size_t)jacobi_rows(h_desc[h_list[0]]) * max_np * 8 *
                          (h_desc[h_list[0]].jrows > 0 ? 1 : 2);
  constexpr size_t kL2Budget = 80ull << 20;
  constexpr int kMinPairs = 296;
  int bsize = count;
  if (batch_env != 0) {
    const int by_l2 = (int)std::max<size_t>(1, kL2Budget / std::max<size_t>(per_gate, 1));
    const int by_par = (kMinPairs + pairs_max - 1) / std::max(pairs_max, 1);
    bsize = batch_env > 0 ? batch_env : std::max(by_l2, by_par);
    bsize = std::min(std::max(bsize, 1), count);
  }
  bool all_done = true;
  static const bool dbg = getenv("EAMPS_TC_DEBUG") != nullptr;
  for (int b0 = 0; b0 < count; b0 += bsize) {
    const int bc = std::min(bsize, count - b0);
    const int32_t* bl = d_list + b0;
    LargeCtl* bctl = ctl + b0;
    const double* bn2 = norm2 + b0;
    static const bool groups_all = getenv("EAMPS_TC_GROUPS_ALL") != nullptr;   // dev A/B: 2 groups at any size
    const int ngroups_want = (!prof && nstreams >= 2 && bc >= 2 && (groups_all || bc * pairs_max < 2048)) ? 2 : 1;
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev_go = nullptr, ev_done = nullptr;
    int ngroups = ngroups_want;
    if (ngroups == 2 && !side_stream(&s2, &ev_go, &ev_done)) ngroups = 1;   // no side stream: one group
    const int gsplit[3] = {0, ngroups == 2 ? bc / 2 : bc, bc};
    if (ngroups == 2) {
      if (cudaEventRecord(ev_go, s) != cudaSuccess) return launches;   // (surfaces as MPS_E_CUDA via CKL)
      cudaStreamWaitEvent(s2, ev_go, 0);      // the preconditioner / init / norms / previous batch are done
    }
    int sweep = 0;
    bool done = false;
    for (; sweep < max_sweeps && !done; ++sweep) {
      static cudaEvent_t ev[4];
      static double acc[3] = {0, 0, 0};
      if (prof && !ev[0])
        for (int e = 0; e < 4; ++e) cudaEventCreate(&ev[e]);
      for (int rnd = 0; rnd < nb_max - 1; ++rnd) {
        for (int gg = 0; gg < ngroups; ++gg) {
          const int g0 = gsplit[gg], gc = gsplit[gg + 1] - g0;
          if (gc <= 0) continue;
          cudaStream_t ss = gg == 0 ? s : s2;
          const dim3 gridg(pairs_max, gc);
          const int32_t* dl = bl + g0;
          LargeCtl* cg = bctl + g0;
          if (prof) cudaEventRecord(ev[0], ss);
          tcj::k_tc_gram<<<gridg, 128, tcj::kGramSmem, ss>>>(d_desc, dl, rnd, slab, cg);
          dbg_sync(ss, "k_tc_gram");
          if (prof) cudaEventRecord(ev[1], ss);
          tcj::k_tc_inner<<<gridg, tcj::kInnerT, tcj::kInnerSmem, ss>>>(d_desc, dl, rnd, slab, cg, bn2 + g0, inner_sweeps,
                                                                       tol_floor, tol_internal);
                                                                       dbg_sync(ss, "k_tc_inner");
          if (prof) cudaEventRecord(ev[2], ss);
          if (rot_simple) tcj::k_tc_rot<<<gridg, 256, tcj::kRotSmem, ss>>>(d_desc, dl, rnd, slab, cg);
          else if (rot_lean)
            tcj::k_tc_rot_ws<tcj::WS_NS_LEAN, tcj::WS_RAW_LEAN><<<gridg, 288, tcj::kRotWsSmemLean, ss>>>(d_desc, dl, rnd, slab, cg);
          else tcj::k_tc_rot_ws<tcj::WS_NS, tcj::WS_RAW><<<gridg, 288, tcj::kRotWsSmem, ss>>>(d_desc, dl, rnd, slab, cg);
          dbg_sync(ss, "k_tc_rot_ws");
          if (prof) {
            cudaEventRecord(ev[3], ss);
            cudaEventSynchronize(ev[3]);
            for (int e = 0; e < 3; ++e) {
              float ms = 0.f;
              cudaEventElapsedTime(&ms, ev[e], ev[e + 1]);
              acc[e] += ms;
            }
          }
          launches += 3;
        }
      }
      if (ngroups == 2) {                     // the second group's round work, before the check
        cudaEventRecord(ev_done, s2);
        cudaStreamWaitEvent(s, ev_done, 0);
      }
      if (prof) fprintf(stderr, "[tc prof] cumulative ms: gram %.1f inner %.1f rot %.1f\n", acc[0], acc[1], acc[2]);
      k_block_check<<<1, 256, 0, s>>>(d_desc, bl, bc, bctl, unconv, 0);
      dbg_sync(s, "k_block_check");
      ++launches;
      cudaMemcpyAsync(h_pinned_flag, unconv, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      done = (h_pinned_flag[0] == 0);
      if (dbg) fprintf(stderr, "[tc] batch %d sweep %d: unconverged gates %d, rotated pairs %d\n", b0, sweep,
                       h_pinned_flag[0], h_pinned_flag[1]);
    }
    all_done &= done;
  }
  return all_done;
}

int run_svd_tc(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* d_list, const int32_t* h_list, int count,
               int max_sweeps, uint8_t* slab, DevState* st, int32_t* d_scratch, int32_t* h_pinned_flag, cudaStream_t s,
               int* error_out) {
  *error_out = 0;
  if (count <= 0) return 0;
  int launches = 0;
  int max_np = 0, max_n = 0;
  for (int g = 0; g < count; ++g) {
    max_np = max(max_np, h_desc[h_list[g]].n_pad);
    max_n = max(max_n, h_desc[h_list[g]].n);
  }
  LargeCtl* ctl = reinterpret_cast<LargeCtl*>(d_scratch);
  double* norm2 = reinterpret_cast<double*>(d_scratch + 2 * ((count + 1) & ~1));
  int32_t* unconv = reinterpret_cast<int32_t*>(norm2 + count);
  cudaMemsetAsync(ctl, 0, sizeof(LargeCtl) * count, s);
  k_large_init<<<dim3(256, count), 256, 0, s>>>(d_desc, d_list, slab);
  k_large_norm<<<count, 256, 0, s>>>(d_desc, d_list, slab, norm2);
  launches += 2;
  bool any_pc = false;
  for (int g = 0; g < count; ++g) any_pc |= h_desc[h_list[g]].jrows > 0;
  if (any_pc) launches += launch_precond_large(d_desc, d_list, count, max_n, slab, s);   // after the norm
  dbg_sync(s, "init/norm/precond");
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(tcj::k_tc_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tcj::kGramSmem);
    cudaFuncSetAttribute(tcj::k_tc_inner, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tcj::kInnerSmem);
    cudaFuncSetAttribute(tcj::k_tc_rot, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tcj::kRotSmem);
    cudaFuncSetAttribute(tcj::k_tc_rot_ws<tcj::WS_NS, tcj::WS_RAW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)tcj::kRotWsSmem);
    cudaFuncSetAttribute(tcj::k_tc_rot_ws<tcj::WS_NS_LEAN, tcj::WS_RAW_LEAN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)tcj::kRotWsSmemLean);
  }
  const int nb_max = max_np / tcj::TB, pairs_max = nb_max / 2;
  static const int inner_sweeps = getenv("EAMPS_INNER_SWEEPS") ? atoi(getenv("EAMPS_INNER_SWEEPS")) : 1;
  // The fused persistent kernel (k_tc_fused) is the EAMPS_TC_FUSED=1 variant: measured slower than the
  // three-launch rounds (chi = 256: 948 vs 1348 updates/s; chi = 1024: 21.0 vs 26.5) -- with its
  // 197 KB of shared memory one CTA per SM runs the latency-bound SIMT inner solve with nothing
  // to overlap it, where the separate kernels keep 2-3 CTAs per SM in flight.
  static const bool fused = getenv("EAMPS_TC_FUSED") != nullptr;
  if (fused) {
    static const float tol_floor_f = getenv("EAMPS_TC_TOL") ? (float)atof(getenv("EAMPS_TC_TOL")) : 7.62939453125e-6f;
    static const float tol_int_f = getenv("EAMPS_TC_TOL_INT") ? (float)atof(getenv("EAMPS_TC_TOL_INT")) : 3.0e38f;
    static std::atomic<unsigned long long> fattr{0};
    if (first_on_device(fattr))
      cudaFuncSetAttribute(tcj::k_tc_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tcj::kFusedSmem);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tcj::k_tc_fused, tcj::FT, tcj::kFusedSmem);
    int32_t* pair_pre = unconv + 2;
    tcj::FusedCtl* fc = reinterpret_cast<tcj::FusedCtl*>(pair_pre + ((count + 1 + 3) & ~3));
    tcj::k_pair_prefix<<<1, 32, 0, s>>>(d_desc, d_list, count, pair_pre, fc);
    int total_pairs = 0;
    for (int g = 0; g < count; ++g) total_pairs += h_desc[h_list[g]].n_pad / tcj::PWC;
    const int grid = std::max(1, std::min(sms * std::max(per_sm, 1), total_pairs));
    GateDesc* a_desc = d_desc;
    const int32_t* a_list = d_list;
    int a_count = count;
    uint8_t* a_slab = slab;
    LargeCtl* a_ctl = ctl;
    const double* a_norm2 = norm2;
    const int32_t* a_pre = pair_pre;
    tcj::FusedCtl* a_fc = fc;
    int a_ms = max_sweeps, a_is = inner_sweeps;
    float a_tf = tol_floor_f, a_ti = tol_int_f;
    void* args[] = {&a_desc, &a_list, &a_count, &a_slab, &a_ctl, &a_norm2, &a_pre, &a_fc, &a_ms, &a_is, &a_tf, &a_ti};
    cudaLaunchCooperativeKernel((const void*)tcj::k_tc_fused, dim3(grid), dim3(tcj::FT), args, tcj::kFusedSmem, s);
    launches += 2;
    cudaMemcpyAsync(h_pinned_flag, &fc->done, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (!h_pinned_flag[0]) *error_out = -6;
    if (any_pc) launches += launch_precond_vnorm(d_desc, d_list, count, max_np, slab, norm2, s);
    launches += launch_spectrum_polish(d_desc, d_list, count, max_n, slab, st, s);
    return launches;
  }
  const bool done = tc_sweep_rounds(d_desc, h_desc, d_list, h_list, count, max_sweeps, slab, ctl, norm2, unconv,
                                    h_pinned_flag, s, launches);
  if (!done) *error_out = -6;
  if (any_pc) launches += launch_precond_vnorm(d_desc, d_list, count, max_np, slab, norm2, s);
  // Opt-in (EAMPS_DEEP=1): measured on config 2 chi = 1024 it lowers the worst sigma error from
  // 7.9e-4 to 1.8e-4 -- still above the 1e-5 bar -- for +7 sweeps (-24 % throughput), and at
  // chi = 512 it raised the error from ~6e-6 to 2.4e-5 (reading 19).
  static const bool deep_on = getenv("EAMPS_DEEP") != nullptr;
  if (!deep_on || max_n <= 256 || !any_pc) {
    launches += launch_spectrum_polish(d_desc, d_list, count, max_n, slab, st, s);
    return launches;
  }
  // ---- deep spectra, n > 256 (n <= 256: the FP64 Rayleigh-Ritz of refine.cu). V = the unit columns
  // of the converged FP32 B = L is accurate only to ~eps32 sigma_max / sigma_j in the small singular
  // directions (L rounded to FP32), which the Rayleigh quotient and the pairwise polish cannot undo
  // when sigma_min / sigma_max < ~5e-5 (config 2 chi = 1024: 7.9e-4 relative error measured). B1 =
  // theta V (FP64-accumulated, FP32 storage: every column keeps its own relative accuracy) has
  // nearly orthogonal columns (coupling <~ 5e-3 relative); more sweeps of the same block Jacobi on
  // B1 converge quadratically, and with rotation angles ~ coupling x sigma_j / sigma_l the FP32 /
  // 3xTF32 rounding they add to a small column is relative to that column; sigma_j = |b1_j| (FP64
  // norms) is then relatively accurate. PAPER.md:114; north_star sigma tolerance.
  k_rayleigh<<<dim3((max_n + 31) / 32, count), 256, 0, s>>>(d_desc, d_list, slab, st, 1);
  ++launches;
  dbg_sync(s, "k_rayleigh");
  static std::atomic<unsigned long long> pattr{0};
  if (first_on_device(pattr))
    cudaFuncSetAttribute(tcj::k_tc_polish, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tcj::kGramSmem);
  const int nbp = ((max_n + tcj::PWC - 1) / tcj::PWC) * 2;
  static const bool no_polish = getenv("EAMPS_NO_POLISH") != nullptr;
  if (!no_polish && nbp >= 2) {
    tcj::k_tc_polish<<<dim3(nbp / 2, count, nbp - 1), 128, tcj::kGramSmem, s>>>(d_desc, d_list, slab);
    dbg_sync(s, "k_tc_polish");
    ++launches;
  }
  int32_t* flags = unconv + 2;                                    // count ints, then the deep list
  k_deep_flags<<<count, 256, 0, s>>>(d_desc, d_list, slab, flags, kDeepRatio * kDeepRatio);
  dbg_sync(s, "k_deep_flags");
  ++launches;
  std::vector<int32_t> hf(count);
  cudaMemcpyAsync(hf.data(), flags, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  std::vector<int32_t> deep_h;                                    // desc indices of the deep gates
  for (int g = 0; g < count; ++g)
    if (hf[g]) deep_h.push_back(h_list[g]);
  const int dc = (int)deep_h.size();
  if (dc > 0) {
    int32_t* dlist = flags + ((count + 1) & ~1);
    double* dnorm2 = reinterpret_cast<double*>(dlist + ((dc + 1) & ~1));
    cudaMemcpyAsync(dlist, deep_h.data(), sizeof(int32_t) * dc, cudaMemcpyHostToDevice, s);
    k_deep_prepare<<<dim3(64, dc), 256, 0, s>>>(d_desc, d_list, count, dlist, slab, ctl, norm2, dnorm2);
    dbg_sync(s, "k_deep_prepare");
    ++launches;
    static const int deep_sweeps = getenv("EAMPS_DEEP_SWEEPS") ? atoi(getenv("EAMPS_DEEP_SWEEPS")) : 8;
    tc_sweep_rounds(d_desc, h_desc, dlist, deep_h.data(), dc, deep_sweeps, slab, ctl, dnorm2, unconv, h_pinned_flag, s,
                    launches);
    k_deep_finish<<<dc, 256, 0, s>>>(d_desc, dlist, slab);
    dbg_sync(s, "k_deep_finish");
    ++launches;
  }
  int npow2 = 1;
  while (npow2 < max_n) npow2 <<= 1;
  const size_t smem = (size_t)npow2 * 12 + 16 + 1024 * 8;
  cudaFuncSetAttribute(k_sort_tails_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_sort_tails_large<<<count, 1024, smem, s>>>(d_desc, d_list, slab, st, 1);
  ++launches;
  dbg_sync(s, "k_sort_tails_large");
  return launches;
}

}  // namespace eamps
