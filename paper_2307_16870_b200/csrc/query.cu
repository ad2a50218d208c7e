// query.cu -- read-out of the MPS: amplitudes <digits|psi> = prod_i B_i[:, d_i, :]
// (E2; B = Gamma lambda so the lambdas are already absorbed) and the full
// statevector for small N. FP64 accumulation of the complex64 site tensors.
#include <algorithm>

#include "eamps_internal.cuh"

namespace eamps {

namespace {

__global__ void k_amp_step(uint8_t* slab, const DevState* st, int site, int digit, const double2* vin, double2* vout) {
  const SiteEntry e = reinterpret_cast<const SiteEntry*>(slab + st->sites_off)[site];
  const float2* B = reinterpret_cast<const float2*>(slab + e.off);
  const int d = st->d;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < e.chr; c += gridDim.x * blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int a = 0; a < e.chl; ++a) {
      double2 v = vin[a];
      float2 b = B[((int64_t)a * d + digit) * e.chr + c];
      re += v.x * b.x - v.y * b.y;
      im += v.x * b.y + v.y * b.x;
    }
    vout[c] = make_double2(re, im);
  }
}

// Sout[(p d + s) r + c] = sum_a Sin[p cols + a] B[(a d + s) r + c]
__global__ void k_sv_step(uint8_t* slab, const DevState* st, int site, int64_t rows, int cols,
                          const double2* Sin, double2* Sout) {
  const SiteEntry e = reinterpret_cast<const SiteEntry*>(slab + st->sites_off)[site];
  const float2* B = reinterpret_cast<const float2*>(slab + e.off);
  const int d = st->d, r = e.chr;
  const int64_t tot = rows * d * r;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = x % r, ps = x / r;
    int64_t s = ps % d, p = ps / d;
    double re = 0.0, im = 0.0;
    for (int a = 0; a < cols; ++a) {
      double2 v = Sin[p * cols + a];
      float2 b = B[((int64_t)a * d + s) * r + c];
      re += v.x * b.x - v.y * b.y;
      im += v.x * b.y + v.y * b.x;
    }
    Sout[x] = make_double2(re, im);
  }
}

// ---- observables (NEXT-4): transfer-matrix contractions, FP64 accumulation ---------------------
template <typename T>
__device__ __forceinline__ double2 ld2(const T* p, int64_t i) {
  const T v = p[i];
  return make_double2((double)v.x, (double)v.y);
}

// T[x, s, yp] = sum_y E[x, y] B[y, s, yp]        E: la x lb, B: (lb, D, rb), T: (la, D, rb)
template <typename TB>
__global__ void k_xfer_T(const double2* __restrict__ E, const TB* __restrict__ B, double2* __restrict__ Tout, int la,
                         int lb, int D, int rb) {
  const int64_t tot = (int64_t)la * D * rb;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < tot; o += (int64_t)gridDim.x * blockDim.x) {
    const int yp = (int)(o % rb);
    const int64_t xs = o / rb;
    const int s = (int)(xs % D), x = (int)(xs / D);
    double re = 0.0, im = 0.0;
    for (int y = 0; y < lb; ++y) {
      const double2 e = E[(int64_t)x * lb + y];
      const double2 b = ld2(B, ((int64_t)y * D + s) * rb + yp);
      re = fma(e.x, b.x, fma(-e.y, b.y, re));
      im = fma(e.x, b.y, fma(e.y, b.x, im));
    }
    Tout[o] = make_double2(re, im);
  }
}

// E'[xp, yp] = sum_{x, s} conj(A[x, s, xp]) T[x, s, yp]     A: (la, D, ra), E': ra x rb
template <typename TA>
__global__ void k_xfer_E(const TA* __restrict__ A, const double2* __restrict__ Tin, double2* __restrict__ Eout, int la,
                         int D, int ra, int rb) {
  const int64_t tot = (int64_t)ra * rb;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < tot; o += (int64_t)gridDim.x * blockDim.x) {
    const int yp = (int)(o % rb), xp = (int)(o / rb);
    double re = 0.0, im = 0.0;
    for (int x = 0; x < la; ++x)
      for (int s = 0; s < D; ++s) {
        const double2 a = ld2(A, ((int64_t)x * D + s) * ra + xp);
        const double2 t = Tin[((int64_t)x * D + s) * rb + yp];
        re = fma(a.x, t.x, fma(a.y, t.y, re));      // conj(a) t
        im = fma(a.x, t.y, fma(-a.y, t.x, im));
      }
    Eout[o] = make_double2(re, im);
  }
}

// theta[a, s d + t, c] = sum_b B_k[a, s, b] B_{k+1}[b, t, c]     (the two-site tensor of E5)
__global__ void k_theta2(const float2* __restrict__ Bk, const float2* __restrict__ Bk1, double2* __restrict__ th, int l,
                         int d, int mid, int r) {
  const int64_t tot = (int64_t)l * d * d * r;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < tot; o += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(o % r);
    const int64_t ast = o / r;
    const int t = (int)(ast % d), s = (int)((ast / d) % d), a = (int)(ast / (d * d));
    double re = 0.0, im = 0.0;
    for (int b = 0; b < mid; ++b) {
      const float2 u = Bk[((int64_t)a * d + s) * mid + b], v = Bk1[((int64_t)b * d + t) * r + c];
      re = fma((double)u.x, (double)v.x, fma(-(double)u.y, (double)v.y, re));
      im = fma((double)u.x, (double)v.y, fma((double)u.y, (double)v.x, im));
    }
    th[o] = make_double2(re, im);
  }
}

// Oth[a, st, c] = sum_{s't'} O[st, s't'] theta[a, s't', c]      O: D x D (D = d^2) complex64
__global__ void k_apply_O(const float2* __restrict__ O, const double2* __restrict__ th, double2* __restrict__ out, int l,
                          int D, int r) {
  const int64_t tot = (int64_t)l * D * r;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < tot; o += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(o % r);
    const int64_t ast = o / r;
    const int st = (int)(ast % D), a = (int)(ast / D);
    double re = 0.0, im = 0.0;
    for (int sp = 0; sp < D; ++sp) {
      const float2 u = O[st * D + sp];
      const double2 v = th[((int64_t)a * D + sp) * r + c];
      re = fma((double)u.x, v.x, fma(-(double)u.y, v.y, re));
      im = fma((double)u.x, v.y, fma((double)u.y, v.x, im));
    }
    out[o] = make_double2(re, im);
  }
}

// v'[c] = sum_x v[x] (B[x, 0, c] + B[x, 3, c])    (Tr rho of a vectorised MPO, s = 2 sigma + sigma')
__global__ void k_trace_step(const float2* __restrict__ B, const double2* __restrict__ vin, double2* __restrict__ vout,
                             int l, int r) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < r; c += gridDim.x * blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int x = 0; x < l; ++x) {
      const float2 b0 = B[((int64_t)x * 4 + 0) * r + c], b3 = B[((int64_t)x * 4 + 3) * r + c];
      const double2 v = vin[x];
      const double br = (double)b0.x + b3.x, bi = (double)b0.y + b3.y;
      re = fma(v.x, br, fma(-v.y, bi, re));
      im = fma(v.x, bi, fma(v.y, br, im));
    }
    vout[c] = make_double2(re, im);
  }
}

inline int grid_for(int64_t n) { return (int)std::min<int64_t>(4096, std::max<int64_t>(1, (n + 255) / 256)); }

}  // namespace

// one transfer step E' = sum_s A^{s dagger} E B^s with FP32 (site) or FP64 (two-site) tensors
void launch_transfer(const double2* E, const void* A, bool a64, const void* B, bool b64, double2* Tbuf, double2* Eout,
                     int la, int lb, int D, int ra, int rb, cudaStream_t s) {
  const int64_t nt = (int64_t)la * D * rb, ne = (int64_t)ra * rb;
  if (b64) k_xfer_T<double2><<<grid_for(nt), 256, 0, s>>>(E, static_cast<const double2*>(B), Tbuf, la, lb, D, rb);
  else k_xfer_T<float2><<<grid_for(nt), 256, 0, s>>>(E, static_cast<const float2*>(B), Tbuf, la, lb, D, rb);
  if (a64) k_xfer_E<double2><<<grid_for(ne), 256, 0, s>>>(static_cast<const double2*>(A), Tbuf, Eout, la, D, ra, rb);
  else k_xfer_E<float2><<<grid_for(ne), 256, 0, s>>>(static_cast<const float2*>(A), Tbuf, Eout, la, D, ra, rb);
}
void launch_theta2(const float2* Bk, const float2* Bk1, double2* th, int l, int d, int mid, int r, cudaStream_t s) {
  k_theta2<<<grid_for((int64_t)l * d * d * r), 256, 0, s>>>(Bk, Bk1, th, l, d, mid, r);
}
void launch_apply_O(const float2* O, const double2* th, double2* out, int l, int D, int r, cudaStream_t s) {
  k_apply_O<<<grid_for((int64_t)l * D * r), 256, 0, s>>>(O, th, out, l, D, r);
}
void launch_trace_step(const float2* B, const double2* vin, double2* vout, int l, int r, cudaStream_t s) {
  k_trace_step<<<grid_for(r), 256, 0, s>>>(B, vin, vout, l, r);
}

void launch_amplitude_step(uint8_t* slab, const DevState* st, int site, int digit, const double2* vin, double2* vout,
                           cudaStream_t s) {
  k_amp_step<<<64, 256, 0, s>>>(slab, st, site, digit, vin, vout);
}
void launch_statevector_step(uint8_t* slab, const DevState* st, int site, int64_t rows, int cols_in,
                             const double2* Sin, double2* Sout, cudaStream_t s) {
  k_sv_step<<<1024, 256, 0, s>>>(slab, st, site, rows, cols_in, Sin, Sout);
}

}  // namespace eamps
