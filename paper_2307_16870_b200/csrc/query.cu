// query.cu -- read-out of the MPS: amplitudes <digits|psi> = prod_i B_i[:, d_i, :]
// (E2; B = Gamma lambda so the lambdas are already absorbed) and the full
// statevector for small N. FP64 accumulation of the complex64 site tensors.
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

}  // namespace

void launch_amplitude_step(uint8_t* slab, const DevState* st, int site, int digit, const double2* vin, double2* vout,
                           cudaStream_t s) {
  k_amp_step<<<64, 256, 0, s>>>(slab, st, site, digit, vin, vout);
}
void launch_statevector_step(uint8_t* slab, const DevState* st, int site, int64_t rows, int cols_in,
                             const double2* Sin, double2* Sout, cudaStream_t s) {
  k_sv_step<<<1024, 256, 0, s>>>(slab, st, site, rows, cols_in, Sin, Sout);
}

}  // namespace eamps
