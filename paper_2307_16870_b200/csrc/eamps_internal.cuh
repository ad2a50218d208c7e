// eamps_internal.cuh -- device-side data structures and kernel entry points of the B200 path.
//
// Product code. It shares nothing with oracle/ (no headers, constants or helpers).
// Layouts:
//   * site tensor B_i: row-major (chi_l, d, chi_r) complex64 in a pool block of the slab
//   * Schmidt vector lambda_b: float32 in a pool block
//   * per-gate workspace (top of the slab): theta, Theta' column-major (m x n, ld m),
//     V column-major (n_pad x n_pad), sigma^2 (f64, n_pad), tails T (f64, n_pad+1), pi (i32)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace eamps {

// cudaFuncSetAttribute (e.g. the >48 KB dynamic shared-memory opt-in) applies to the CURRENT
// device only: a per-call-site bit mask of the devices already configured. Returns true exactly
// once per device (thread-safe).
inline bool first_on_device(std::atomic<unsigned long long>& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return true;
  const unsigned long long bit = 1ull << (dev & 63);
  return (mask.fetch_or(bit) & bit) == 0;
}

// Pool size classes (round 2): class c holds blocks of class_bytes(c) = 2^(c/2) (c even) or
// 1.5 x 2^((c-1)/2) (c odd, from 768 B up), so a block wastes at most a third of itself instead of
// half (power-of-two classes put a chi = 4096 site tensor of 268 MB into a 512 MB block: config 5 ran
// out of slab at layer 20, r01). All classes are multiples of 256 B. 96 classes cover 2^47 B.
constexpr int kMaxClasses = 96;
constexpr int kMinClass = 16;       // 256 B

struct SiteEntry {                  // B_i
  int64_t off;                      // byte offset in the slab (0 = none)
  int32_t chl, chr;
  int32_t cls, pad;
};
struct BondEntry {                  // lambda of bond b, stored at index b+1 (b = -1 .. N-1)
  int64_t off;
  int32_t len, cls;
};

struct DevLedger {                  // E12/E14 ledger, log space (reading 10)
  double logE;
  int64_t j;
  int32_t guarantee;                // 1 until a cap fires
  int32_t error;                    // sticky device error (MPS_E_*), 0 = none
  double log_fmin, log_ffixed;
  int64_t n_planned;
  int32_t strategy, rule, chi_cap, d;
};

struct DevPool {
  uint64_t bump;                    // next never-used byte (absolute slab offset)
  uint64_t ceiling;                 // host-set upper limit of pool allocations
  int32_t count[kMaxClasses];       // free-stack depth per size class
  int64_t stack_off;                // slab offset of the free stacks: kMaxClasses x stack_cap int64
  int64_t stack_cap;
  int64_t npending;                 // deferred frees (released at the next commit launch)
  int64_t pending_cap;
  int64_t pending_off;              // slab offset of the pending array (int64 pairs: off, cls)
};

// One per gate of a wave (device array, built by the host).
struct GateDesc {
  int32_t site, l, mid, r;          // chi_l, chi_m, chi_r
  int32_t m, n, n_pad, regime;      // theta is m x n (m = d l, n = d r); regime 0 small, 1 large, 2 medium, 3 QR
  int64_t ws_theta, ws_thetap, ws_V, ws_sig2, ws_T, ws_pi;   // slab offsets
  int64_t ws_E;                     // Newton-Schulz correction E (k x k) of the kept V columns
  int64_t ws_log;                   // medium: rotation log, log_sweeps x (n-1) x n/2 float4 (c, s, e); large: TC scratch
  int32_t log_sweeps;
  int32_t eig, eig_pad;             // 1: the eigen route (refine_large.cu: FP64 Gram eigensolver, no Jacobi)
  int32_t jrows;                    // large regime: 0 = Jacobi on theta (m rows) with V accumulated;
                                    // > 0 = preconditioned, Jacobi on B = L (jrows = n rows), no V
  int32_t u_index, sweeps;          // gate matrix index in the staged array; sweeps used
  int32_t k, capped;                // outputs of the selector
  int64_t off_newL, off_newR, off_newLam;                    // outputs of the selector
  double nu;                        // sqrt(kept weight)
  double f, t;                      // achieved / target truncation fidelity
  double dlogE, disc;               // log f, discarded weight T_k / P
};

__host__ __device__ inline int jacobi_rows(const GateDesc& g) { return g.jrows > 0 ? g.jrows : g.m; }

struct Record {                     // == mps_record
  int64_t gate_index;
  int32_t bond, chi_before, chi_after, capped;
  double target_f, achieved_f, discarded_weight;
};

struct ImportEntry {                // bulk site import (mps_import_sites)
  int32_t site, chl, chr, resetL, resetR, pad;   // reset*: lambda extents to set to ones (0 = keep)
  int64_t src_elem;                 // first complex element of this site in the source buffer
  int64_t dst_off, lamL_off, lamR_off;           // written by the device allocator
};

struct ExportEntry {                // bulk site export (mps_export_sites)
  int64_t src_off;                  // byte offset of the site tensor in the slab
  int64_t dst_elem;                 // first complex element of this site in the destination buffer
  int64_t elems;                    // chl * d * chr
};

struct DevState {                   // lives at slab offset 0
  DevLedger led;
  DevPool pool;
  int32_t n_sites, d;
  int64_t sites_off, bonds_off;     // SiteEntry[N], BondEntry[N+1]
};

__host__ __device__ inline uint64_t class_bytes(int c) {
  return (c & 1) ? (3ull << ((c - 3) >> 1)) : (1ull << (c >> 1));
}
__host__ __device__ inline int size_class(uint64_t bytes) {
  if (bytes <= 256) return kMinClass;
  int k = 9;                                  // smallest k with 2^k >= bytes
  while ((1ull << k) < bytes) ++k;
  if (k - 1 >= 9 && bytes <= (3ull << (k - 2))) return 2 * k - 1;   // 1.5 x 2^(k-1)
  return 2 * k;
}

template <typename T>
__host__ __device__ inline T* at(uint8_t* slab, int64_t off) { return reinterpret_cast<T*>(slab + off); }

// ---- kernels (launched by capi.cu) -------------------------------------------------------------
void launch_contract(const GateDesc* d_desc, const int32_t* d_tile_prefix, int G, int total_tiles, int d,
                     uint8_t* slab, const DevState* st, const float2* d_us, cudaStream_t s);
// rows per lane for a GT-lane group over `rows` rows: a power of two <= 16, or 0 (no register path)
inline int rows_per_lane(int rows, int gt) {
  const int need = (rows + gt - 1) / gt;
  int r = 1;
  while (r < need) r <<= 1;
  return r <= 16 ? r : 0;
}
size_t svd_qr_smem(int m, int n);
bool svd_qr_fits(int m, int n, int* gt_out, int* rpl_out);
bool qr_block_order(int m, int n);
// packed = 1: n == rpl * gt and m even (16-byte row pairs); buckets must not mix packed and unpacked
void launch_svd_qr(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem, int max_sweeps, int gt, int rpl,
                   int packed, uint8_t* slab, DevState* st, cudaStream_t s);
size_t svd_small_smem(int m, int n);
bool svd_small_fits(int m, int n);
int small_group(int m);
void launch_svd_small(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem, int max_sweeps, int gt, int rpl,
                      int threads, uint8_t* slab, DevState* st, cudaStream_t s);
size_t svd_theta_smem(int m, int n);
size_t svd_vrep_smem(int n, int tile_rows);
bool svd_medium_fits(int m, int n);
int vrep_tile_rows(int m, int n);
void launch_svd_medium(GateDesc* d_desc, const int32_t* d_list, int count, size_t smem_theta, size_t smem_vrep,
                       int tile_rows, int max_sweeps, int gt, int rpl, int threads, uint8_t* slab, DevState* st,
                       cudaStream_t s);
// blocked (large) path: returns launches issued
int run_svd_blocked(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* d_list, const int32_t* h_list, int count,
                    int max_sweeps, uint8_t* slab, DevState* st, int32_t* d_counters, int32_t* h_pinned_flag,
                    cudaStream_t s, int* error_out);
// tensor-core (tcgen05 3xTF32) blocked Jacobi: n_pad multiple of 64, per-gate scratch at ws_log
size_t svd_tc_scratch_bytes(int n_pad);
// large-regime R-preconditioner (precond_large.cu): FP64 Gram + Cholesky -> B = L, no V accumulation
bool large_precond_enabled();
bool large_precond_wide();
size_t large_precond_scratch(int n);
int launch_precond_large(GateDesc* d_desc, const int32_t* d_list, int count, int max_n, uint8_t* slab, cudaStream_t s);
int launch_precond_vnorm(GateDesc* d_desc, const int32_t* d_list, int count, int max_np, uint8_t* slab,
                         const double* norm2, cudaStream_t s);
int run_svd_tc(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* d_list, const int32_t* h_list, int count,
               int max_sweeps, uint8_t* slab, DevState* st, int32_t* d_counters, int32_t* h_pinned_flag,
               cudaStream_t s, int* error_out);
int launch_spectrum_polish(GateDesc* d_desc, const int32_t* d_list, int count, int max_n, uint8_t* slab, DevState* st,
                           cudaStream_t s);
// FP64 Rayleigh-Ritz refinement of deep spectra (refine.cu): one CTA per gate of the wave (desc[0..G)),
// gates with n > 256 or a shallow spectrum exit at once. refine_scratch_bytes: the global C
// scratch a gate with n in (128, 256] needs at ws_log (0 otherwise).
size_t refine_scratch_bytes(int n);
int launch_refine(GateDesc* d_desc, int G, int max_n, uint8_t* slab, DevState* st, const float2* d_us,
                  int32_t* d_list /* G + 1 ints */, cudaStream_t s);
// FP64 eigenvalues of the Gram of the FP64-recontracted theta for deep large-regime gates with
// 256 < n <= 4096 (refine_large.cu). cand = the wave's large-regime gates (host and device copies);
// iscr: wave scratch of 2 nc + 2 ints + 19 KB (barrier lines). Returns launches issued.
// profiling hook: mark(ctx) records an event on the stream and returns its id (or -1); the front
// stores the ids taken just before and after the tridiagonalisation kernel in at[0], at[1]
struct RlgMarks {
  int (*mark)(void*);
  void* ctx;
  mutable int at[2];
};
bool refine_large_candidate(const GateDesc& gd);
bool eig_route(const GateDesc& gd);
int launch_eig_front(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* h_cand, const int32_t* d_cand, int nc,
                     uint8_t* slab, DevState* st, const float2* d_us, int d, int32_t* iscr, int32_t* fb,
                     cudaStream_t s, const RlgMarks* mk);
int launch_eig_vectors(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* h_cand, const int32_t* d_cand, int nc,
                       uint8_t* slab, cudaStream_t s, int want);
// the eigen route for QR-regime thetas (n <= 128): one CTA per gate (refine_large.cu, k_eig_cta)
bool eig_route_small(const GateDesc& gd);
int launch_eig_small_front(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* h_cand, const int32_t* d_cand,
                           int nc, uint8_t* slab, DevState* st, const float2* d_us, int d, int32_t* iscr,
                           cudaStream_t s, const struct RlgMarks* mk);
size_t refine_large_scratch(int m, int n);
int launch_refine_large(GateDesc* d_desc, const GateDesc* h_desc, const int32_t* h_cand, const int32_t* d_cand, int nc,
                        uint8_t* slab, DevState* st, const float2* d_us, int d, int32_t* iscr, cudaStream_t s);
// parallel = 1: FIXED / NAIVE (target independent of the ledger): one warp per gate;
// parallel = 0: GLOBAL / NEAREST: one warp walks the gates in canonical order.
void launch_select(GateDesc* d_desc, int G, uint8_t* slab, DevState* st, Record* d_rec, int parallel, cudaStream_t s);
int launch_reabsorb(const GateDesc* d_desc, const int32_t* d_pre_gram, int tiles_gram, const int32_t* d_pre_apply,
                    int tiles_apply, const int32_t* d_pre_reab, int tiles_reab, int G, uint8_t* slab, cudaStream_t s);
// small gates (m, n <= 64): the reabsorb fused in one CTA per gate (list = wave-local indices)
bool reabsorb_small_fits(int m, int n);
size_t reabsorb_small_smem(int m, int n);
void launch_reabsorb_small(const GateDesc* d_desc, const int32_t* d_list, int count, size_t smem, uint8_t* slab,
                           cudaStream_t s);
void launch_import(uint8_t* slab, DevState* st, ImportEntry* d_ent, int count, const float2* src, int d,
                   cudaStream_t s);
// gather of `count` site tensors into one contiguous buffer (mps_export_sites); `split` CTAs per site
void launch_export(const uint8_t* slab, const ExportEntry* d_ent, int count, int split, float2* dst, cudaStream_t s);
void launch_pool_alloc(uint8_t* slab, DevState* st, uint64_t bytes, int64_t* d_out, cudaStream_t s);
void launch_pool_free(uint8_t* slab, DevState* st, int64_t off, int cls, cudaStream_t s);
void launch_gate1(uint8_t* slab, DevState* st, int site, int d, const float2* d_u, cudaStream_t s);
void launch_gate1_layer(uint8_t* slab, DevState* st, int count, const int32_t* d_sites, const float2* d_us, int d,
                        cudaStream_t s);
void launch_amplitude_step(uint8_t* slab, const DevState* st, int site, int digit, const double2* vin, double2* vout,
                           cudaStream_t s);
// observables (NEXT-4, query.cu)
void launch_transfer(const double2* E, const void* A, bool a64, const void* B, bool b64, double2* Tbuf, double2* Eout,
                     int la, int lb, int D, int ra, int rb, cudaStream_t s);
void launch_theta2(const float2* Bk, const float2* Bk1, double2* th, int l, int d, int mid, int r, cudaStream_t s);
void launch_apply_O(const float2* O, const double2* th, double2* out, int l, int D, int r, cudaStream_t s);
void launch_trace_step(const float2* B, const double2* vin, double2* vout, int l, int r, cudaStream_t s);
void launch_statevector_step(uint8_t* slab, const DevState* st, int site, int64_t rows, int cols_in,
                             const double2* Sin, double2* Sout, cudaStream_t s);

}  // namespace eamps
