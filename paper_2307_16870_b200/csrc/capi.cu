// capi.cu -- the C ABI (include/eamps.h) and the host-side layer scheduler (step a0):
// validate the brickwork layer (disjoint LNN pairs), bucket its gates by SVD regime,
// plan waves against the slab, stage the gates with one H2D copy, launch the grouped kernels
//   contract (all) -> SVD small (one CTA per theta) | SVD blocked (large) -> select (one warp,
//   canonical order) -> reabsorb (all)
// and read back the new bond profile, ledger and truncation records (one sync per wave).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstddef>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <array>
#include <chrono>
#include <map>
#include <vector>

#include "eamps.h"
#include "eamps_internal.cuh"

using namespace eamps;

static_assert(sizeof(Record) == sizeof(mps_record), "record layout");

// NVTX range over a host-side scope (a timeline tool shows the layer / wave / step structure over
// the kernels launched inside it; header-only NVTX 3: a no-op call when no tool is attached)
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};

struct LayerPlan {                 // per gate of a layer (a0 planning)
  GateDesc gd;
  size_t ws, reserve;
  int ctiles, rtiles, gtiles, atiles;
};

struct LayerJob {                  // the layer in flight (mps_layer_begin / mps_layer_step)
  bool active = false, front = false;
  int G = 0, d4 = 0, g0 = 0, g1 = 0, Gw = 0;
  std::vector<std::pair<int, int>> ord;
  std::vector<LayerPlan> plan;
  std::vector<float> us;             // the caller's gates, copied at begin
  std::vector<GateDesc> hd;          // the current wave
  std::vector<int32_t> rpre, gpre, apre;
  size_t o_desc = 0, o_rec = 0, o_gpre = 0, o_apre = 0, o_rpre = 0, tail = 0;
  std::vector<int32_t> rsm;          // wave-local gates of the fused small reabsorb
  size_t o_rsm = 0, rsm_smem = 0;
  std::vector<int32_t> eigl;         // wave-local gates of the eigen route (refine_large.cu)
  size_t o_eigl = 0;
  std::vector<int32_t> eigs;         // ... its one-CTA form for QR-regime thetas (n <= 128)
  size_t o_eigs = 0;
  bool ran[5] = {false, false, false, false, false};
};

constexpr int kPhases = 10;

// EAMPS_HOST_PROF=1: host-side time of the layer path (planning before the first launch, the
// launch calls, the post-sync bookkeeping), printed by mps_destroy -- the GPU idles through the
// first and the last. Development instrumentation; off by default.
struct HostProf {
  bool on = getenv("EAMPS_HOST_PROF") != nullptr;
  double plan = 0, launch = 0, wait = 0, post = 0, wplan = 0, mark = 0;
  int64_t layers = 0;
  static double now() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
};

struct mps_handle {
  int N = 0, d = 0;
  int device = 0;                          // the device of the slab: made current at every ABI entry
  mps_config cfg{};
  cudaStream_t s = nullptr;
  uint8_t* slab = nullptr;
  size_t slab_bytes = 0;
  DevState* dst = nullptr;
  uint64_t pool_base = 0;
  std::vector<int32_t> chl, chr, lamlen;  // host mirror of the bond profile
  DevState hstate{};                       // host copy after the last sync
  std::vector<mps_record> records;
  std::vector<GateDesc> last_desc;         // every wave of the last layer (k, sweeps)
  LayerJob job;
  int last_wave_begin = 0;                 // spectra are readable for the final wave only ...
  bool keep_spectra = false;               // ... unless mps_keep_spectra: a host copy per gate, every wave
  std::vector<std::vector<double>> spectra;   // parallel to last_desc (sigma^2, sorted), when kept
  bool poisoned = false;
  int sticky = 0;
  std::string err;
  int64_t launches = 0;
  void* pinned[2] = {nullptr, nullptr};   // [0] general / readback, [1] layer upload staging
  uint8_t* pinned_dev[2] = {nullptr, nullptr};   // their device (UVA-mapped) addresses
  size_t pinned_bytes[2] = {0, 0};
  // phase timers (mps_set_profiling): CUDA events recorded on the launch stream around each phase
  bool profiling = false;
  bool jacobi_only = false;              // mps_set_svd_route(h, 1): no eigen route (A/B, tests)
  // [0] contract [1] svd_small (small / medium / QR regimes) [2] svd_blocked (large regime) [3] select
  // [4] reabsorb, and sub-phases of the SVD (spans, one per bucket launch group): [5] preconditioner
  // (FP64 Gram + Cholesky + B = L) [6] the Jacobi kernel itself [7] spectrum (Rayleigh + polish + sort)
  double phase_ms[kPhases] = {};
  int64_t phase_n[kPhases] = {};
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  HostProf hp;
  std::vector<cudaEvent_t> span_ev;          // event pool for the sub-phase spans of one wave
  int span_used = 0;
  std::vector<std::array<int, 3>> spans;     // (phase, begin event, end event)
  // host side of a snapshot
  struct Snap {
    bool valid = false;
    std::vector<int32_t> chl, chr, lamlen;
    DevState hstate{};
    size_t nrec = 0;
  } snap;
};

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }

mps_status set_err(mps_t h, mps_status st, const std::string& msg) {
  if (h) h->err = msg;
  return st;
}

// Makes the handle's device current for the duration of an ABI call (the library never assumes
// that the caller's current device is the slab's), and restores the caller's device after.
struct DeviceGuard {
  int prev = -1, want = -1;
  explicit DeviceGuard(const mps_handle* h) {
    if (!h) return;
    want = h->device;
    if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); prev = -1; }
    if (prev != want) cudaSetDevice(want);
  }
  ~DeviceGuard() {
    if (prev >= 0 && prev != want) cudaSetDevice(prev);
  }
};
#define DEVICE_GUARD(h) DeviceGuard _device_guard(h)

mps_status cuda_check(mps_t h, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return MPS_OK;
  h->poisoned = true;
  return set_err(h, MPS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                            \
  do {                                                      \
    mps_status _st = cuda_check(h, (call), #call);          \
    if (_st != MPS_OK) return _st;                          \
  } while (0)

#define CKL(what)                                           \
  do {                                                      \
    mps_status _st = cuda_check(h, cudaGetLastError(), what); \
    if (_st != MPS_OK) return _st;                          \
  } while (0)

// Sub-phase timing (profiling only): record a pooled event on the launch stream; returns its index.
int prof_mark(mps_t h) {
  if (h->span_used == (int)h->span_ev.size()) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    h->span_ev.push_back(e);
  }
  if (cudaEventRecord(h->span_ev[h->span_used], h->s) != cudaSuccess) return -1;
  return h->span_used++;
}
void prof_span(mps_t h, int phase, int a, int b) {
  if (a >= 0 && b >= 0) h->spans.push_back({phase, a, b});
}

// Pinned staging buffers. Growing one first drains the stream so that no in-flight async copy
// still reads or writes the old buffer.
void* pinned_buf(mps_t h, size_t bytes, int which = 0) {
  if (bytes > h->pinned_bytes[which]) {
    if (h->s) cudaStreamSynchronize(h->s); else cudaDeviceSynchronize();
    if (h->pinned[which]) cudaFreeHost(h->pinned[which]);
    size_t nb = std::max(bytes, h->pinned_bytes[which] * 2);
    // mapped: the small uploads below read it from the SMs (h2d_small)
    void* dp = nullptr;
    if (cudaHostAlloc(&h->pinned[which], nb, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
        cudaHostGetDevicePointer(&dp, h->pinned[which], 0) != cudaSuccess) {
      if (h->pinned[which]) cudaFreeHost(h->pinned[which]);
      h->pinned[which] = nullptr;
      h->pinned_bytes[which] = 0;
      return nullptr;
    }
    h->pinned_dev[which] = static_cast<uint8_t*>(dp);
    h->pinned_bytes[which] = nb;
  }
  return h->pinned[which];
}

// Small host->device uploads (layer descriptors, gate matrices, import entries, scalars) are read
// by a copy kernel from the mapped pinned buffer instead of going through a DMA copy: a DMA H2D
// on this stream queues behind whatever bulk H2D the caller has in flight on another stream (the
// e2e pipeline copies the next chunk's site tensors while this chunk updates), which stalled the
// whole layer for the length of that bulk copy (measured: tools/dev/e2e_overlap.py). `src` must
// lie in one of the handle's pinned buffers.
__global__ void k_h2d_mapped(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src, size_t bytes) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t done = 0;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    const size_t n16 = bytes >> 4;
    for (size_t x = i; x < n16; x += stride) reinterpret_cast<uint4*>(dst)[x] = reinterpret_cast<const uint4*>(src)[x];
    done = n16 << 4;
  }
  for (size_t x = done + i; x < bytes; x += stride) dst[x] = src[x];
}

cudaError_t h2d_small(mps_t h, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  const uint8_t* hs = static_cast<const uint8_t*>(src);
  const uint8_t* ds = nullptr;
  for (int w = 0; w < 2; ++w) {
    const uint8_t* b = static_cast<const uint8_t*>(h->pinned[w]);
    if (b && hs >= b && hs + bytes <= b + h->pinned_bytes[w]) ds = h->pinned_dev[w] + (hs - b);
  }
  if (!ds) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->s);
  const size_t n16 = (bytes + 15) / 16;
  const int blocks = (int)std::min<size_t>(296, std::max<size_t>(1, (n16 + 255) / 256));
  k_h2d_mapped<<<blocks, 256, 0, h->s>>>(static_cast<uint8_t*>(dst), ds, bytes);
  ++h->launches;
  return cudaGetLastError();
}

mps_status sync_state(mps_t h) {
  DevState* hs = static_cast<DevState*>(pinned_buf(h, sizeof(DevState)));
  if (!hs) return set_err(h, MPS_E_NOMEM, "pinned host allocation failed");
  CK(cudaMemcpyAsync(hs, h->dst, sizeof(DevState), cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  h->hstate = *hs;
  return MPS_OK;
}

mps_status check_sticky(mps_t h) {
  if (h->poisoned) return set_err(h, MPS_E_CUDA, h->err.empty() ? "handle poisoned" : h->err);
  if (h->sticky) return h->sticky;
  return MPS_OK;
}

const char* status_name(mps_status s) {
  switch (s) {
    case MPS_OK: return "ok";
    case MPS_E_INVAL: return "invalid argument";
    case MPS_E_RANGE: return "index out of range";
    case MPS_E_NOMEM: return "out of slab / pool memory";
    case MPS_E_CUDA: return "CUDA error";
    case MPS_E_NCCL: return "NCCL error";
    case MPS_E_NOCONV: return "Jacobi SVD did not converge";
    case MPS_E_NUMERIC: return "non-finite singular value";
    case MPS_E_STATE: return "ledger/state error";
    case MPS_E_TOOBIG: return "query too large";
    default: return "unknown";
  }
}

mps_status device_error(mps_t h) {
  int e = h->hstate.led.error;
  if (e == 0) return MPS_OK;
  h->sticky = e;
  if (e == MPS_E_NOMEM) h->poisoned = true;  // the site table may be half-updated
  std::string detail;
  if (e == MPS_E_NOMEM) {
    const DevPool& P = h->hstate.pool;
    char buf[256];
    int worst = 0;
    for (int c = 0; c < kMaxClasses; ++c) worst = std::max(worst, (int)P.count[c]);
    snprintf(buf, sizeof buf, " (pool bump %llu, ceiling %llu, slab %zu, fullest free stack %d of %lld)",
             (unsigned long long)P.bump, (unsigned long long)P.ceiling, h->slab_bytes, worst, (long long)P.stack_cap);
    detail = buf;
  }
  return set_err(h, e, std::string("device: ") + status_name(e) + detail);
}

// ---- device pool helpers for host-side operations (not on the hot path) -------------------
mps_status dev_alloc(mps_t h, uint64_t bytes, int64_t* off, int* cls) {
  // scratch: the last 256 bytes of the slab
  int64_t* dout = reinterpret_cast<int64_t*>(h->slab + h->slab_bytes - kAlign);
  launch_pool_alloc(h->slab, h->dst, bytes, dout, h->s);
  ++h->launches;
  CKL("pool_alloc");
  int64_t* hb = static_cast<int64_t*>(pinned_buf(h, 16));
  CK(cudaMemcpyAsync(hb, dout, 16, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  *off = hb[0];
  *cls = (int)hb[1];
  if (*off == 0) {
    mps_status st = sync_state(h);
    if (st != MPS_OK) return st;
    return device_error(h) != MPS_OK ? h->sticky : set_err(h, MPS_E_NOMEM, "pool exhausted");
  }
  return MPS_OK;
}

mps_status read_site(mps_t h, int site, SiteEntry* e) {
  SiteEntry* hb = static_cast<SiteEntry*>(pinned_buf(h, sizeof(SiteEntry)));
  CK(cudaMemcpyAsync(hb, h->slab + h->hstate.sites_off + sizeof(SiteEntry) * site, sizeof(SiteEntry),
                     cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  *e = *hb;
  return MPS_OK;
}

mps_status read_bond(mps_t h, int bond, BondEntry* e) {
  BondEntry* hb = static_cast<BondEntry*>(pinned_buf(h, sizeof(BondEntry)));
  CK(cudaMemcpyAsync(hb, h->slab + h->hstate.bonds_off + sizeof(BondEntry) * (bond + 1), sizeof(BondEntry),
                     cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  *e = *hb;
  return MPS_OK;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// write `len` floats (lambda) for bond b into a fresh pool block
mps_status put_lambda(mps_t h, int bond, const float* lam, int len, bool ones) {
  int64_t off;
  int cls;
  mps_status st = dev_alloc(h, (uint64_t)len * 4, &off, &cls);
  if (st != MPS_OK) return st;
  BondEntry old;
  st = read_bond(h, bond, &old);
  if (st != MPS_OK) return st;
  float* hb = static_cast<float*>(pinned_buf(h, (size_t)len * 4 + sizeof(BondEntry) + 64));
  for (int x = 0; x < len; ++x) hb[x] = ones ? 1.f : lam[x];
  BondEntry* ne = reinterpret_cast<BondEntry*>(reinterpret_cast<uint8_t*>(hb) + align_up((size_t)len * 4, 16));
  ne->off = off;
  ne->len = len;
  ne->cls = cls;
  CK(cudaMemcpyAsync(h->slab + off, hb, (size_t)len * 4, cudaMemcpyHostToDevice, h->s));
  CK(cudaMemcpyAsync(h->slab + h->hstate.bonds_off + sizeof(BondEntry) * (bond + 1), ne, sizeof(BondEntry),
                     cudaMemcpyHostToDevice, h->s));
  if (old.off) {
    launch_pool_free(h->slab, h->dst, old.off, old.cls, h->s);
    ++h->launches;
  }
  CK(cudaStreamSynchronize(h->s));
  h->lamlen[bond + 1] = len;
  return MPS_OK;
}

// ---- one wave of a layer: the front half (a0 staging, a1 contract, a2+a3 SVD) is issued by
// wave_front; the back half (a4 select + ledger, a5 reabsorb, readback) by wave_back. Between the
// two the caller may replace the ledger (mps_ledger_set): the multi-rank token chain of §8(e).
// lane-group size of the small (reg 0) and medium (reg 2) Jacobi kernels: a power of two in
// [4, 32], from the rows (small_group(m)) and the CTA width (2048 / n resp. 1024 / n lanes per pair)
size_t large_scratch_bytes(const GateDesc& gd) {
  const size_t b = std::max(svd_tc_scratch_bytes(gd.n_pad), gd.jrows > 0 ? large_precond_scratch(gd.n) : (size_t)0);
  // the eigen route (128 < n <= 4096) and the FP64 spectrum of deep 256 < n <= 4096 Jacobi-route
  // gates (refine_large.cu) reuse the dead scratch
  return (refine_large_candidate(gd) || eig_route(gd)) ? std::max(b, refine_large_scratch(gd.m, gd.n)) : b;
}

int lane_group(int m, int n, int reg) {
  int cap = std::max(4, (reg == 0 ? 2048 : 1024) / std::max(n, 1));
  int p2 = 4;
  while (p2 * 2 <= cap && p2 < 32) p2 *= 2;
  return std::min(small_group(m), p2);
}

mps_status wave_front_impl(mps_t h);
mps_status wave_front(mps_t h) {
  NvtxScope nv("eamps:wave_front (a0 plan/stage, a1 contract, a2 SVD, a3 sort+tails)");
  const double t0 = h->hp.on ? HostProf::now() : 0.0;
  mps_status st = wave_front_impl(h);
  if (h->hp.on) {
    const double t1 = HostProf::now();
    if (h->hp.layers > 3) {            // the first layers allocate the pinned buffers
      h->hp.wplan += h->hp.mark - t0;
      h->hp.launch += t1 - h->hp.mark;
    }
  }
  return st;
}

mps_status wave_front_impl(mps_t h) {
  LayerJob& J = h->job;
  std::vector<LayerPlan>& plan = J.plan;
  const int G = J.G, d = h->d, d4 = J.d4;
  const int g0 = J.g0;
  const size_t top = h->slab_bytes - 4 * kAlign;  // the top 1 KB is scratch for small host ops
  const uint64_t bump = h->hstate.pool.bump;
  size_t fixed = 0, ws = 0, reserve = 0;
  int g1 = g0;
  while (g1 < G) {
    const int cnt = g1 - g0 + 1;
    size_t fx = align_up(sizeof(GateDesc) * cnt) + 4 * align_up(4 * (cnt + 1)) + 5 * align_up(4 * cnt) +
                align_up((size_t)cnt * d4 * 8) + align_up(sizeof(Record) * cnt) + align_up(32 * (size_t)cnt + 64 + 24576);
    size_t w2 = ws + plan[g1].ws, r2 = reserve + plan[g1].reserve;
    if (bump + r2 + fx + w2 + kAlign > top) break;
    fixed = fx;
    ws = w2;
    reserve = r2;
    ++g1;
  }
  if (g1 == g0) return set_err(h, MPS_E_NOMEM, "one gate's workspace does not fit the slab");
  const int Gw = g1 - g0;
  J.g1 = g1;
  J.Gw = Gw;
  // device addresses of the wave's staging block (just below `top`)
  const size_t base = align_up(top - fixed - ws - kAlign);
  size_t cur = base;
  auto take = [&](size_t bytes) {
    size_t o = cur;
    cur = align_up(cur + bytes);
    return o;
  };
  const size_t o_desc = take(sizeof(GateDesc) * Gw);
  const size_t o_cpre = take(4 * (Gw + 1));
  const size_t o_rpre = take(4 * (Gw + 1));
  const size_t o_gpre = take(4 * (Gw + 1));
  const size_t o_apre = take(4 * (Gw + 1));
  const size_t o_small = take(4 * Gw);
  const size_t o_large = take(4 * Gw);
  const size_t o_rsm = take(4 * Gw);
  const size_t o_eigl = take(4 * Gw);
  const size_t o_eigs = take(4 * Gw);
  const size_t o_us = take((size_t)Gw * d4 * 8);
  const size_t o_rec = take(sizeof(Record) * Gw);
  const size_t o_scr = take(32 * (size_t)Gw + 64 + 24576);
  const size_t staged_bytes = o_rec - base;  // desc .. us are uploaded
  std::vector<int32_t> cpre(Gw + 1, 0), small, large;
  std::vector<int32_t>& eigl = J.eigl;
  eigl.clear();
  std::vector<int32_t>& eigs = J.eigs;
  eigs.clear();
  J.rsm.clear();
  J.rsm_smem = 0;
  J.rpre.assign(Gw + 1, 0);
  J.gpre.assign(Gw + 1, 0);
  J.apre.assign(Gw + 1, 0);
  std::vector<int32_t>&rpre = J.rpre, &gpre = J.gpre, &apre = J.apre;
  J.hd.assign(Gw, GateDesc{});
  std::vector<GateDesc>& hd = J.hd;
  // small / medium buckets by lane-group size GT (one launch per bucket); `small` holds them
  // back to back, [bstart, bend) per bucket
  struct Bucket {
    int regime, gt, begin, end, threads, tile_rows, rpl;
    size_t smem, smem2;
  };
  std::vector<Bucket> buckets;
  size_t span = 0;                     // workspace bytes of the previous gate
  for (int x = 0; x < Gw; ++x) {
    LayerPlan& p = plan[g0 + x];
    if (x > 0) {   // same shape as the previous gate: the same workspace layout one span further
      const GateDesc& q = hd[x - 1];
      if (q.l == p.gd.l && q.mid == p.gd.mid && q.r == p.gd.r) {
        GateDesc gd = q;
        gd.site = p.gd.site;
        gd.u_index = x;
        const int64_t sp = (int64_t)span;
        gd.ws_theta += sp;
        gd.ws_thetap += sp;
        gd.ws_V += sp;
        gd.ws_sig2 += sp;
        gd.ws_T += sp;
        gd.ws_pi += sp;
        gd.ws_E += sp;
        if (gd.ws_log) gd.ws_log += sp;
        cur += span;
        hd[x] = gd;
        cpre[x + 1] = cpre[x] + p.ctiles;
        rpre[x + 1] = rpre[x] + p.rtiles;
        gpre[x + 1] = gpre[x] + p.gtiles;
        apre[x + 1] = apre[x] + p.atiles;
        if (gd.regime == 1) (gd.eig ? eigl : large).push_back(x);
        else if (gd.eig) eigs.push_back(x);
        if (!J.rsm.empty() && J.rsm.back() == x - 1) J.rsm.push_back(x);   // same shape as gate x - 1
        continue;
      }
    }
    const size_t cur0 = cur;
    GateDesc gd = p.gd;
    gd.u_index = x;
    const size_t mn = (size_t)gd.m * gd.n * 8, mnp = (size_t)std::max(gd.m, gd.jrows) * gd.n_pad * 8;   // B = L (jrows rows) reuses it
    gd.ws_theta = (int64_t)take(mnp);
    gd.ws_thetap = (int64_t)take(mn);
    gd.ws_V = (int64_t)take((size_t)gd.n_pad * gd.n_pad * 8);
    gd.ws_sig2 = (int64_t)take((size_t)gd.n_pad * 8);
    gd.ws_T = (int64_t)take((size_t)(gd.n_pad + 1) * 8);
    gd.ws_pi = (int64_t)take((size_t)gd.n_pad * 4);
    const size_t kmn = (size_t)std::min(gd.m, gd.n);
    // E (k x k, reabsorb); the large regime's polish also keeps shift | den (2 n_pad doubles) there
    gd.ws_E = (int64_t)take(std::max(kmn * kmn * 8, (gd.regime == 1 || gd.regime == 3) ? (size_t)16 * gd.n_pad : (size_t)0));
    gd.ws_log = gd.regime == 2   ? (int64_t)take((size_t)gd.log_sweeps * (gd.n - 1) * (gd.n / 2) * 16)
                : gd.regime == 1 ? (int64_t)take(large_scratch_bytes(gd))
                : (gd.regime == 3 && gd.eig) ? (int64_t)take(refine_large_scratch(gd.m, gd.n))
                : (gd.regime == 3 && gd.jrows > 0) ? (int64_t)take(large_precond_scratch(gd.n))
                : refine_scratch_bytes(gd.n) > 0 ? (int64_t)take(refine_scratch_bytes(gd.n))
                                 : 0;
    span = cur - cur0;
    hd[x] = gd;
    cpre[x + 1] = cpre[x] + p.ctiles;
    rpre[x + 1] = rpre[x] + p.rtiles;
    gpre[x + 1] = gpre[x] + p.gtiles;
    apre[x + 1] = apre[x] + p.atiles;
    if (gd.regime == 1) (gd.eig ? eigl : large).push_back(x);
    else if (gd.eig) eigs.push_back(x);
    if (reabsorb_small_fits(gd.m, gd.n)) {
      J.rsm.push_back(x);
      J.rsm_smem = std::max(J.rsm_smem, reabsorb_small_smem(gd.m, gd.n));
    }
  }
  // SVD buckets, one launch each; `small` holds their gates back to back, [begin, end) per bucket.
  //  QR regime (3): (GT, R) as chosen by svd_qr_fits, and packed (n = R GT, m even) or not, or the
  //    block-recursive ordering (n = 64, 128; its own lane groups, see svd_qr.cu);
  //  small (0) / medium (2): lane-group size GT, rows per lane R (R > 0 keeps a pair's rows in
  //    registers). Each gate's key is computed once; the map keeps the launch order by key.
  {
    auto gidx = [](int gt) { return gt == 4 ? 0 : gt == 8 ? 1 : gt == 16 ? 2 : 3; };
    auto ridx = [](int r) { return r == 1 ? 0 : r == 2 ? 1 : r == 4 ? 2 : r == 8 ? 3 : r == 16 ? 4 : 5; };
    // key = ((class * 4 + gt) * 6 + rpl) * 3 + pk; a handful of keys per layer: a small vector
    // (launch order = ascending key), and the key of a gate with the previous gate's shape is reused
    std::vector<std::pair<int, std::vector<int32_t>>> keyed;
    std::vector<std::pair<int, std::array<int, 4>>> kparm;     // regime, gt, rpl, pk
    int last_m = -1, last_n = -1, last_reg = -1, last_slot = -1;
    for (int x = 0; x < Gw; ++x) {
      const GateDesc& gd = hd[x];
      int reg = gd.regime, gt = 0, rpl = 0, pk = 0, cls = 0;
      if (reg == 1 || gd.eig) continue;   // large regime / eigen route: not bucketed
      if (gd.m == last_m && gd.n == last_n && reg == last_reg) {
        keyed[last_slot].second.push_back(x);
        continue;
      }
      if (reg == 3) {
        if (!svd_qr_fits(gd.m, gd.n, &gt, &rpl)) return set_err(h, MPS_E_STATE, "internal: QR regime without a QR fit");
        pk = qr_block_order(gd.m, gd.n) ? 2 : (gd.n == rpl * gt && gd.m % 2 == 0 && rpl >= 2) ? 1 : 0;
        cls = 0;
      } else {
        gt = lane_group(gd.m, gd.n, reg);
        const int rm = rows_per_lane(gd.m, gt), rn = rows_per_lane(gd.n, gt);
        rpl = (rm == 0 || rn == 0) ? 0 : std::max(rm, rn);
        cls = reg == 0 ? 1 : 2;
      }
      const int key = ((cls * 4 + gidx(gt)) * 6 + ridx(rpl)) * 3 + pk;
      int slot = 0;
      while (slot < (int)keyed.size() && keyed[slot].first != key) ++slot;
      if (slot == (int)keyed.size()) {
        keyed.push_back({key, {}});
        kparm.push_back({key, {reg, gt, rpl, pk}});
      }
      keyed[slot].second.push_back(x);
      last_m = gd.m;
      last_n = gd.n;
      last_reg = reg;
      last_slot = slot;
    }
    std::vector<int> korder(keyed.size());
    for (size_t i = 0; i < korder.size(); ++i) korder[i] = (int)i;
    std::sort(korder.begin(), korder.end(), [&](int a, int b) { return keyed[a].first < keyed[b].first; });
    for (int ki : korder) {
      auto& kv = keyed[ki];
      const std::array<int, 4>& pr = kparm[ki].second;
      const int reg = pr[0], gt = pr[1], rpl = pr[2];
      if (reg == 3) {
        Bucket b{3, gt, (int)small.size(), 0, 512, pr[3], rpl, 0, 0};   // (tile_rows carries the packed flag)
        int pm = -1, pn = -1;
        for (int x : kv.second) {
          small.push_back(x);
          if (hd[x].m == pm && hd[x].n == pn) continue;
          pm = hd[x].m;
          pn = hd[x].n;
          b.smem = std::max(b.smem, svd_qr_smem(pm, pn));
        }
        b.end = (int)small.size();
        buckets.push_back(b);
        continue;
      }
      Bucket b{reg, gt, (int)small.size(), 0, 64, 64, rpl, 0, 0};
      int maxn = 2, pm = -1, pn = -1;
      for (int x : kv.second) {
        const GateDesc& gd = hd[x];
        small.push_back(x);
        if (gd.m == pm && gd.n == pn) continue;
        pm = gd.m;
        pn = gd.n;
        maxn = std::max(maxn, gd.n);
        if (reg == 0) {
          b.smem = std::max(b.smem, svd_small_smem(gd.m, gd.n));
        } else {
          const int tr = vrep_tile_rows(gd.m, gd.n);
          b.tile_rows = std::min(b.tile_rows, tr);
          b.smem = std::max(b.smem, svd_theta_smem(gd.m, gd.n));
        }
      }
      b.end = (int)small.size();
      if (reg == 2) {
        int qn = -1;
        for (int i = b.begin; i < b.end; ++i) {
          if (hd[small[i]].n == qn) continue;
          qn = hd[small[i]].n;
          b.smem2 = std::max(b.smem2, svd_vrep_smem(qn, b.tile_rows));
        }
      }
      b.threads = (int)std::min<size_t>(reg == 0 ? 1024 : 512, std::max<size_t>(64, align_up((size_t)(maxn / 2) * gt, 32)));
      buckets.push_back(b);
    }
  }
  if (cur > top) return set_err(h, MPS_E_NOMEM, "workspace planning overflow");
  {   // every gate of the small / medium / QR regimes must sit in exactly one bucket
    size_t want = 0;
    for (int x = 0; x < Gw; ++x) want += hd[x].regime != 1 && !hd[x].eig;
    if (want != small.size()) return set_err(h, MPS_E_STATE, "internal: SVD bucketing lost a gate");
  }
  // stage desc | prefixes | lists | gates in one pinned buffer, one H2D copy
  const size_t tail = align_up(staged_bytes, 64);  // 3 small pinned slots after the staged block
  uint8_t* hb = static_cast<uint8_t*>(pinned_buf(h, tail + 256 + 4 * (size_t)Gw, 1));   // + eigen-route fallback flags
  if (!hb) return set_err(h, MPS_E_NOMEM, "pinned host allocation failed");
  J.tail = tail;
  std::memcpy(hb + (o_desc - base), hd.data(), sizeof(GateDesc) * Gw);
  std::memcpy(hb + (o_cpre - base), cpre.data(), 4 * (Gw + 1));
  std::memcpy(hb + (o_rpre - base), rpre.data(), 4 * (Gw + 1));
  std::memcpy(hb + (o_gpre - base), gpre.data(), 4 * (Gw + 1));
  std::memcpy(hb + (o_apre - base), apre.data(), 4 * (Gw + 1));
  if (!small.empty()) std::memcpy(hb + (o_small - base), small.data(), 4 * small.size());
  if (!large.empty()) std::memcpy(hb + (o_large - base), large.data(), 4 * large.size());
  if (!eigl.empty()) std::memcpy(hb + (o_eigl - base), eigl.data(), 4 * eigl.size());
  J.o_eigl = o_eigl;
  if (!eigs.empty()) std::memcpy(hb + (o_eigs - base), eigs.data(), 4 * eigs.size());
  J.o_eigs = o_eigs;
  if (!J.rsm.empty()) std::memcpy(hb + (o_rsm - base), J.rsm.data(), 4 * J.rsm.size());
  J.o_rsm = o_rsm;
  for (int x = 0; x < Gw; ++x)
    std::memcpy(hb + (o_us - base) + (size_t)x * d4 * 8, J.us.data() + (size_t)J.ord[g0 + x].second * d4 * 2,
                (size_t)d4 * 8);
  if (h->hp.on) h->hp.mark = HostProf::now();
  CK(h2d_small(h, h->slab + base, hb, staged_bytes));
  // the pool may not grow into the workspace
  uint64_t* hceil = reinterpret_cast<uint64_t*>(hb + tail);
  *hceil = base;
  CK(h2d_small(h, &h->dst->pool.ceiling, hceil, 8));

  GateDesc* d_desc = reinterpret_cast<GateDesc*>(h->slab + o_desc);
  J.o_desc = o_desc;
  J.o_rec = o_rec;
  J.o_gpre = o_gpre;
  J.o_apre = o_apre;
  J.o_rpre = o_rpre;
  const int32_t* d_cpre = reinterpret_cast<const int32_t*>(h->slab + o_cpre);
  const int32_t* d_small = reinterpret_cast<const int32_t*>(h->slab + o_small);
  const int32_t* d_large = reinterpret_cast<const int32_t*>(h->slab + o_large);
  const float2* d_us = reinterpret_cast<const float2*>(h->slab + o_us);

  const bool prof = h->profiling;
  J.ran[0] = true;
  J.ran[1] = !buckets.empty();
  J.ran[2] = !large.empty();
  J.ran[3] = J.ran[4] = true;
  if (prof) CK(cudaEventRecord(h->ev[0], h->s));
  // a1 contract (all gates of the wave)
  launch_contract(d_desc, d_cpre, Gw, cpre[Gw], d, h->slab, h->dst, d_us, h->s);
  ++h->launches;
  CKL("contract");
  if (prof) CK(cudaEventRecord(h->ev[1], h->s));
  // a2 + a3 SVD, small regime: one CTA per theta
  for (const Bucket& b : buckets) {
    if (b.regime == 3) {
      int maxn = 0;
      bool pc = false;
      for (int i = b.begin; i < b.end; ++i) {
        maxn = std::max(maxn, hd[small[i]].n);
        pc |= hd[small[i]].jrows > 0;
      }
      // Cholesky preconditioner (FP64 Gram + Cholesky -> B = L in the theta workspace) instead of
      // the in-CTA FP32 Householder QR
      const int e0 = prof ? prof_mark(h) : -1;
      if (pc) h->launches += launch_precond_large(d_desc, d_small + b.begin, b.end - b.begin, maxn, h->slab, h->s);
      const int e1 = prof ? prof_mark(h) : -1;
      launch_svd_qr(d_desc, d_small + b.begin, b.end - b.begin, b.smem, h->cfg.max_sweeps, b.gt, b.rpl, b.tile_rows,
                    h->slab, h->dst, h->s);
      const int e2 = prof ? prof_mark(h) : -1;
      h->launches += 1 + launch_spectrum_polish(d_desc, d_small + b.begin, b.end - b.begin, maxn, h->slab, h->dst, h->s);
      if (prof) {
        const int e3 = prof_mark(h);
        if (pc) prof_span(h, 5, e0, e1);
        prof_span(h, 6, e1, e2);
        prof_span(h, 7, e2, e3);
      }
    } else if (b.regime == 0) {
      launch_svd_small(d_desc, d_small + b.begin, b.end - b.begin, b.smem, h->cfg.max_sweeps, b.gt, b.rpl, b.threads,
                       h->slab, h->dst, h->s);
      ++h->launches;
    } else {
      launch_svd_medium(d_desc, d_small + b.begin, b.end - b.begin, b.smem, b.smem2, b.tile_rows, h->cfg.max_sweeps,
                        b.gt, b.rpl, b.threads, h->slab, h->dst, h->s);
      h->launches += 2;
    }
    CKL("svd_small/medium");
  }
  // a2 + a3, the eigen route for QR-regime thetas (n <= 128): one CTA per gate; a spectrum deeper than
  // 2e-4 sigma_max gets all its eigenvectors now and the FP64 Rayleigh-Ritz refinement below
  if (!eigs.empty()) {
    const int32_t* d_eigs = reinterpret_cast<const int32_t*>(h->slab + o_eigs);
    const int e0 = prof ? prof_mark(h) : -1;
    RlgMarks mk{[](void* c) { return prof_mark(static_cast<mps_t>(c)); }, h, {-1, -1}};
    h->launches += launch_eig_small_front(d_desc, hd.data(), eigs.data(), d_eigs, (int)eigs.size(), h->slab, h->dst,
                                          d_us, d, reinterpret_cast<int32_t*>(h->slab + o_scr) + Gw + 2, h->s,
                                          prof ? &mk : nullptr);
    CKL("eig_small_front");
    h->launches += launch_eig_vectors(d_desc, hd.data(), eigs.data(), d_eigs, (int)eigs.size(), h->slab, h->s, 2);
    CKL("eig_small_vectors_deep");
    if (prof && mk.at[0] >= 0) {   // [8] the one-CTA eigensolver, [9] the rest
      const int e1 = prof_mark(h);
      prof_span(h, 9, e0, mk.at[0]);
      prof_span(h, 8, mk.at[0], mk.at[1]);
      prof_span(h, 9, mk.at[1], e1);
    }
  }
  if (prof) CK(cudaEventRecord(h->ev[2], h->s));
  // a2 + a3, the eigen route (large regime, 128 < n <= 4096): sigma^2 = eigenvalues of the FP64 Gram
  // of the FP64-recontracted theta (refine_large.cu); a spectrum too deep for it (flag read back
  // here) goes to the Jacobi route below
  if (!eigl.empty()) {
    const int32_t* d_eigl = reinterpret_cast<const int32_t*>(h->slab + o_eigl);
    int32_t* fbd = reinterpret_cast<int32_t*>(h->slab + o_scr) + 4 * Gw + 5000;   // after the refine lists and barrier lines
    const int e0 = prof ? prof_mark(h) : -1;
    RlgMarks mk{[](void* c) { return prof_mark(static_cast<mps_t>(c)); }, h, {-1, -1}};
    h->launches += launch_eig_front(d_desc, hd.data(), eigl.data(), d_eigl, (int)eigl.size(), h->slab, h->dst, d_us, d,
                                    reinterpret_cast<int32_t*>(h->slab + o_scr) + Gw + 2, fbd, h->s, prof ? &mk : nullptr);
    CKL("eig_front");
    if (prof && mk.at[0] >= 0) {   // [8] the tridiagonalisation, [9] the rest of the eigen route
      const int e1 = prof_mark(h);
      prof_span(h, 9, e0, mk.at[0]);
      prof_span(h, 8, mk.at[0], mk.at[1]);
      prof_span(h, 9, mk.at[1], e1);
    }
    int32_t* fbh = reinterpret_cast<int32_t*>(hb + tail + 256);
    CK(cudaMemcpyAsync(fbh, fbd, 4 * eigl.size(), cudaMemcpyDeviceToHost, h->s));
    CK(cudaStreamSynchronize(h->s));
    bool moved = false;
    for (size_t c = 0; c < eigl.size(); ++c)
      if (fbh[c]) {
        hd[eigl[c]].eig = 0;
        large.push_back(eigl[c]);
        moved = true;
      }
    if (moved) {
      std::memcpy(hb + (o_large - base), large.data(), 4 * large.size());
      CK(h2d_small(h, h->slab + o_large, hb + (o_large - base), 4 * large.size()));
    }
  }
  // a2 + a3 SVD, large regime: blocked Jacobi
  if (!large.empty()) {
    int err = 0;
    int32_t* hflag = reinterpret_cast<int32_t*>(hb + tail + 64);
    static const bool simt = getenv("EAMPS_LARGE_SIMT") != nullptr;   // dev A/B switch: SIMT blocked path
    h->launches += (simt ? run_svd_blocked : run_svd_tc)(d_desc, hd.data(), d_large, large.data(), (int)large.size(),
                                                         h->cfg.max_sweeps, h->slab, h->dst,
                                                         reinterpret_cast<int32_t*>(h->slab + o_scr), hflag, h->s, &err);
    CKL("svd_blocked");
    if (err) {
      // record on device so that it is sticky like the small-path error
      int32_t* he = reinterpret_cast<int32_t*>(hb + tail + 128);
      *he = err;
      CK(h2d_small(h, &h->dst->led.error, he, 4));
    }
  }
  // FP64 Rayleigh-Ritz refinement of deep spectra (refine.cu; gates with n <= 256)
  {
    int maxn = 0;
    for (int x = 0; x < Gw; ++x) maxn = std::max(maxn, hd[x].n);
    static const bool no_refine = getenv("EAMPS_NO_REFINE") != nullptr;   // dev A/B switch
    if (!no_refine) {
      const int e0 = prof ? prof_mark(h) : -1;
      h->launches += launch_refine(d_desc, Gw, maxn, h->slab, h->dst, d_us, reinterpret_cast<int32_t*>(h->slab + o_scr), h->s);
      CKL("refine");
      // deep large-regime gates with 256 < n <= 4096: FP64 eigenvalues of the recontracted Gram
      if (!large.empty()) {
        h->launches += launch_refine_large(d_desc, hd.data(), large.data(), d_large, (int)large.size(), h->slab, h->dst,
                                           d_us, d, reinterpret_cast<int32_t*>(h->slab + o_scr) + Gw + 2, h->s);
        CKL("refine_large");
      }
      if (prof) prof_span(h, 7, e0, prof_mark(h));
    }
  }
  if (prof) CK(cudaEventRecord(h->ev[3], h->s));
  J.front = true;
  return MPS_OK;
}

mps_status wave_back(mps_t h) {
  NvtxScope nv("eamps:wave_back (a4 select+ledger, a5 reabsorb)");
  LayerJob& J = h->job;
  if (!J.front) return set_err(h, MPS_E_STATE, "no wave in flight");
  J.front = false;
  const int Gw = J.Gw;
  std::vector<GateDesc>& hd = J.hd;
  GateDesc* d_desc = reinterpret_cast<GateDesc*>(h->slab + J.o_desc);
  Record* d_rec = reinterpret_cast<Record*>(h->slab + J.o_rec);
  const int32_t* d_gpre = reinterpret_cast<const int32_t*>(h->slab + J.o_gpre);
  const int32_t* d_apre = reinterpret_cast<const int32_t*>(h->slab + J.o_apre);
  const int32_t* d_rpre = reinterpret_cast<const int32_t*>(h->slab + J.o_rpre);
  const bool prof = h->profiling;
  // a4 select + ledger + pool
  const int par = (h->cfg.strategy == MPS_STRAT_FIXED || h->cfg.strategy == MPS_STRAT_NAIVE) ? 1 : 0;
  launch_select(d_desc, Gw, h->slab, h->dst, d_rec, par, h->s);
  h->launches += 2;
  CKL("select");
  // the eigen route's right singular vectors, for the kept k only
  if (!J.eigl.empty()) {
    const int e0 = prof ? prof_mark(h) : -1;
    h->launches += launch_eig_vectors(d_desc, hd.data(), J.eigl.data(),
                                      reinterpret_cast<const int32_t*>(h->slab + J.o_eigl), (int)J.eigl.size(),
                                      h->slab, h->s, 1);
    CKL("eig_vectors");
    if (prof) prof_span(h, 9, e0, prof_mark(h));
  }
  if (!J.eigs.empty()) {
    const int e0 = prof ? prof_mark(h) : -1;
    h->launches += launch_eig_vectors(d_desc, hd.data(), J.eigs.data(),
                                      reinterpret_cast<const int32_t*>(h->slab + J.o_eigs), (int)J.eigs.size(),
                                      h->slab, h->s, 1);
    CKL("eig_small_vectors");
    if (prof) prof_span(h, 9, e0, prof_mark(h));
  }
  if (prof) CK(cudaEventRecord(h->ev[4], h->s));
  // a5 reabsorb
  h->launches += launch_reabsorb(d_desc, d_gpre, J.gpre[Gw], d_apre, J.apre[Gw], d_rpre, J.rpre[Gw], Gw, h->slab, h->s);
  launch_reabsorb_small(d_desc, reinterpret_cast<const int32_t*>(h->slab + J.o_rsm), (int)J.rsm.size(), J.rsm_smem,
                        h->slab, h->s);
  if (!J.rsm.empty()) ++h->launches;
  CKL("reabsorb");
  if (prof) CK(cudaEventRecord(h->ev[5], h->s));
  // read back: descriptors (k, sweeps), records, device state
  const size_t back = sizeof(GateDesc) * Gw + sizeof(Record) * Gw + sizeof(DevState);
  uint8_t* rb = static_cast<uint8_t*>(pinned_buf(h, back + 64));
  CK(cudaMemcpyAsync(rb, d_desc, sizeof(GateDesc) * Gw, cudaMemcpyDeviceToHost, h->s));
  CK(cudaMemcpyAsync(rb + sizeof(GateDesc) * Gw, d_rec, sizeof(Record) * Gw, cudaMemcpyDeviceToHost, h->s));
  CK(cudaMemcpyAsync(rb + sizeof(GateDesc) * Gw + sizeof(Record) * Gw, h->dst, sizeof(DevState),
                     cudaMemcpyDeviceToHost, h->s));
  const double hw0 = h->hp.on ? HostProf::now() : 0.0;
  CK(cudaStreamSynchronize(h->s));
  const double hw1 = h->hp.on ? HostProf::now() : 0.0;
  if (h->hp.on && h->hp.layers > 3) h->hp.wait += hw1 - hw0;
  std::memcpy(hd.data(), rb, sizeof(GateDesc) * Gw);
  const Record* rr = reinterpret_cast<const Record*>(rb + sizeof(GateDesc) * Gw);
  std::memcpy(&h->hstate, rb + sizeof(GateDesc) * Gw + sizeof(Record) * Gw, sizeof(DevState));
  if (prof) {
    for (int p = 0; p < 5; ++p) {
      if (!J.ran[p]) continue;
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, h->ev[p], h->ev[p + 1]));
      h->phase_ms[p] += ms;
      h->phase_n[p] += 1;
    }
    for (const auto& sp : h->spans) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, h->span_ev[sp[1]], h->span_ev[sp[2]]));
      h->phase_ms[sp[0]] += ms;
      h->phase_n[sp[0]] += 1;
    }
  }
  h->spans.clear();
  h->span_used = 0;
  mps_status de = device_error(h);
  for (int x = 0; x < Gw; ++x) {
    const GateDesc& gd = hd[x];
    if (gd.k <= 0) continue;
    h->chr[gd.site] = gd.k;
    h->chl[gd.site + 1] = gd.k;
    h->lamlen[gd.site + 1] = gd.k;
    mps_record rec;
    std::memcpy(&rec, &rr[x], sizeof(rec));
    h->records.push_back(rec);
  }
  if (h->keep_spectra && de == MPS_OK) {
    // parity export of multi-wave layers: this wave's workspace is reused by the next front
    h->spectra.resize(h->last_desc.size());
    for (int x = 0; x < Gw; ++x) {
      h->spectra.emplace_back((size_t)std::max(hd[x].n, 0));
      if (hd[x].n > 0)
        CK(cudaMemcpyAsync(h->spectra.back().data(), h->slab + hd[x].ws_sig2, 8 * (size_t)hd[x].n,
                           cudaMemcpyDeviceToHost, h->s));
    }
    CK(cudaStreamSynchronize(h->s));
  }
  h->last_wave_begin = (int)h->last_desc.size();
  h->last_desc.insert(h->last_desc.end(), hd.begin(), hd.end());
  if (h->hp.on && h->hp.layers > 3) h->hp.post += HostProf::now() - hw1;
  if (de != MPS_OK) return de;
  J.g0 = J.g1;
  return MPS_OK;
}

}  // namespace

extern "C" {

const char* mps_status_string(mps_status s) { return status_name(s); }

const char* mps_last_error(mps_t h) { return h ? h->err.c_str() : "null handle"; }

mps_status mps_create(int32_t n_sites, int32_t d, const mps_config* cfg, mps_t* out) {
  if (!out || !cfg) return MPS_E_INVAL;
  *out = nullptr;
  if (n_sites < 2 || (d != 2 && d != 4)) return MPS_E_INVAL;
  if (!(cfg->f_min > 0.0 && cfg->f_min <= 1.0)) return MPS_E_INVAL;
  if (cfg->strategy < 0 || cfg->strategy > 3 || cfg->rule < 0 || cfg->rule > 2) return MPS_E_INVAL;
  if (cfg->strategy == MPS_STRAT_FIXED && !(cfg->f_fixed > 0.0 && cfg->f_fixed <= 1.0)) return MPS_E_INVAL;
  if (!cfg->dev_slab || cfg->slab_bytes < (1u << 20)) return MPS_E_INVAL;
  int slab_dev = -1;
  {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, cfg->dev_slab) != cudaSuccess || a.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      return MPS_E_INVAL;   // the slab must be device memory
    }
    slab_dev = a.device;
  }
  mps_t h = new mps_handle();
  h->device = slab_dev;
  DEVICE_GUARD(h);
  h->N = n_sites;
  h->d = d;
  h->cfg = *cfg;
  if (h->cfg.max_sweeps <= 0) h->cfg.max_sweeps = 60;
  h->s = static_cast<cudaStream_t>(cfg->stream);
  h->slab = static_cast<uint8_t*>(cfg->dev_slab);
  h->slab_bytes = cfg->slab_bytes;
  h->dst = reinterpret_cast<DevState*>(h->slab);
  h->chl.assign(n_sites, 1);
  h->chr.assign(n_sites, 1);
  h->lamlen.assign(n_sites + 1, 1);

  // slab layout: DevState | SiteEntry[N] | BondEntry[N+1] | pending frees | pool ...
  const size_t sites_off = align_up(sizeof(DevState));
  const size_t bonds_off = align_up(sites_off + sizeof(SiteEntry) * n_sites);
  const int64_t pend_cap = 3 * (int64_t)n_sites + 64;
  const size_t pend_off = align_up(bonds_off + sizeof(BondEntry) * (n_sites + 1));
  // Free-stack capacity per size class. A class's population only grows when an allocation finds
  // its stack empty, i.e. when population = live + pending (<= (2N+1) + 1.5N, the frees are
  // deferred one commit), plus that commit's allocations (<= 1.5N): population <= 5N + 2. (3N + 64
  // overflowed on config 5 at layer 10: the deferred frees of the first layer double the
  // population of the smallest class.)
  const int64_t stack_cap = 6 * (int64_t)n_sites + 256;
  const size_t stack_off = align_up(pend_off + 16 * pend_cap);
  const size_t pool_base = align_up(stack_off + 8 * (size_t)kMaxClasses * stack_cap);
  const size_t init_end = pool_base + kAlign * (2 * (size_t)n_sites + 1);
  if (init_end + (1u << 16) > h->slab_bytes) {
    delete h;
    return MPS_E_NOMEM;
  }
  h->pool_base = pool_base;
  std::vector<uint8_t> img(init_end, 0);
  DevState& S = *reinterpret_cast<DevState*>(img.data());
  S.led.logE = 0.0;
  S.led.j = 0;
  S.led.guarantee = 1;
  S.led.error = 0;
  S.led.log_fmin = std::log(cfg->f_min);
  S.led.log_ffixed = cfg->strategy == MPS_STRAT_FIXED ? std::log(cfg->f_fixed) : 0.0;
  S.led.n_planned = cfg->n_planned;
  S.led.strategy = cfg->strategy;
  S.led.rule = cfg->rule;
  S.led.chi_cap = cfg->chi_cap;
  S.led.d = d;
  S.pool.bump = init_end;
  S.pool.ceiling = h->slab_bytes - kAlign;
  S.pool.npending = 0;
  S.pool.stack_off = (int64_t)stack_off;
  S.pool.stack_cap = stack_cap;
  S.pool.pending_cap = pend_cap;
  S.pool.pending_off = (int64_t)pend_off;
  S.n_sites = n_sites;
  S.d = d;
  S.sites_off = (int64_t)sites_off;
  S.bonds_off = (int64_t)bonds_off;
  SiteEntry* se = reinterpret_cast<SiteEntry*>(img.data() + sites_off);
  BondEntry* be = reinterpret_cast<BondEntry*>(img.data() + bonds_off);
  // |0...0>: B_i[0,0,0] = 1 (MPO: s = 2 sigma + sigma' = 0), lambda = [1]
  for (int i = 0; i < n_sites; ++i) {
    size_t off = pool_base + kAlign * i;
    se[i].off = (int64_t)off;
    se[i].chl = se[i].chr = 1;
    se[i].cls = kMinClass;
    reinterpret_cast<float*>(img.data() + off)[0] = 1.f;
  }
  for (int b = 0; b <= n_sites; ++b) {
    size_t off = pool_base + kAlign * (n_sites + b);
    be[b].off = (int64_t)off;
    be[b].len = 1;
    be[b].cls = kMinClass;
    reinterpret_cast<float*>(img.data() + off)[0] = 1.f;
  }
  void* pb = pinned_buf(h, img.size());
  if (!pb) {
    delete h;
    return MPS_E_NOMEM;
  }
  std::memcpy(pb, img.data(), img.size());
  if (cudaMemcpyAsync(h->slab, pb, img.size(), cudaMemcpyHostToDevice, h->s) != cudaSuccess ||
      cudaStreamSynchronize(h->s) != cudaSuccess) {
    cudaFreeHost(h->pinned[0]);
    delete h;
    return MPS_E_CUDA;
  }
  h->hstate = S;
  *out = h;
  return MPS_OK;
}

mps_status mps_destroy(mps_t h) {
  DEVICE_GUARD(h);
  if (!h) return MPS_E_INVAL;
  if (h->s) cudaStreamSynchronize(h->s);
  if (h->hp.on && h->hp.layers > 3)
    fprintf(stderr, "[eamps host] %lld layers, ms per layer: plan %.3f wave-plan %.3f launch %.3f wait %.3f post %.3f\n",
            (long long)h->hp.layers - 3, h->hp.plan / (h->hp.layers - 3), h->hp.wplan / (h->hp.layers - 3),
            h->hp.launch / (h->hp.layers - 3), h->hp.wait / (h->hp.layers - 3), h->hp.post / (h->hp.layers - 3));
  for (int w = 0; w < 2; ++w)
    if (h->pinned[w]) cudaFreeHost(h->pinned[w]);
  for (int e = 0; e < 6; ++e)
    if (h->ev[e]) cudaEventDestroy(h->ev[e]);
  for (cudaEvent_t e : h->span_ev) cudaEventDestroy(e);
  delete h;
  return MPS_OK;
}

mps_status mps_sync(mps_t h) {
  DEVICE_GUARD(h);
  if (!h) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  st = sync_state(h);
  if (st != MPS_OK) return st;
  return device_error(h);
}

mps_status mps_set_profiling(mps_t h, int32_t on) {
  DEVICE_GUARD(h);
  if (!h) return MPS_E_INVAL;
  if (on && !h->ev[0])
    for (int e = 0; e < 6; ++e) CK(cudaEventCreate(&h->ev[e]));
  h->profiling = on != 0;
  for (int p = 0; p < kPhases; ++p) { h->phase_ms[p] = 0; h->phase_n[p] = 0; }
  return MPS_OK;
}

mps_status mps_keep_spectra(mps_t h, int32_t on) {
  if (!h) return MPS_E_INVAL;
  if (h->job.active) return set_err(h, MPS_E_STATE, "mps_keep_spectra inside a layer");
  h->keep_spectra = on != 0;
  h->spectra.clear();
  return MPS_OK;
}

mps_status mps_set_svd_route(mps_t h, int32_t route) {
  if (!h || route < 0 || route > 1) return MPS_E_INVAL;
  if (h->job.active) return set_err(h, MPS_E_STATE, "mps_set_svd_route inside a layer");
  h->jacobi_only = route == 1;
  return MPS_OK;
}

mps_status mps_phase_times(mps_t h, double* ms, int64_t* counts) {
  if (!h || !ms) return MPS_E_INVAL;
  for (int p = 0; p < kPhases; ++p) {
    ms[p] = h->phase_ms[p];
    if (counts) counts[p] = h->phase_n[p];
  }
  return MPS_OK;
}

mps_status mps_launch_count(mps_t h, int64_t* c) {
  if (!h || !c) return MPS_E_INVAL;
  *c = h->launches;
  return MPS_OK;
}

mps_status mps_apply_gate1(mps_t h, int32_t site, const float* U) {
  DEVICE_GUARD(h);
  if (!h || !U) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  if (site < 0 || site >= h->N) return set_err(h, MPS_E_RANGE, "site out of range");
  const int dd = h->d * h->d;
  for (int x = 0; x < 2 * dd; ++x)
    if (!std::isfinite(U[x])) return set_err(h, MPS_E_INVAL, "non-finite gate entry");
  float* hb = static_cast<float*>(pinned_buf(h, 8 * dd));
  std::memcpy(hb, U, 8 * dd);
  float2* du = reinterpret_cast<float2*>(h->slab + h->slab_bytes - 2 * kAlign);  // 2 KB scratch below the top
  CK(h2d_small(h, du, hb, 8 * dd));
  launch_gate1(h->slab, h->dst, site, h->d, du, h->s);
  ++h->launches;
  CKL("gate1");
  CK(cudaStreamSynchronize(h->s));
  return MPS_OK;
}

mps_status mps_apply_layer1(mps_t h, int32_t G, const int32_t* sites, const float* Us) {
  DEVICE_GUARD(h);
  if (!h) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  if (G < 0 || (G > 0 && (!sites || !Us))) return set_err(h, MPS_E_INVAL, "bad arguments");
  if (h->job.active) return set_err(h, MPS_E_STATE, "a layer is still in progress (mps_layer_step)");
  if (G == 0) return MPS_OK;
  const int dd = h->d * h->d;
  std::vector<char> seen(h->N, 0);
  for (int g = 0; g < G; ++g) {
    if (sites[g] < 0 || sites[g] >= h->N) return set_err(h, MPS_E_RANGE, "gate site out of range");
    if (seen[sites[g]]) return set_err(h, MPS_E_INVAL, "two single-site gates on one site in a layer");
    seen[sites[g]] = 1;
  }
  for (int64_t x = 0; x < (int64_t)G * dd * 2; ++x)
    if (!std::isfinite(Us[x])) return set_err(h, MPS_E_INVAL, "non-finite gate entry");
  st = sync_state(h);
  if (st != MPS_OK) return st;
  const size_t sb = align_up((size_t)G * 4), ub = (size_t)G * dd * 8;
  const size_t need = align_up(sb + ub) + kAlign;
  if (h->hstate.pool.bump + need + 4 * kAlign > h->slab_bytes) return set_err(h, MPS_E_NOMEM, "no room for the layer");
  const size_t base = align_up(h->slab_bytes - 4 * kAlign - need);
  uint8_t* hb = static_cast<uint8_t*>(pinned_buf(h, sb + ub, 1));
  if (!hb) return set_err(h, MPS_E_NOMEM, "pinned host allocation failed");
  std::memcpy(hb, sites, 4 * (size_t)G);
  std::memcpy(hb + sb, Us, ub);
  CK(h2d_small(h, h->slab + base, hb, sb + ub));
  launch_gate1_layer(h->slab, h->dst, G, reinterpret_cast<const int32_t*>(h->slab + base),
                     reinterpret_cast<const float2*>(h->slab + base + sb), h->d, h->s);
  ++h->launches;
  CKL("gate1_layer");
  CK(cudaStreamSynchronize(h->s));   // the pinned staging buffer is reused by the next call
  return MPS_OK;
}

mps_status mps_layer_begin(mps_t h, int32_t G, const int32_t* sites, const float* Us, int32_t* n_waves) {
  DEVICE_GUARD(h);
  if (n_waves) *n_waves = 0;
  if (!h) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  if (G < 0 || (G > 0 && (!sites || !Us))) return set_err(h, MPS_E_INVAL, "bad arguments");
  if (h->job.active) return set_err(h, MPS_E_STATE, "a layer is still in progress (mps_layer_step)");
  if (G == 0) return MPS_OK;
  const double hp0 = h->hp.on ? HostProf::now() : 0.0;
  if (h->hp.on) ++h->hp.layers;
  const int d = h->d, d4 = d * d * d * d;
  // ---- a0: validate (in range, disjoint pairs), canonical order = ascending site
  std::vector<std::pair<int, int>> ord(G);
  for (int g = 0; g < G; ++g) {
    if (sites[g] < 0 || sites[g] >= h->N - 1) return set_err(h, MPS_E_RANGE, "gate site out of range");
    ord[g] = {sites[g], g};
  }
  if (!std::is_sorted(ord.begin(), ord.end())) std::sort(ord.begin(), ord.end());
  for (int g = 1; g < G; ++g)
    if (ord[g].first < ord[g - 1].first + 2) return set_err(h, MPS_E_INVAL, "overlapping gates in a layer");
  {   // non-finite entries: exponent bits all ones (branch-free OR over the layer, vectorisable)
    const uint32_t* ub = reinterpret_cast<const uint32_t*>(Us);
    uint32_t bad = 0;
    const int64_t ne = (int64_t)G * d4 * 2;
    for (int64_t x = 0; x < ne; ++x) bad |= (uint32_t)((ub[x] & 0x7f800000u) == 0x7f800000u);
    if (bad) return set_err(h, MPS_E_INVAL, "non-finite gate entry");
  }
  if (h->cfg.strategy != MPS_STRAT_FIXED && h->hstate.led.j + G > h->cfg.n_planned)
    return set_err(h, MPS_E_STATE, "more truncations than n_planned");
  for (int g = 0; g < G; ++g) {
    int i = ord[g].first;
    if (h->chr[i] != h->chl[i + 1] || h->lamlen[i] != h->chl[i])
      return set_err(h, MPS_E_INVAL, "inconsistent bond extents at the gate");
  }

  // ---- per-gate shapes, regimes and workspace sizes
  LayerJob& J = h->job;
  J.plan.assign(G, LayerPlan{});
  std::vector<LayerPlan>& plan = J.plan;
  const int TA = 64 / d;
  for (int g = 0; g < G; ++g) {
    LayerPlan& p = plan[g];
    GateDesc& gd = p.gd;
    const int i = ord[g].first;
    if (g > 0) {   // the plan depends on the gate's shape only: reuse the previous gate's when equal
      const GateDesc& q = plan[g - 1].gd;
      if (q.l == h->chl[i] && q.mid == h->chr[i] && q.r == h->chr[i + 1]) {
        p = plan[g - 1];
        gd.site = i;
        gd.u_index = ord[g].second;
        continue;
      }
    }
    std::memset(&gd, 0, sizeof(gd));
    gd.site = i;
    gd.l = h->chl[i];
    gd.mid = h->chr[i];
    gd.r = h->chr[i + 1];
    gd.m = gd.l * d;
    gd.n = d * gd.r;
    // SVD regime: 0 small (theta + V in one CTA), 2 medium (theta in one CTA, V replayed from a
    // rotation log), 1 large (blocked, HBM-resident)
    // SVD regime: 3 QR-preconditioned Jacobi (m >= n, fits one CTA, no V accumulation), else
    // 0 small (theta + V in one CTA), 2 medium (theta in one CTA, V replayed from a rotation log),
    // 1 large (tcgen05 block Jacobi, HBM-resident)
    int qgt = 0, qr = 0;
    static const bool no_qr = getenv("EAMPS_NO_QR") != nullptr;   // dev A/B switch
    gd.regime = (!no_qr && svd_qr_fits(gd.m, gd.n, &qgt, &qr)) ? 3
                : svd_small_fits(gd.m, gd.n)                  ? 0
                : (svd_medium_fits(gd.m, gd.n) ? 2 : 1);
    gd.n_pad = gd.regime != 1 ? gd.n : (int)align_up(gd.n, 64);
    // the rotation log holds every sweep the Jacobi may run (cfg.max_sweeps, default 60), so the medium
    // regime has the same sweep limit as the others (MPS_E_NOCONV only past max_sweeps)
    gd.log_sweeps = gd.regime == 2 ? h->cfg.max_sweeps : 0;
    // medium regime: the rotation log; large regime: the tensor-core Jacobi scratch (G, E images)
    // large regime: the R-preconditioner (FP64 Gram + Cholesky, Jacobi on B = L with n rows, no V
    // accumulation; for m < n the Gram has rank <= m and B gets zero columns); its FP64 Gram shares
    // the tensor-core scratch (dead until the sweeps)
    gd.jrows = (gd.regime == 1 && (gd.m >= gd.n || large_precond_wide()) && large_precond_enabled()) ? gd.n : 0;
    // QR regime, block-recursive kernels: B = L from the FP64 Gram + Cholesky (EAMPS_QR_HOUSEHOLDER=1:
    // the in-CTA Householder QR instead)
    static const bool qr_hh = getenv("EAMPS_QR_HOUSEHOLDER") != nullptr;
    if (gd.regime == 3 && !qr_hh) gd.jrows = gd.n;
    // large regime, 128 < n <= 4096: the eigen route (FP64 Gram eigensolver, no Jacobi sweeps;
    // measured 1.46x / 1.9x / 2.2x the Jacobi route at n = 256 / 512 / 2048)
    gd.eig = (!h->jacobi_only && (eig_route(gd) || eig_route_small(gd))) ? 1 : 0;
    const size_t logb = gd.regime == 2   ? (size_t)gd.log_sweeps * (gd.n - 1) * (gd.n / 2) * 16
                        : gd.regime == 1 ? large_scratch_bytes(gd)
                        : (gd.regime == 3 && gd.eig) ? refine_large_scratch(gd.m, gd.n)
                        : (gd.regime == 3 && gd.jrows > 0) ? large_precond_scratch(gd.n)
                                         : refine_scratch_bytes(gd.n);
    gd.u_index = ord[g].second;
    const size_t mn = (size_t)gd.m * gd.n * 8, mnp = (size_t)std::max(gd.m, gd.jrows) * gd.n_pad * 8;   // B = L (jrows rows) reuses it
    const int kmn = std::min(gd.m, gd.n);
    p.ws = align_up(mnp) + align_up(mn) + align_up((size_t)gd.n_pad * gd.n_pad * 8) + align_up((size_t)gd.n_pad * 8) +
           align_up((size_t)(gd.n_pad + 1) * 8) + align_up((size_t)gd.n_pad * 4) +
           align_up(std::max((size_t)kmn * kmn * 8, (gd.regime == 1 || gd.regime == 3) ? (size_t)16 * gd.n_pad : (size_t)0)) +
           align_up(logb);
    int kmax = std::min(gd.m, gd.n);
    if (h->cfg.chi_cap > 0) kmax = std::min(kmax, h->cfg.chi_cap);
    p.reserve = ((size_t)class_bytes(size_class((uint64_t)gd.l * d * kmax * 8))) +
                ((size_t)class_bytes(size_class((uint64_t)kmax * d * gd.r * 8))) + ((size_t)class_bytes(size_class((uint64_t)kmax * 4))) +
                3 * kAlign;
    p.ctiles = ((gd.l + TA - 1) / TA) * ((gd.r + TA - 1) / TA);
    const int km = std::min(gd.m, gd.n);
    p.rtiles = ((gd.m + 63) / 64) * ((km + 63) / 64) + (km + 63) / 64;
    p.gtiles = ((km + 31) / 32) * ((km + 31) / 32);
    p.atiles = ((gd.n + 63) / 64) * ((km + 63) / 64);
    if (reabsorb_small_fits(gd.m, gd.n)) p.rtiles = p.gtiles = p.atiles = 0;   // k_reabsorb_small
  }

  J.G = G;
  J.d4 = d4;
  J.ord = ord;
  J.us.assign(Us, Us + (size_t)G * d4 * 2);
  J.g0 = 0;
  J.front = false;
  J.active = true;
  h->last_desc.clear();
  h->spectra.clear();
  h->last_wave_begin = 0;
  if (h->hp.on && h->hp.layers > 3) h->hp.plan += HostProf::now() - hp0;
  mps_status fs = wave_front(h);
  if (fs != MPS_OK) {
    J.active = false;
    return fs;
  }
  if (n_waves) *n_waves = 1;
  return MPS_OK;
}

mps_status mps_layer_step(mps_t h, int32_t* remaining) {
  DEVICE_GUARD(h);
  if (!h) return MPS_E_INVAL;
  if (remaining) *remaining = 0;
  LayerJob& J = h->job;
  if (!J.active) return MPS_OK;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) { J.active = false; return st; }
  st = wave_back(h);
  if (st != MPS_OK) { J.active = false; return st; }
  if (J.g0 >= J.G) {
    J.active = false;
    return MPS_OK;
  }
  st = wave_front(h);
  if (st != MPS_OK) { J.active = false; return st; }
  if (remaining) *remaining = J.G - J.g0;
  return MPS_OK;
}

mps_status mps_apply_layer(mps_t h, int32_t G, const int32_t* sites, const float* Us) {
  NvtxScope nv("eamps:mps_apply_layer");
  int32_t w = 0;
  mps_status st = mps_layer_begin(h, G, sites, Us, &w);
  if (st != MPS_OK || w == 0) return st;
  int32_t rem = 1;
  while (rem > 0) {
    st = mps_layer_step(h, &rem);
    if (st != MPS_OK) return st;
  }
  return MPS_OK;
}

mps_status mps_apply_gate2(mps_t h, int32_t site, const float* U) { return mps_apply_layer(h, 1, &site, U); }

mps_status mps_fidelity_estimate(mps_t h, double* est, double* log_est, int64_t* n_done, int32_t* guarantee_held,
                                 int32_t* is_lower_bound) {
  DEVICE_GUARD(h);
  if (!h) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  st = sync_state(h);
  if (st != MPS_OK) return st;
  st = device_error(h);
  if (st != MPS_OK) return st;
  if (est) *est = std::exp(h->hstate.led.logE);
  if (log_est) *log_est = h->hstate.led.logE;
  if (n_done) *n_done = h->hstate.led.j;
  if (guarantee_held) *guarantee_held = h->hstate.led.guarantee;
  if (is_lower_bound) *is_lower_bound = h->d == 4 ? 1 : 0;
  return MPS_OK;
}

// The ledger token of the multi-rank chain (§8(e)): (log E, j, guarantee). get synchronises;
// set is stream-ordered (it lands before the next wave's select).
// Planning introspection (host only, no device work): the SVD regime of an m x n theta and the
// lane-group size / rows per lane its bucket launches with -- the invariants the CPU tests check.
mps_status mps_plan_regime(int32_t m, int32_t n, int32_t* regime, int32_t* gt, int32_t* rpl, int32_t* n_pad) {
  if (m < 1 || n < 1 || !regime || !gt || !rpl || !n_pad) return MPS_E_INVAL;
  int qgt = 0, qr = 0;
  if (svd_qr_fits(m, n, &qgt, &qr)) {
    *regime = 3; *gt = qgt; *rpl = qr; *n_pad = n;
    return MPS_OK;
  }
  const int reg = svd_small_fits(m, n) ? 0 : (svd_medium_fits(m, n) ? 2 : 1);
  *regime = reg;
  if (reg == 1) {
    *gt = 0; *rpl = 0; *n_pad = (int)align_up((size_t)n, 64);
    return MPS_OK;
  }
  *gt = lane_group(m, n, reg);
  const int rm = rows_per_lane(m, *gt), rn = rows_per_lane(n, *gt);
  *rpl = (rm == 0 || rn == 0) ? 0 : std::max(rm, rn);
  *n_pad = n;
  return MPS_OK;
}

mps_status mps_ledger_get(mps_t h, double* log_E, int64_t* j, int32_t* guarantee) {
  DEVICE_GUARD(h);
  if (!h) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  st = sync_state(h);
  if (st != MPS_OK) return st;
  st = device_error(h);
  if (st != MPS_OK) return st;
  if (log_E) *log_E = h->hstate.led.logE;
  if (j) *j = h->hstate.led.j;
  if (guarantee) *guarantee = h->hstate.led.guarantee;
  return MPS_OK;
}

mps_status mps_ledger_set(mps_t h, double log_E, int64_t j, int32_t guarantee) {
  DEVICE_GUARD(h);
  if (!h) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  if (!std::isfinite(log_E) || log_E > 0.0 || j < 0) return set_err(h, MPS_E_INVAL, "bad ledger token");
  if (h->cfg.strategy != MPS_STRAT_FIXED && j > h->cfg.n_planned) return set_err(h, MPS_E_STATE, "j > n_planned");
  // logE (8) | j (8) | guarantee (4): the first 20 bytes of DevLedger; staged in its own pinned slot
  static_assert(offsetof(DevLedger, logE) == 0 && offsetof(DevLedger, j) == 8 && offsetof(DevLedger, guarantee) == 16,
                "ledger layout");
  uint8_t* hb = static_cast<uint8_t*>(pinned_buf(h, 64));
  // the general pinned slot may be reused by the next call before this copy runs: drain first
  std::memcpy(hb, &log_E, 8);
  std::memcpy(hb + 8, &j, 8);
  std::memcpy(hb + 16, &guarantee, 4);
  CK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(h->dst), hb, 20, cudaMemcpyHostToDevice, h->s));
  CK(cudaStreamSynchronize(h->s));
  h->hstate.led.logE = log_E;
  h->hstate.led.j = j;
  h->hstate.led.guarantee = guarantee;
  return MPS_OK;
}

mps_status mps_bond_dims(mps_t h, int32_t* out) {
  if (!h || !out) return MPS_E_INVAL;
  for (int i = 0; i < h->N - 1; ++i) out[i] = h->chr[i];
  return MPS_OK;
}

mps_status mps_schmidt_values(mps_t h, int32_t bond, float* out, int32_t cap, int32_t* len) {
  DEVICE_GUARD(h);
  if (!h || !len) return MPS_E_INVAL;
  if (bond < -1 || bond > h->N - 1) return set_err(h, MPS_E_RANGE, "bond out of range");
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  BondEntry e;
  st = read_bond(h, bond, &e);
  if (st != MPS_OK) return st;
  *len = e.len;
  if (out && cap > 0) {
    int nc = std::min(cap, e.len);
    CK(cudaMemcpyAsync(out, h->slab + e.off, 4 * (size_t)nc, cudaMemcpyDefault, h->s));  // host or device out
    CK(cudaStreamSynchronize(h->s));
  }
  return MPS_OK;
}

mps_status mps_truncation_log(mps_t h, mps_record* rows, int64_t cap, int64_t* len) {
  if (!h || !len) return MPS_E_INVAL;
  *len = (int64_t)h->records.size();
  if (rows)
    for (int64_t r = 0; r < *len && r < cap; ++r) rows[r] = h->records[r];
  return MPS_OK;
}

mps_status mps_last_spectrum(mps_t h, int32_t g, double* out, int32_t cap, int32_t* len) {
  if (!h || !len) return MPS_E_INVAL;
  if (g < 0 || g >= (int)h->last_desc.size()) return set_err(h, MPS_E_RANGE, "gate index out of range");
  const GateDesc& gd = h->last_desc[g];
  if (g < (int)h->spectra.size() && (int)h->spectra[g].size() == gd.n && h->keep_spectra) {   // kept host copy
    *len = gd.n;
    if (out)
      for (int j = 0; j < std::min(cap, gd.n); ++j) out[j] = std::sqrt(std::max(h->spectra[g][j], 0.0));
    return MPS_OK;
  }
  if (g < h->last_wave_begin) return set_err(h, MPS_E_STATE, "spectrum of an earlier wave (workspace reused)");
  *len = gd.n;
  if (out && cap > 0) {
    CK(cudaMemcpyAsync(out, h->slab + gd.ws_sig2, 8 * (size_t)std::min(cap, gd.n), cudaMemcpyDeviceToHost, h->s));
    CK(cudaStreamSynchronize(h->s));
    for (int j = 0; j < std::min(cap, gd.n); ++j) out[j] = std::sqrt(std::max(out[j], 0.0));
  }
  return MPS_OK;
}

mps_status mps_last_sweeps(mps_t h, int32_t g, int32_t* sweeps) {
  if (!h || !sweeps) return MPS_E_INVAL;
  if (g < 0 || g >= (int)h->last_desc.size()) return MPS_E_RANGE;
  *sweeps = h->last_desc[g].sweeps;
  return MPS_OK;
}

mps_status mps_export_site(mps_t h, int32_t site, float* B, int32_t* dims3) {
  DEVICE_GUARD(h);
  if (!h || !dims3) return MPS_E_INVAL;
  if (site < 0 || site >= h->N) return set_err(h, MPS_E_RANGE, "site out of range");
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  SiteEntry e;
  st = read_site(h, site, &e);
  if (st != MPS_OK) return st;
  dims3[0] = e.chl;
  dims3[1] = h->d;
  dims3[2] = e.chr;
  if (B) {
    CK(cudaMemcpyAsync(B, h->slab + e.off, (size_t)e.chl * h->d * e.chr * 8, cudaMemcpyDefault, h->s));
    CK(cudaStreamSynchronize(h->s));
  }
  return MPS_OK;
}

mps_status mps_import_site(mps_t h, int32_t site, const float* B, const int32_t* dims3) {
  DEVICE_GUARD(h);
  if (!h || !B || !dims3) return MPS_E_INVAL;
  if (h->job.active) return set_err(h, MPS_E_STATE, "a layer is in flight");
  if (site < 0 || site >= h->N) return set_err(h, MPS_E_RANGE, "site out of range");
  if (dims3[1] != h->d || dims3[0] < 1 || dims3[2] < 1) return set_err(h, MPS_E_INVAL, "bad dims");
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  const size_t bytes = (size_t)dims3[0] * h->d * dims3[2] * 8;
  int64_t off;
  int cls;
  st = dev_alloc(h, bytes, &off, &cls);
  if (st != MPS_OK) return st;
  SiteEntry old;
  st = read_site(h, site, &old);
  if (st != MPS_OK) return st;
  CK(cudaMemcpyAsync(h->slab + off, B, bytes, is_device_ptr(B) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     h->s));
  SiteEntry* ne = static_cast<SiteEntry*>(pinned_buf(h, sizeof(SiteEntry)));
  ne->off = off;
  ne->chl = dims3[0];
  ne->chr = dims3[2];
  ne->cls = cls;
  ne->pad = 0;
  CK(cudaMemcpyAsync(h->slab + h->hstate.sites_off + sizeof(SiteEntry) * site, ne, sizeof(SiteEntry),
                     cudaMemcpyHostToDevice, h->s));
  if (old.off) {
    launch_pool_free(h->slab, h->dst, old.off, old.cls, h->s);
    ++h->launches;
  }
  CK(cudaStreamSynchronize(h->s));
  h->chl[site] = dims3[0];
  h->chr[site] = dims3[2];
  if (h->lamlen[site] != dims3[0]) {
    st = put_lambda(h, site - 1, nullptr, dims3[0], true);
    if (st != MPS_OK) return st;
  }
  if (h->lamlen[site + 1] != dims3[2]) {
    st = put_lambda(h, site, nullptr, dims3[2], true);
    if (st != MPS_OK) return st;
  }
  return sync_state(h);
}

mps_status mps_import_sites(mps_t h, int32_t first, int32_t count, const float* B, const int32_t* dims) {
  NvtxScope nv("eamps:mps_import_sites");
  DEVICE_GUARD(h);
  if (!h || !B || !dims || count < 1) return MPS_E_INVAL;
  if (h->job.active) return set_err(h, MPS_E_STATE, "a layer is in flight");
  if (first < 0 || first + count > h->N) return set_err(h, MPS_E_RANGE, "sites out of range");
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  std::vector<ImportEntry> ent(count);
  std::vector<int32_t> lamlen = h->lamlen;
  int64_t elems = 0;
  for (int x = 0; x < count; ++x) {
    const int32_t* dm = dims + 3 * x;
    if (dm[1] != h->d || dm[0] < 1 || dm[2] < 1) return set_err(h, MPS_E_INVAL, "bad dims");
    ImportEntry& e = ent[x];
    std::memset(&e, 0, sizeof(e));
    e.site = first + x;
    e.chl = dm[0];
    e.chr = dm[2];
    e.src_elem = elems;
    elems += (int64_t)dm[0] * h->d * dm[2];
    if (lamlen[e.site] != e.chl) {
      e.resetL = e.chl;
      lamlen[e.site] = e.chl;
      // the previous entry may already reset this bond (its right bond): the device scatter runs
      // the entries in parallel, so only the later reset may stay (sequential import semantics)
      if (x > 0) ent[x - 1].resetR = 0;
    }
    if (lamlen[e.site + 1] != e.chr) { e.resetR = e.chr; lamlen[e.site + 1] = e.chr; }
  }
  st = sync_state(h);
  if (st != MPS_OK) return st;
  const bool dev = is_device_ptr(B);
  const size_t ent_bytes = align_up(sizeof(ImportEntry) * count);
  const size_t data_bytes = dev ? 0 : align_up((size_t)elems * 8);
  const size_t top = h->slab_bytes - 4 * kAlign;
  // worst case the new blocks take fresh pool memory: keep the staging area above that
  size_t reserve = 0;
  for (const ImportEntry& e : ent)
    reserve += ((size_t)class_bytes(size_class((uint64_t)e.chl * h->d * e.chr * 8))) + 2 * kAlign +
               (e.resetL ? ((size_t)class_bytes(size_class((uint64_t)e.resetL * 4))) : 0) +
               (e.resetR ? ((size_t)class_bytes(size_class((uint64_t)e.resetR * 4))) : 0);
  if (h->hstate.pool.bump + reserve + ent_bytes + data_bytes + kAlign > top) {
    // host data is staged through the top of the slab: import it in two halves (each half's
    // blocks land in the pool before the next half is staged)
    if (!dev && count > 1) {
      const int c0 = count / 2;
      st = mps_import_sites(h, first, c0, B, dims);
      if (st != MPS_OK) return st;
      return mps_import_sites(h, first + c0, count - c0, B + 2 * ent[c0].src_elem, dims + 3 * c0);
    }
    return set_err(h, MPS_E_NOMEM, "no room to stage the import");
  }
  const size_t base = align_up(top - ent_bytes - data_bytes - kAlign);
  uint8_t* hb = static_cast<uint8_t*>(pinned_buf(h, ent_bytes + 64, 1));
  std::memcpy(hb, ent.data(), sizeof(ImportEntry) * count);
  uint64_t* hceil = reinterpret_cast<uint64_t*>(hb + ent_bytes);
  *hceil = base;
  CK(h2d_small(h, &h->dst->pool.ceiling, hceil, 8));
  CK(h2d_small(h, h->slab + base, hb, sizeof(ImportEntry) * count));
  const float2* src = reinterpret_cast<const float2*>(B);
  if (!dev) {
    CK(cudaMemcpyAsync(h->slab + base + ent_bytes, B, (size_t)elems * 8, cudaMemcpyHostToDevice, h->s));
    src = reinterpret_cast<const float2*>(h->slab + base + ent_bytes);
  }
  launch_import(h->slab, h->dst, reinterpret_cast<ImportEntry*>(h->slab + base), count, src, h->d, h->s);
  h->launches += 2;
  CKL("import");
  st = sync_state(h);
  if (st != MPS_OK) return st;
  st = device_error(h);
  if (st != MPS_OK) return st;
  for (const ImportEntry& e : ent) {
    h->chl[e.site] = e.chl;
    h->chr[e.site] = e.chr;
  }
  h->lamlen = lamlen;
  return MPS_OK;
}

mps_status mps_export_sites(mps_t h, int32_t first, int32_t count, float* B, size_t cap_elems, int32_t* dims,
                            size_t* elems_out) {
  NvtxScope nv("eamps:mps_export_sites");
  DEVICE_GUARD(h);
  if (!h || !dims || count < 1) return MPS_E_INVAL;
  if (h->job.active) return set_err(h, MPS_E_STATE, "a layer is in flight");
  if (first < 0 || first + count > h->N) return set_err(h, MPS_E_RANGE, "sites out of range");
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  st = sync_state(h);
  if (st != MPS_OK) return st;
  // the site table slice [first, first + count): offsets and extents as the device holds them
  SiteEntry* se = static_cast<SiteEntry*>(pinned_buf(h, sizeof(SiteEntry) * (size_t)count));
  if (!se) return set_err(h, MPS_E_NOMEM, "pinned host allocation failed");
  CK(cudaMemcpyAsync(se, h->slab + h->hstate.sites_off + sizeof(SiteEntry) * (size_t)first,
                     sizeof(SiteEntry) * (size_t)count, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  std::vector<ExportEntry> ent(count);
  int64_t elems = 0, maxe = 1;
  for (int x = 0; x < count; ++x) {
    dims[3 * x] = se[x].chl;
    dims[3 * x + 1] = h->d;
    dims[3 * x + 2] = se[x].chr;
    ent[x].src_off = se[x].off;
    ent[x].dst_elem = elems;
    ent[x].elems = (int64_t)se[x].chl * h->d * se[x].chr;
    if (!se[x].off) return set_err(h, MPS_E_STATE, "site without a tensor");
    elems += ent[x].elems;
    maxe = std::max(maxe, ent[x].elems);
  }
  if (elems_out) *elems_out = (size_t)elems;
  if (!B) return MPS_OK;
  if (cap_elems < (size_t)elems) return set_err(h, MPS_E_RANGE, "export buffer too small");
  const bool dev = is_device_ptr(B);
  const size_t ent_bytes = align_up(sizeof(ExportEntry) * (size_t)count);
  const size_t data_bytes = dev ? 0 : align_up((size_t)elems * 8);
  const size_t top = h->slab_bytes - 4 * kAlign;
  if (h->hstate.pool.bump + ent_bytes + data_bytes + 2 * kAlign > top) {
    // a host destination is staged through the top of the slab: export it in two halves
    if (!dev && count > 1) {
      const int c0 = count / 2;
      const size_t e0 = (size_t)ent[c0].dst_elem;
      st = mps_export_sites(h, first, c0, B, e0, dims, nullptr);
      if (st != MPS_OK) return st;
      return mps_export_sites(h, first + c0, count - c0, B + 2 * e0, cap_elems - e0, dims + 3 * c0, nullptr);
    }
    return set_err(h, MPS_E_NOMEM, "no room to stage the export");
  }
  const size_t base = align_up(top - ent_bytes - data_bytes - kAlign);
  uint8_t* hb = static_cast<uint8_t*>(pinned_buf(h, ent_bytes, 1));
  if (!hb) return set_err(h, MPS_E_NOMEM, "pinned host allocation failed");
  std::memcpy(hb, ent.data(), sizeof(ExportEntry) * (size_t)count);
  CK(h2d_small(h, h->slab + base, hb, sizeof(ExportEntry) * (size_t)count));
  float2* dstp = dev ? reinterpret_cast<float2*>(B) : reinterpret_cast<float2*>(h->slab + base + ent_bytes);
  // enough CTAs per site to fill the GPU when the sites are few and large
  const int split = (int)std::max<int64_t>(1, std::min<int64_t>({64, (maxe + 8191) / 8192, (1184 + count - 1) / count}));
  launch_export(h->slab, reinterpret_cast<const ExportEntry*>(h->slab + base), count, split, dstp, h->s);
  ++h->launches;
  CKL("export");
  if (!dev) CK(cudaMemcpyAsync(B, dstp, (size_t)elems * 8, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  return device_error(h);
}

mps_status mps_set_lambda(mps_t h, int32_t bond, const float* lam, int32_t len) {
  DEVICE_GUARD(h);
  if (!h || !lam || len < 1) return MPS_E_INVAL;
  if (h->job.active) return set_err(h, MPS_E_STATE, "a layer is in flight");
  if (bond < -1 || bond > h->N - 1) return set_err(h, MPS_E_RANGE, "bond out of range");
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  std::vector<float> tmp(len);
  if (is_device_ptr(lam)) {
    CK(cudaMemcpy(tmp.data(), lam, 4 * (size_t)len, cudaMemcpyDeviceToHost));
  } else {
    std::memcpy(tmp.data(), lam, 4 * (size_t)len);
  }
  st = put_lambda(h, bond, tmp.data(), len, false);
  if (st != MPS_OK) return st;
  return sync_state(h);
}

mps_status mps_amplitude(mps_t h, const uint8_t* digits, double* re_im) {
  DEVICE_GUARD(h);
  if (!h || !digits || !re_im) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  if (h->chl[0] != 1 || h->chr[h->N - 1] != 1) return set_err(h, MPS_E_STATE, "open boundary legs");
  int maxchi = 1;
  for (int i = 0; i < h->N; ++i) {
    if (digits[i] >= h->d) return set_err(h, MPS_E_INVAL, "digit out of range");
    maxchi = std::max(maxchi, h->chr[i]);
  }
  st = sync_state(h);
  if (st != MPS_OK) return st;
  const size_t need = 2 * align_up((size_t)maxchi * 16) + kAlign;
  if (h->hstate.pool.bump + need + 4 * kAlign > h->slab_bytes) return set_err(h, MPS_E_NOMEM, "no room for query");
  const size_t base = align_up(h->slab_bytes - 4 * kAlign - need);
  double2* v0 = reinterpret_cast<double2*>(h->slab + base);
  double2* v1 = reinterpret_cast<double2*>(h->slab + base + align_up((size_t)maxchi * 16));
  double2* one = static_cast<double2*>(pinned_buf(h, 16));
  *one = make_double2(1.0, 0.0);
  CK(cudaMemcpyAsync(v0, one, 16, cudaMemcpyHostToDevice, h->s));
  for (int i = 0; i < h->N; ++i) {
    launch_amplitude_step(h->slab, h->dst, i, digits[i], v0, v1, h->s);
    ++h->launches;
    std::swap(v0, v1);
  }
  CKL("amplitude");
  CK(cudaMemcpyAsync(one, v0, 16, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  re_im[0] = one->x;
  re_im[1] = one->y;
  return device_error(h);
}

mps_status mps_to_statevector(mps_t h, double* out, size_t n_doubles) {
  DEVICE_GUARD(h);
  if (!h || !out) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  if (h->chl[0] != 1 || h->chr[h->N - 1] != 1) return set_err(h, MPS_E_STATE, "open boundary legs");
  double total = std::pow((double)h->d, h->N);
  if (total > (double)(1 << 26)) return set_err(h, MPS_E_TOOBIG, "d^N > 2^26");
  const int64_t tot = (int64_t)total;
  if (n_doubles < 2 * (size_t)tot) return set_err(h, MPS_E_RANGE, "output buffer too small");
  // largest intermediate: rows * chi <= d^N (chi_i <= d^(N-i-1)); allow slack
  size_t maxel = 1;
  {
    double rows = 1;
    for (int i = 0; i < h->N; ++i) {
      rows *= h->d;
      maxel = std::max(maxel, (size_t)(rows * h->chr[i]));
    }
  }
  st = sync_state(h);
  if (st != MPS_OK) return st;
  const size_t need = 2 * align_up(maxel * 16) + kAlign;
  if (h->hstate.pool.bump + need + 4 * kAlign > h->slab_bytes) return set_err(h, MPS_E_NOMEM, "no room for query");
  const size_t base = align_up(h->slab_bytes - 4 * kAlign - need);
  double2* S0 = reinterpret_cast<double2*>(h->slab + base);
  double2* S1 = reinterpret_cast<double2*>(h->slab + base + align_up(maxel * 16));
  double2* one = static_cast<double2*>(pinned_buf(h, 16));
  *one = make_double2(1.0, 0.0);
  CK(cudaMemcpyAsync(S0, one, 16, cudaMemcpyHostToDevice, h->s));
  int64_t rows = 1;
  int cols = 1;
  for (int i = 0; i < h->N; ++i) {
    launch_statevector_step(h->slab, h->dst, i, rows, cols, S0, S1, h->s);
    ++h->launches;
    rows *= h->d;
    cols = h->chr[i];
    std::swap(S0, S1);
  }
  CKL("statevector");
  CK(cudaMemcpyAsync(out, S0, (size_t)tot * 16, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  return device_error(h);
}

// ---- NEXT-1: exact canonicalisation -----------------------------------------------
// Two sweeps of exact two-site updates with the identity gate through the regular layer path (the
// same kernels): right to left (bonds N-2 .. 0: every B_1 .. B_{N-1} becomes right-orthonormal,
// B_{i+1} = V^H), then left to right (bonds 0 .. N-2: theta = lambda_{i-1} B_i B_{i+1} is then the
// exact Schmidt decomposition at bond i, lambda_i <- its renormalised singular values). PAPER.md:76
// (QR / RQ sweeps "the state is now in canonical form"), :84 ("enforced throughout"). The device
// ledger runs in per-update exact mode (FIXED, t = 1, no cap) during the sweeps and is restored after
// (log E, j, guarantee and the records are untouched); the GPU's exact mode keeps sigma > 1e-6 sigma_0
// (reading 8), i.e. drops at most n 1e-12 of the weight per bond.
mps_status mps_canonicalize(mps_t h) {
  NvtxScope nv("eamps:mps_canonicalize");
  DEVICE_GUARD(h);
  if (!h) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  if (h->job.active) return set_err(h, MPS_E_STATE, "a layer is still in progress (mps_layer_step)");
  st = sync_state(h);
  if (st != MPS_OK) return st;
  const DevLedger saved = h->hstate.led;
  const mps_config cfg_saved = h->cfg;
  const size_t nrec = h->records.size();
  DevLedger tmp = saved;
  tmp.strategy = MPS_STRAT_FIXED;
  tmp.log_ffixed = 0.0;
  tmp.chi_cap = 0;
  DevLedger* hb = static_cast<DevLedger*>(pinned_buf(h, sizeof(DevLedger)));
  *hb = tmp;
  CK(cudaMemcpyAsync(&h->dst->led, hb, sizeof(DevLedger), cudaMemcpyHostToDevice, h->s));
  CK(cudaStreamSynchronize(h->s));
  h->cfg.strategy = MPS_STRAT_FIXED;
  h->cfg.f_fixed = 1.0;
  h->cfg.chi_cap = 0;
  const int dd = h->d * h->d;
  std::vector<float> ident((size_t)2 * dd * dd, 0.f);
  for (int x = 0; x < dd; ++x) ident[2 * (x * dd + x)] = 1.f;
  for (int i = h->N - 2; i >= 0 && st == MPS_OK; --i) st = mps_apply_layer(h, 1, &i, ident.data());
  for (int i = 0; i <= h->N - 2 && st == MPS_OK; ++i) st = mps_apply_layer(h, 1, &i, ident.data());
  // restore the caller's ledger and configuration (the sweeps' f_j = 1 - T_k/P ~ 1 are not counted)
  h->cfg = cfg_saved;
  h->records.resize(nrec);
  if (st != MPS_OK) return st;
  st = sync_state(h);
  if (st != MPS_OK) return st;
  DevLedger back = h->hstate.led;
  back.logE = saved.logE;
  back.j = saved.j;
  back.guarantee = saved.guarantee;
  back.strategy = saved.strategy;
  back.log_ffixed = saved.log_ffixed;
  back.chi_cap = saved.chi_cap;
  hb = static_cast<DevLedger*>(pinned_buf(h, sizeof(DevLedger)));
  *hb = back;
  CK(cudaMemcpyAsync(&h->dst->led, hb, sizeof(DevLedger), cudaMemcpyHostToDevice, h->s));
  CK(cudaStreamSynchronize(h->s));
  h->hstate.led = back;
  return device_error(h);
}

// ---- observables (NEXT-4) ---------------------------------------------------------
namespace {

mps_status site_table(mps_t h, std::vector<SiteEntry>& out) {
  mps_status st = sync_state(h);
  if (st != MPS_OK) return st;
  out.resize(h->N);
  SiteEntry* hb = static_cast<SiteEntry*>(pinned_buf(h, sizeof(SiteEntry) * h->N));
  if (!hb) return set_err(h, MPS_E_NOMEM, "pinned host allocation failed");
  CK(cudaMemcpyAsync(hb, h->slab + h->hstate.sites_off, sizeof(SiteEntry) * h->N, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  std::copy(hb, hb + h->N, out.begin());
  return MPS_OK;
}

// scratch carved from the top of the slab (above the pool), like the amplitude / statevector queries
mps_status query_scratch(mps_t h, size_t bytes, uint8_t** base) {
  const size_t need = align_up(bytes) + kAlign;
  if (h->hstate.pool.bump + need + 4 * kAlign > h->slab_bytes) return set_err(h, MPS_E_NOMEM, "no room for query");
  *base = h->slab + align_up(h->slab_bytes - 4 * kAlign - need);
  return MPS_OK;
}

// <a|b> by left-to-right transfer matrices E_{i+1} = sum_s A_i^{s dagger} E_i B_i^s (FP64), the
// two-site step at `site` (if O != nullptr) contracting the bra theta with O theta (E5)
mps_status transfer_chain(mps_t a, mps_t b, const std::vector<SiteEntry>& sa, const std::vector<SiteEntry>& sb,
                          int site, const float2* dO, double2* result) {
  const int N = a->N, d = a->d;
  size_t maxe = 1, maxt = 1;
  for (int i = 0; i < N; ++i) {
    maxe = std::max(maxe, (size_t)sa[i].chr * sb[i].chr);
    maxt = std::max(maxt, (size_t)sa[i].chl * d * sb[i].chr);
  }
  size_t th_el = 0;
  if (dO) {
    th_el = (size_t)sa[site].chl * d * d * sa[site + 1].chr;
    maxt = std::max(maxt, (size_t)sa[site].chl * d * d * sb[site + 1].chr);
  }
  uint8_t* base = nullptr;
  const size_t eb = align_up(maxe * 16), tb = align_up(maxt * 16), thb = align_up(th_el * 16);
  mps_status st = query_scratch(a, 2 * eb + tb + 2 * thb + kAlign, &base);
  if (st != MPS_OK) return st;
  double2* E0 = reinterpret_cast<double2*>(base);
  double2* E1 = reinterpret_cast<double2*>(base + eb);
  double2* Tb = reinterpret_cast<double2*>(base + 2 * eb);
  double2* th = reinterpret_cast<double2*>(base + 2 * eb + tb);
  double2* oth = reinterpret_cast<double2*>(base + 2 * eb + tb + thb);
  double2* one = static_cast<double2*>(pinned_buf(a, 16));
  *one = make_double2(1.0, 0.0);
  mps_t h = a;
  CK(cudaMemcpyAsync(E0, one, 16, cudaMemcpyHostToDevice, a->s));
  for (int i = 0; i < N; ++i) {
    if (dO && i == site) {
      const float2* Bk = reinterpret_cast<const float2*>(a->slab + sa[i].off);
      const float2* Bk1 = reinterpret_cast<const float2*>(a->slab + sa[i + 1].off);
      const int l = sa[i].chl, mid = sa[i].chr, r = sa[i + 1].chr;
      launch_theta2(Bk, Bk1, th, l, d, mid, r, a->s);
      launch_apply_O(dO, th, oth, l, d * d, r, a->s);
      launch_transfer(E0, th, true, oth, true, Tb, E1, l, l, d * d, r, r, a->s);
      a->launches += 4;
      std::swap(E0, E1);
      ++i;
      continue;
    }
    const void* A = a->slab + sa[i].off;
    const void* B = b->slab + sb[i].off;
    launch_transfer(E0, A, false, B, false, Tb, E1, sa[i].chl, sb[i].chl, d, sa[i].chr, sb[i].chr, a->s);
    a->launches += 2;
    std::swap(E0, E1);
  }
  CKL("transfer");
  CK(cudaMemcpyAsync(one, E0, 16, cudaMemcpyDeviceToHost, a->s));
  CK(cudaStreamSynchronize(a->s));
  *result = *one;
  return MPS_OK;
}

}  // namespace

mps_status mps_overlap(mps_t a, mps_t b, double* re_im) {
  DEVICE_GUARD(a);
  if (!a || !b || !re_im) return MPS_E_INVAL;
  mps_t h = a;
  if (a->N != b->N || a->d != b->d) return set_err(a, MPS_E_INVAL, "overlap: different N or d");
  if (a->device != b->device) return set_err(a, MPS_E_INVAL, "overlap: handles on different devices");
  if (a->job.active || b->job.active) return set_err(a, MPS_E_STATE, "a layer is in progress");
  mps_status st = check_sticky(a);
  if (st != MPS_OK) return st;
  st = check_sticky(b);
  if (st != MPS_OK) return set_err(a, st, "overlap: the other handle has a sticky error");
  if (a->chl[0] != 1 || a->chr[a->N - 1] != 1 || b->chl[0] != 1 || b->chr[b->N - 1] != 1)
    return set_err(a, MPS_E_STATE, "open boundary legs");
  if (b != a) CK(cudaStreamSynchronize(b->s));
  std::vector<SiteEntry> sa, sb;
  st = site_table(a, sa);
  if (st != MPS_OK) return st;
  st = b == a ? MPS_OK : site_table(b, sb);
  if (st != MPS_OK) return set_err(a, st, "overlap: reading the other handle");
  double2 v;
  st = transfer_chain(a, b, sa, b == a ? sa : sb, -1, nullptr, &v);
  if (st != MPS_OK) return st;
  re_im[0] = v.x;
  re_im[1] = v.y;
  return device_error(a);
}

mps_status mps_trace(mps_t h, double* re_im) {
  DEVICE_GUARD(h);
  if (!h || !re_im) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  if (h->d != 4) return set_err(h, MPS_E_STATE, "trace: d = 4 (vectorised MPO) only");
  if (h->chl[0] != 1 || h->chr[h->N - 1] != 1) return set_err(h, MPS_E_STATE, "open boundary legs");
  std::vector<SiteEntry> se;
  st = site_table(h, se);
  if (st != MPS_OK) return st;
  int maxchi = 1;
  for (int i = 0; i < h->N; ++i) maxchi = std::max(maxchi, (int)se[i].chr);
  uint8_t* base = nullptr;
  const size_t vb = align_up((size_t)maxchi * 16);
  st = query_scratch(h, 2 * vb, &base);
  if (st != MPS_OK) return st;
  double2* v0 = reinterpret_cast<double2*>(base);
  double2* v1 = reinterpret_cast<double2*>(base + vb);
  double2* one = static_cast<double2*>(pinned_buf(h, 16));
  *one = make_double2(1.0, 0.0);
  CK(cudaMemcpyAsync(v0, one, 16, cudaMemcpyHostToDevice, h->s));
  for (int i = 0; i < h->N; ++i) {
    launch_trace_step(reinterpret_cast<const float2*>(h->slab + se[i].off), v0, v1, se[i].chl, se[i].chr, h->s);
    ++h->launches;
    std::swap(v0, v1);
  }
  CKL("trace");
  CK(cudaMemcpyAsync(one, v0, 16, cudaMemcpyDeviceToHost, h->s));
  CK(cudaStreamSynchronize(h->s));
  re_im[0] = one->x;
  re_im[1] = one->y;
  return device_error(h);
}

mps_status mps_expectation2(mps_t h, int32_t site, const float* O, double* re_im) {
  DEVICE_GUARD(h);
  if (!h || !O || !re_im) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  if (h->d != 2) return set_err(h, MPS_E_STATE, "expectation2: d = 2 (MPS) only");
  if (site < 0 || site >= h->N - 1) return set_err(h, MPS_E_RANGE, "site out of range");
  if (h->job.active) return set_err(h, MPS_E_STATE, "a layer is in progress");
  if (h->chl[0] != 1 || h->chr[h->N - 1] != 1) return set_err(h, MPS_E_STATE, "open boundary legs");
  const int D = h->d * h->d;
  for (int x = 0; x < 2 * D * D; ++x)
    if (!std::isfinite(O[x])) return set_err(h, MPS_E_INVAL, "non-finite operator entry");
  std::vector<SiteEntry> se;
  st = site_table(h, se);
  if (st != MPS_OK) return st;
  // the operator and the identity staged below the query scratch (the top 2 KB of the slab)
  float2* hO = static_cast<float2*>(pinned_buf(h, 16 * D * D));
  std::memcpy(hO, O, 8 * (size_t)D * D);
  for (int x = 0; x < D * D; ++x) hO[D * D + x] = make_float2((x / D) == (x % D) ? 1.f : 0.f, 0.f);
  float2* dO = reinterpret_cast<float2*>(h->slab + h->slab_bytes - 3 * kAlign);   // 2 x 16 x 8 B = 256 B
  CK(cudaMemcpyAsync(dO, hO, 16 * (size_t)D * D, cudaMemcpyHostToDevice, h->s));
  double2 num, den;
  st = transfer_chain(h, h, se, se, site, dO, &num);
  if (st != MPS_OK) return st;
  st = transfer_chain(h, h, se, se, site, dO + D * D, &den);
  if (st != MPS_OK) return st;
  const double dd = den.x * den.x + den.y * den.y;
  if (!(dd > 0.0)) return set_err(h, MPS_E_STATE, "zero norm");
  re_im[0] = (num.x * den.x + num.y * den.y) / dd;
  re_im[1] = (num.y * den.x - num.x * den.y) / dd;
  return device_error(h);
}

mps_status mps_snapshot_save(mps_t h, void* buf, size_t buf_bytes, size_t* bytes_needed) {
  DEVICE_GUARD(h);
  if (!h) return MPS_E_INVAL;
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  st = sync_state(h);
  if (st != MPS_OK) return st;
  const size_t need = h->hstate.pool.bump;
  if (bytes_needed) *bytes_needed = need;
  if (!buf) return MPS_OK;
  if (buf_bytes < need) return set_err(h, MPS_E_RANGE, "snapshot buffer too small");
  CK(cudaMemcpyAsync(buf, h->slab, need, cudaMemcpyDeviceToDevice, h->s));
  CK(cudaStreamSynchronize(h->s));
  h->snap.valid = true;
  h->snap.chl = h->chl;
  h->snap.chr = h->chr;
  h->snap.lamlen = h->lamlen;
  h->snap.hstate = h->hstate;
  h->snap.nrec = h->records.size();
  return MPS_OK;
}

mps_status mps_snapshot_load(mps_t h, const void* buf, size_t buf_bytes) {
  DEVICE_GUARD(h);
  if (!h || !buf) return MPS_E_INVAL;
  if (h->job.active) return set_err(h, MPS_E_STATE, "a layer is in flight");
  if (!h->snap.valid) return set_err(h, MPS_E_STATE, "no snapshot saved by this handle");
  const size_t need = h->snap.hstate.pool.bump;
  if (buf_bytes < need) return set_err(h, MPS_E_RANGE, "snapshot buffer too small");
  mps_status st = check_sticky(h);
  if (st != MPS_OK) return st;
  CK(cudaMemcpyAsync(h->slab, buf, need, cudaMemcpyDeviceToDevice, h->s));
  CK(cudaStreamSynchronize(h->s));
  h->chl = h->snap.chl;
  h->chr = h->snap.chr;
  h->lamlen = h->snap.lamlen;
  h->hstate = h->snap.hstate;
  h->records.resize(h->snap.nrec);
  h->last_desc.clear();
  return MPS_OK;
}

}  // extern "C"
