// select.cu -- step a4: target, rank selection and ledger, plus the device-side
// pool allocator of the site store (north-star: "a per-site HBM tensor store with variable chi
// and a device-side pool allocator").
//
// Rank selection, per gate (one warp):
//   log t_j  (E14; strategies PAPER.md:153/158 in log space, DESIGN reading 6)
//     naive   : log F_min / n
//     global  : min(0, (log F_min - log E) / R)                R = n - j
//     nearest : min(0, log F_min - log E - (R - 1) log F_min / n)
//     fixed   : log f_fixed (config-2 microbench)
//   tau = 1 - t (pure / ratio) or 1 - t^2 (wang)      (E10/E11 readings 1-2)
//   k = min{k >= 1 : T_k <= tau P}  ("as close to but not lower than f_t")
//       -- a 32-ary warp search over the non-increasing tails T
//   k <= min(m, n); k > chi_cap -> k = chi_cap, guarantee lost
//   f = 1 - T_k/P (pure/ratio) or sqrt(1 - T_k/P) (wang)
// FIXED / NAIVE targets do not depend on the ledger: one warp per gate, all gates in parallel.
// GLOBAL / NEAREST: t_j depends on E_{j-1}, so one warp walks the wave in canonical order.
//
// Commit (one CTA): log E += log f_j in canonical order (E12), the truncation records, and the
// pool: the old blocks of B_i, B_{i+1}, lambda_i are deferred-freed (released at the next commit,
// after the reabsorb that never reads them has finished); the new blocks come from per-class
// free stacks (power-of-two classes) or the bump pointer. One thread plans every request with
// shared-memory counters only (no global loads on the sequential path); all threads then resolve
// the stack pops and write the site tables in parallel.
#include "eamps_internal.cuh"

namespace eamps {

namespace {

// ---- single-threaded pool ops (host-side helpers and import; not on the layer hot path) ----
__device__ uint64_t pool_alloc(uint8_t* slab, DevState* st, uint64_t bytes, int* cls_out) {
  DevPool& P = st->pool;
  int c = size_class(bytes);
  *cls_out = c;
  int64_t* stk = reinterpret_cast<int64_t*>(slab + P.stack_off);
  if (P.count[c] > 0) return (uint64_t)stk[(int64_t)c * P.stack_cap + (--P.count[c])];
  uint64_t o = (P.bump + 255ull) & ~255ull;
  uint64_t sz = 1ull << c;
  if (o + sz > P.ceiling) {
    if (st->led.error == 0) st->led.error = -3;  // MPS_E_NOMEM
    return 0;
  }
  P.bump = o + sz;
  return o;
}

__device__ void pool_free_now(uint8_t* slab, DevState* st, uint64_t off, int cls) {
  if (!off) return;
  DevPool& P = st->pool;
  if (P.count[cls] >= P.stack_cap) {  // cannot happen with stack_cap >= live + pending blocks
    if (st->led.error == 0) st->led.error = -3;
    return;
  }
  int64_t* stk = reinterpret_cast<int64_t*>(slab + P.stack_off);
  stk[(int64_t)cls * P.stack_cap + (P.count[cls]++)] = (int64_t)off;
}

__device__ __forceinline__ double target_log(int strategy, double log_fmin, double log_ffixed, int64_t n_planned,
                                             double logE, int64_t j, bool* bad) {
  *bad = false;
  double lt;
  if (strategy == 3) {
    lt = log_ffixed;
  } else {
    if (j >= n_planned) { *bad = true; return 0.0; }
    double R = (double)(n_planned - j);
    if (strategy == 0) lt = log_fmin / (double)n_planned;
    else if (strategy == 2) lt = (log_fmin - logE) / R;
    else lt = log_fmin - logE - (R - 1.0) * log_fmin / (double)n_planned;
  }
  return lt < 0.0 ? lt : 0.0;
}

// Rank search for one gate by one warp; writes k, capped, f, t, nu, dlogE, disc into gd.
__device__ void rank_one(GateDesc& gd, const uint8_t* slab, int rule, int chi_cap, double lt) {
  const int lane = threadIdx.x & 31;
  const double* T = reinterpret_cast<const double*>(slab + gd.ws_T);
  const double* s2 = reinterpret_cast<const double*>(slab + gd.ws_sig2);
  const int n = gd.n;
  const double P = T[0];
  const double tau = rule == 1 ? -expm1(2.0 * lt) : -expm1(lt);
  int k;
  if (!(P > 0.0)) {
    k = 1;
  } else if (tau <= 0.0) {
    // exact mode: keep sigma > 1e-6 sigma_0 (the FP32 noise floor; reading 8)
    const double thr = 1e-12 * s2[0];
    int cnt = 0;
    for (int j0 = 0; j0 < n; j0 += 32) {
      int j = j0 + lane;
      unsigned b = __ballot_sync(0xffffffffu, j < n && s2[j] > thr);
      cnt += __popc(b);
    }
    k = max(1, cnt);
  } else {
    const double thr = tau * P;
    int lo = 1, hi = n;  // invariant: answer in [lo, hi] and T[hi] <= thr (T[n] = 0)
    while (lo < hi) {
      const int step = (hi - lo + 31) / 32;
      const int cand = lo + lane * step;
      const bool pred = cand < hi ? (T[cand] <= thr) : true;
      const unsigned b = __ballot_sync(0xffffffffu, pred);
      if (b == 0u) {
        lo = lo + 31 * step + 1;
      } else {
        const int f = __ffs(b) - 1;
        hi = min(hi, lo + f * step);
        if (f > 0) lo = lo + (f - 1) * step + 1;
      }
    }
    k = lo;
  }
  const int kmax = min(gd.m, n);
  if (k > kmax) k = kmax;
  int capped = 0;
  if (chi_cap > 0 && k > chi_cap) { k = chi_cap; capped = 1; }
  double kw = 0.0;  // nu^2 = kept weight: lane-strided FP64 sum + xor tree (deterministic)
  for (int j = lane; j < k; j += 32) kw += s2[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) kw += __shfl_xor_sync(0xffffffffu, kw, o);
  if (lane == 0) {
    const double r = P > 0.0 ? T[k] / P : 0.0;
    if (rule == 1) { gd.f = sqrt(1.0 - r); gd.dlogE = 0.5 * log1p(-r); }
    else { gd.f = 1.0 - r; gd.dlogE = log1p(-r); }
    gd.k = k; gd.capped = capped; gd.t = exp(lt); gd.nu = sqrt(kw); gd.disc = r;
  }
  __syncwarp();
}

__global__ void k_select_parallel(GateDesc* desc, int G, const uint8_t* slab, const DevState* st) {
  const int g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= G) return;
  const DevLedger& L = st->led;
  bool bad;
  // the target does not depend on the ledger here: j only guards n_planned (checked on the host)
  double lt = target_log(L.strategy, L.log_fmin, L.log_ffixed, L.n_planned, 0.0, 0, &bad);
  rank_one(desc[g], slab, L.rule, L.chi_cap, lt);
}

__global__ void k_select_sequential(GateDesc* desc, int G, const uint8_t* slab, DevState* st) {
  const int lane = threadIdx.x;
  const DevLedger L = st->led;
  double logE = L.logE;
  int64_t j = L.j;
  for (int g = 0; g < G; ++g) {
    bool bad;
    double lt = target_log(L.strategy, L.log_fmin, L.log_ffixed, L.n_planned, logE, j, &bad);
    if (bad) {
      if (lane == 0) { st->led.error = -8; for (int x = g; x < G; ++x) desc[x].k = 0; }
      return;
    }
    rank_one(desc[g], slab, L.rule, L.chi_cap, lt);
    logE += desc[g].dlogE;  // the same summation order as the commit kernel
    ++j;
  }
}

constexpr int kCommitThreads = 1024;
constexpr int kChunk = 2048;  // gates planned per shared-memory chunk

__global__ void __launch_bounds__(kCommitThreads) k_commit(GateDesc* desc, int G, uint8_t* slab, DevState* st,
                                                            Record* rec) {
  extern __shared__ __align__(16) uint8_t sm[];
  // chunk scratch: plan[3*kChunk] (uint64: offset, or stack slot with the top bit set), cls[3*kChunk]
  uint64_t* plan = reinterpret_cast<uint64_t*>(sm);
  int32_t* pcls = reinterpret_cast<int32_t*>(plan + 3 * kChunk);
  int64_t* ordv = reinterpret_cast<int64_t*>(pcls + 3 * kChunk);  // ledger index per gate of the chunk
  double* gdl = reinterpret_cast<double*>(ordv + kChunk);             // per-gate fields, preloaded in parallel
  int32_t* gk = reinterpret_cast<int32_t*>(gdl + kChunk);
  int32_t* gl = gk + kChunk;
  int32_t* gr = gl + kChunk;
  int32_t* gc = gr + kChunk;
  __shared__ int32_t cnt[kMaxClasses];
  __shared__ uint64_t s_bump;
  __shared__ int s_err;
  const int tid = threadIdx.x;
  DevPool& P = st->pool;
  int64_t* stk = reinterpret_cast<int64_t*>(slab + P.stack_off);
  int64_t* pend = reinterpret_cast<int64_t*>(slab + P.pending_off);
  SiteEntry* sites = reinterpret_cast<SiteEntry*>(slab + st->sites_off);
  BondEntry* bonds = reinterpret_cast<BondEntry*>(slab + st->bonds_off);
  const int d = st->d;
  const int64_t cap = P.stack_cap;
  const uint64_t ceiling = P.ceiling;
  if (tid < kMaxClasses) cnt[tid] = P.count[tid];
  if (tid == 0) { s_bump = P.bump; s_err = st->led.error; }
  __syncthreads();

  // A. release the previous wave's deferred frees onto the class stacks
  const int64_t npend = P.npending;
  for (int64_t c0 = 0; c0 < npend; c0 += 3 * kChunk) {
    const int64_t cn = min((int64_t)3 * kChunk, npend - c0);
    for (int64_t x = tid; x < cn; x += kCommitThreads) {
      plan[x] = (uint64_t)pend[2 * (c0 + x)];
      pcls[x] = (int32_t)pend[2 * (c0 + x) + 1];
    }
    __syncthreads();
    if (tid == 0) {
      for (int64_t x = 0; x < cn; ++x) {
        if (!plan[x]) continue;
        int c = pcls[x];
        if (cnt[c] >= cap) { s_err = -3; plan[x] = 0; continue; }
        pcls[x] = c | (cnt[c]++ << 6);  // class (6 bits) + stack slot
      }
    }
    __syncthreads();
    for (int64_t x = tid; x < cn; x += kCommitThreads) {
      if (!plan[x]) continue;
      int c = pcls[x] & 63, slot = pcls[x] >> 6;
      stk[(int64_t)c * cap + slot] = (int64_t)plan[x];
    }
    __syncthreads();
  }

  // B/C. per chunk of gates: sequential plan (ledger + allocation) then parallel resolve
  double logE = st->led.logE;
  int64_t j = st->led.j;
  int guarantee = st->led.guarantee;
  for (int g0 = 0; g0 < G; g0 += kChunk) {
    const int gn = min(kChunk, G - g0);
    for (int x = tid; x < gn; x += kCommitThreads) {  // parallel preload: no global loads below
      const GateDesc& gd = desc[g0 + x];
      gk[x] = gd.k; gl[x] = gd.l; gr[x] = gd.r; gc[x] = gd.capped; gdl[x] = gd.dlogE;
    }
    __syncthreads();
    if (tid == 0) {
      for (int x = 0; x < gn; ++x) {
        ordv[x] = -1;
        const int kk = gk[x];
        if (kk <= 0 || s_err) { plan[3 * x] = plan[3 * x + 1] = plan[3 * x + 2] = 0; continue; }
        logE += gdl[x];
        ordv[x] = j++;
        if (gc[x]) guarantee = 0;
        const uint64_t bytes[3] = {(uint64_t)gl[x] * d * kk * 8, (uint64_t)kk * d * gr[x] * 8, (uint64_t)kk * 4};
        for (int q = 0; q < 3; ++q) {
          int c = size_class(bytes[q]);
          pcls[3 * x + q] = c;
          if (cnt[c] > 0) {
            plan[3 * x + q] = (1ull << 63) | (uint64_t)(--cnt[c]);
          } else {
            uint64_t o = (s_bump + 255ull) & ~255ull;
            if (o + (1ull << c) > ceiling) { s_err = -3; plan[3 * x + q] = 0; continue; }
            s_bump = o + (1ull << c);
            plan[3 * x + q] = o;
          }
        }
      }
    }
    __syncthreads();
    for (int x = tid; x < gn; x += kCommitThreads) {
      GateDesc& gd = desc[g0 + x];
      const int i = gd.site;
      uint64_t off[3] = {0, 0, 0};
      bool ok = ordv[x] >= 0;
      for (int q = 0; q < 3 && ok; ++q) {
        uint64_t p = plan[3 * x + q];
        if (!p) { ok = false; break; }
        off[q] = (p >> 63) ? (uint64_t)stk[(int64_t)pcls[3 * x + q] * cap + (int64_t)(p & ~(1ull << 63))] : p;
      }
      const int64_t pb = 3 * (int64_t)(g0 + x);
      if (!ok) {
        gd.k = 0;
        pend[2 * pb] = pend[2 * pb + 2] = pend[2 * pb + 4] = 0;
        continue;
      }
      // deferred frees of the old blocks
      pend[2 * pb] = sites[i].off; pend[2 * pb + 1] = sites[i].cls;
      pend[2 * pb + 2] = sites[i + 1].off; pend[2 * pb + 3] = sites[i + 1].cls;
      pend[2 * pb + 4] = bonds[i + 1].off; pend[2 * pb + 5] = bonds[i + 1].cls;
      sites[i].off = (int64_t)off[0]; sites[i].chr = gd.k; sites[i].cls = pcls[3 * x];
      sites[i + 1].off = (int64_t)off[1]; sites[i + 1].chl = gd.k; sites[i + 1].cls = pcls[3 * x + 1];
      bonds[i + 1].off = (int64_t)off[2]; bonds[i + 1].len = gd.k; bonds[i + 1].cls = pcls[3 * x + 2];
      gd.off_newL = (int64_t)off[0]; gd.off_newR = (int64_t)off[1]; gd.off_newLam = (int64_t)off[2];
      Record& R = rec[g0 + x];
      R.gate_index = ordv[x]; R.bond = i; R.chi_before = gd.mid; R.chi_after = gd.k; R.capped = gd.capped;
      R.target_f = gd.t; R.achieved_f = gd.f; R.discarded_weight = gd.disc;
    }
    __syncthreads();
  }
  if (tid < kMaxClasses) P.count[tid] = cnt[tid];
  if (tid == 0) {
    P.bump = s_bump;
    P.npending = 3 * (int64_t)G;
    st->led.logE = logE;
    st->led.j = j;
    st->led.guarantee = guarantee;
    if (s_err && !st->led.error) st->led.error = s_err;
  }
}

__global__ void k_pool_alloc(uint8_t* slab, DevState* st, uint64_t bytes, int64_t* out) {
  int c;
  uint64_t o = pool_alloc(slab, st, bytes, &c);
  out[0] = (int64_t)o;
  out[1] = c;
}
__global__ void k_pool_free(uint8_t* slab, DevState* st, int64_t off, int cls) {
  pool_free_now(slab, st, (uint64_t)off, cls);
}

// single-site gate: B[a,s,c] <- sum_s' U[s,s'] B[a,s',c]   (unitary -> canonical form kept)
template <int D>
__global__ void k_gate1(uint8_t* slab, DevState* st, int site, const float2* U) {
  const SiteEntry e = reinterpret_cast<const SiteEntry*>(slab + st->sites_off)[site];
  float2* B = reinterpret_cast<float2*>(slab + e.off);
  const int64_t tot = (int64_t)e.chl * e.chr;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = x / e.chr, c = x % e.chr;
    float2 in[D];
#pragma unroll
    for (int s = 0; s < D; ++s) in[s] = B[(a * D + s) * e.chr + c];
#pragma unroll
    for (int s = 0; s < D; ++s) {
      float2 o = make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < D; ++t) {
        float2 u = U[s * D + t];
        o.x += u.x * in[t].x - u.y * in[t].y;
        o.y += u.x * in[t].y + u.y * in[t].x;
      }
      B[(a * D + s) * e.chr + c] = o;
    }
  }
}

__global__ void k_import_alloc(uint8_t* slab, DevState* st, ImportEntry* ent, int count) {
  SiteEntry* sites = reinterpret_cast<SiteEntry*>(slab + st->sites_off);
  BondEntry* bonds = reinterpret_cast<BondEntry*>(slab + st->bonds_off);
  const int d = st->d;
  for (int x = 0; x < count; ++x) {
    ImportEntry& e = ent[x];
    const int i = e.site;
    pool_free_now(slab, st, (uint64_t)sites[i].off, sites[i].cls);
    int c;
    uint64_t o = pool_alloc(slab, st, (uint64_t)e.chl * d * e.chr * 8, &c);
    if (!o) return;
    sites[i].off = (int64_t)o; sites[i].chl = e.chl; sites[i].chr = e.chr; sites[i].cls = c;
    e.dst_off = (int64_t)o;
    for (int side = 0; side < 2; ++side) {
      const int len = side == 0 ? e.resetL : e.resetR;
      const int b = side == 0 ? i : i + 1;  // bond index + 1
      if (len <= 0) continue;
      pool_free_now(slab, st, (uint64_t)bonds[b].off, bonds[b].cls);
      uint64_t ol = pool_alloc(slab, st, (uint64_t)len * 4, &c);
      if (!ol) return;
      bonds[b].off = (int64_t)ol; bonds[b].len = len; bonds[b].cls = c;
      if (side == 0) e.lamL_off = (int64_t)ol; else e.lamR_off = (int64_t)ol;
    }
  }
}

__global__ void k_import_scatter(uint8_t* slab, const ImportEntry* ent, const float2* src, int d) {
  const ImportEntry e = ent[blockIdx.x];
  if (!e.dst_off) return;
  float2* dst = reinterpret_cast<float2*>(slab + e.dst_off);
  const float2* s = src + e.src_elem;
  const int64_t cnt = (int64_t)e.chl * d * e.chr;
  for (int64_t x = threadIdx.x; x < cnt; x += blockDim.x) dst[x] = s[x];
  if (e.lamL_off)
    for (int x = threadIdx.x; x < e.resetL; x += blockDim.x) reinterpret_cast<float*>(slab + e.lamL_off)[x] = 1.f;
  if (e.lamR_off)
    for (int x = threadIdx.x; x < e.resetR; x += blockDim.x) reinterpret_cast<float*>(slab + e.lamR_off)[x] = 1.f;
}

}  // namespace

void launch_import(uint8_t* slab, DevState* st, ImportEntry* d_ent, int count, const float2* src, int d,
                   cudaStream_t s) {
  if (count <= 0) return;
  k_import_alloc<<<1, 1, 0, s>>>(slab, st, d_ent, count);
  k_import_scatter<<<count, 256, 0, s>>>(slab, d_ent, src, d);
}

void launch_select(GateDesc* d_desc, int G, uint8_t* slab, DevState* st, Record* d_rec, int parallel, cudaStream_t s) {
  if (G <= 0) return;
  if (parallel)
    k_select_parallel<<<(G + 7) / 8, 256, 0, s>>>(d_desc, G, slab, st);
  else
    k_select_sequential<<<1, 32, 0, s>>>(d_desc, G, slab, st);
  const size_t smem = (size_t)3 * kChunk * 8 + (size_t)3 * kChunk * 4 + (size_t)kChunk * 8 + (size_t)kChunk * 8 +
                      (size_t)4 * kChunk * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_commit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_commit<<<1, kCommitThreads, smem, s>>>(d_desc, G, slab, st, d_rec);
}
void launch_pool_alloc(uint8_t* slab, DevState* st, uint64_t bytes, int64_t* d_out, cudaStream_t s) {
  k_pool_alloc<<<1, 1, 0, s>>>(slab, st, bytes, d_out);
}
void launch_pool_free(uint8_t* slab, DevState* st, int64_t off, int cls, cudaStream_t s) {
  k_pool_free<<<1, 1, 0, s>>>(slab, st, off, cls);
}
void launch_gate1(uint8_t* slab, DevState* st, int site, int d, const float2* d_u, cudaStream_t s) {
  if (d == 2) k_gate1<2><<<64, 256, 0, s>>>(slab, st, site, d_u);
  else k_gate1<4><<<64, 256, 0, s>>>(slab, st, site, d_u);
}

}  // namespace eamps
