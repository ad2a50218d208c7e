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
#include "pool.cuh"

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
  uint64_t sz = class_bytes(c);
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
constexpr int kChunk = 1024;  // gates per shared-memory chunk (3 pool requests each)
constexpr int kReq = 3 * kChunk;

struct CommitSmem {
  int32_t cls[kReq], rank[kReq];
  uint64_t val[kReq], tmp[kReq];
  double gdl[kChunk];
  int32_t gk[kChunk], gl[kChunk], gr[kChunk], gc[kChunk], ord[kChunk];
  int32_t cnt[kMaxClasses], present[kMaxClasses], iws[32];
  uint64_t uws[32];
  uint64_t bump;
  int err;
};

__device__ inline PoolBatch make_batch(CommitSmem& S) {
  return PoolBatch{S.cls, S.rank, S.val, S.tmp, S.cnt, S.iws, S.uws};
}

__global__ void __launch_bounds__(kCommitThreads) k_commit(GateDesc* desc, int G, uint8_t* slab, DevState* st,
                                                            Record* rec) {
  extern __shared__ __align__(16) uint8_t sm[];
  CommitSmem& S = *reinterpret_cast<CommitSmem*>(sm);
  PoolBatch B = make_batch(S);
  const int tid = threadIdx.x;
  DevPool& P = st->pool;
  int64_t* pend = reinterpret_cast<int64_t*>(slab + P.pending_off);
  SiteEntry* sites = reinterpret_cast<SiteEntry*>(slab + st->sites_off);
  BondEntry* bonds = reinterpret_cast<BondEntry*>(slab + st->bonds_off);
  const int d = st->d;
  if (tid < kMaxClasses) S.cnt[tid] = P.count[tid];
  if (tid == 0) { S.bump = P.bump; S.err = st->led.error; }
  __syncthreads();

  // A. release the previous wave's deferred frees onto the class stacks (canonical order)
  const int64_t npend = P.npending;
  for (int64_t c0 = 0; c0 < npend; c0 += kReq) {
    const int cn = (int)min((int64_t)kReq, npend - c0);
    for (int i = tid; i < cn; i += kCommitThreads) {
      S.val[i] = (uint64_t)pend[2 * (c0 + i)];
      S.cls[i] = (int32_t)pend[2 * (c0 + i) + 1];
    }
    __syncthreads();
    if (!pool_batch_free(B, cn, slab, P, S.present) && tid == 0) S.err = -3;
  }
  __syncthreads();

  // B. per chunk of gates: ledger, batched allocation, table updates, records
  double logE = st->led.logE;   // meaningful in thread 0 only
  int64_t j0 = st->led.j;
  int guarantee = st->led.guarantee;
  for (int g0 = 0; g0 < G; g0 += kChunk) {
    const int gn = min(kChunk, G - g0);
    for (int x = tid; x < gn; x += kCommitThreads) {
      const GateDesc& gd = desc[g0 + x];
      S.gk[x] = gd.k; S.gl[x] = gd.l; S.gr[x] = gd.r; S.gc[x] = gd.capped; S.gdl[x] = gd.dlogE;
    }
    __syncthreads();
    const bool err0 = S.err != 0;
    // ledger indices = exclusive count of valid gates (canonical order)
    {
      const int per = (gn + kCommitThreads - 1) / kCommitThreads;
      const int b = tid * per, e = min(gn, b + per);
      int32_t cnt = 0;
      for (int x = b; x < e; ++x) cnt += (S.gk[x] > 0 && !err0);
      int32_t tot;
      int32_t pre = cta_exclusive_scan<int32_t>(cnt, S.iws, &tot);
      for (int x = b; x < e; ++x) S.ord[x] = (S.gk[x] > 0 && !err0) ? pre++ : -1;
      // the chunk's ledger update, committed only if its allocations succeed (a failed chunk's gates
      // are dropped with k = 0 and must not count)
      double logE_c = logE;
      int guarantee_c = guarantee;
      if (tid == 0) {
        for (int x = 0; x < gn; ++x)
          if (S.ord[x] >= 0) {  // sequential in canonical order: the same summation as the sequential selector
            logE_c += S.gdl[x];
            if (S.gc[x]) guarantee_c = 0;
          }
      }
      __syncthreads();
      // requests: new B_i, new B_{i+1}, new lambda_i
      for (int x = tid; x < gn; x += kCommitThreads) {
        const int k = S.gk[x];
        const bool v = S.ord[x] >= 0;
        S.val[3 * x] = v ? (uint64_t)S.gl[x] * d * k * 8 : 0;
        S.val[3 * x + 1] = v ? (uint64_t)k * d * S.gr[x] * 8 : 0;
        S.val[3 * x + 2] = v ? (uint64_t)k * 4 : 0;
      }
      __syncthreads();
      const bool ok = pool_batch_alloc(B, 3 * gn, slab, P, &S.bump, P.ceiling, S.present);
      if (!ok && tid == 0) S.err = -3;
      if (ok) {
        logE = logE_c;
        guarantee = guarantee_c;
      }
      __syncthreads();
      for (int x = tid; x < gn; x += kCommitThreads) {
        GateDesc& gd = desc[g0 + x];
        const int64_t pb = 3 * (int64_t)(g0 + x);
        if (!ok || S.ord[x] < 0) {
          gd.k = 0;
          pend[2 * pb] = pend[2 * pb + 2] = pend[2 * pb + 4] = 0;
          continue;
        }
        const int i = gd.site, k = S.gk[x];
        // deferred frees of the old blocks (released at the next commit)
        pend[2 * pb] = sites[i].off; pend[2 * pb + 1] = sites[i].cls;
        pend[2 * pb + 2] = sites[i + 1].off; pend[2 * pb + 3] = sites[i + 1].cls;
        pend[2 * pb + 4] = bonds[i + 1].off; pend[2 * pb + 5] = bonds[i + 1].cls;
        const uint64_t oL = S.val[3 * x], oR = S.val[3 * x + 1], oLam = S.val[3 * x + 2];
        sites[i].off = (int64_t)oL; sites[i].chr = k; sites[i].cls = S.cls[3 * x];
        sites[i + 1].off = (int64_t)oR; sites[i + 1].chl = k; sites[i + 1].cls = S.cls[3 * x + 1];
        bonds[i + 1].off = (int64_t)oLam; bonds[i + 1].len = k; bonds[i + 1].cls = S.cls[3 * x + 2];
        gd.off_newL = (int64_t)oL; gd.off_newR = (int64_t)oR; gd.off_newLam = (int64_t)oLam;
        Record& R = rec[g0 + x];
        R.gate_index = j0 + S.ord[x]; R.bond = i; R.chi_before = gd.mid; R.chi_after = k; R.capped = gd.capped;
        R.target_f = gd.t; R.achieved_f = gd.f; R.discarded_weight = gd.disc;
      }
      if (ok) j0 += tot;
      __syncthreads();
    }
  }
  if (tid < kMaxClasses) P.count[tid] = S.cnt[tid];
  if (tid == 0) {
    P.bump = S.bump;
    P.npending = 3 * (int64_t)G;
    st->led.logE = logE;
    st->led.j = j0;
    st->led.guarantee = guarantee;
    if (S.err && !st->led.error) st->led.error = S.err;
  }
}

// Bulk import: free the replaced blocks, allocate the new ones (one batch each), fill tables.
__global__ void __launch_bounds__(kCommitThreads) k_import_batch(uint8_t* slab, DevState* st, ImportEntry* ent,
                                                                  int count) {
  extern __shared__ __align__(16) uint8_t sm[];
  CommitSmem& S = *reinterpret_cast<CommitSmem*>(sm);
  PoolBatch B = make_batch(S);
  const int tid = threadIdx.x;
  DevPool& P = st->pool;
  SiteEntry* sites = reinterpret_cast<SiteEntry*>(slab + st->sites_off);
  BondEntry* bonds = reinterpret_cast<BondEntry*>(slab + st->bonds_off);
  const int d = st->d;
  if (tid < kMaxClasses) S.cnt[tid] = P.count[tid];
  if (tid == 0) { S.bump = P.bump; S.err = st->led.error; }
  __syncthreads();
  for (int e0 = 0; e0 < count; e0 += kChunk) {
    const int en = min(kChunk, count - e0);
    // frees of the replaced site blocks and reset lambdas
    for (int x = tid; x < en; x += kCommitThreads) {
      const ImportEntry& e = ent[e0 + x];
      S.val[3 * x] = (uint64_t)sites[e.site].off; S.cls[3 * x] = sites[e.site].cls;
      S.val[3 * x + 1] = e.resetL > 0 ? (uint64_t)bonds[e.site].off : 0; S.cls[3 * x + 1] = bonds[e.site].cls;
      S.val[3 * x + 2] = e.resetR > 0 ? (uint64_t)bonds[e.site + 1].off : 0; S.cls[3 * x + 2] = bonds[e.site + 1].cls;
    }
    __syncthreads();
    if (!pool_batch_free(B, 3 * en, slab, P, S.present) && tid == 0) S.err = -3;
    for (int x = tid; x < en; x += kCommitThreads) {
      const ImportEntry& e = ent[e0 + x];
      S.val[3 * x] = (uint64_t)e.chl * d * e.chr * 8;
      S.val[3 * x + 1] = e.resetL > 0 ? (uint64_t)e.resetL * 4 : 0;
      S.val[3 * x + 2] = e.resetR > 0 ? (uint64_t)e.resetR * 4 : 0;
    }
    __syncthreads();
    const bool ok = pool_batch_alloc(B, 3 * en, slab, P, &S.bump, P.ceiling, S.present);
    if (!ok) {
      if (tid == 0) S.err = -3;
      break;
    }
    for (int x = tid; x < en; x += kCommitThreads) {
      ImportEntry& e = ent[e0 + x];
      const int i = e.site;
      sites[i].off = (int64_t)S.val[3 * x]; sites[i].chl = e.chl; sites[i].chr = e.chr; sites[i].cls = S.cls[3 * x];
      e.dst_off = (int64_t)S.val[3 * x];
      if (e.resetL > 0) {
        bonds[i].off = (int64_t)S.val[3 * x + 1]; bonds[i].len = e.resetL; bonds[i].cls = S.cls[3 * x + 1];
        e.lamL_off = (int64_t)S.val[3 * x + 1];
      }
      if (e.resetR > 0) {
        bonds[i + 1].off = (int64_t)S.val[3 * x + 2]; bonds[i + 1].len = e.resetR; bonds[i + 1].cls = S.cls[3 * x + 2];
        e.lamR_off = (int64_t)S.val[3 * x + 2];
      }
    }
    __syncthreads();
  }
  if (tid < kMaxClasses) P.count[tid] = S.cnt[tid];
  if (tid == 0) {
    P.bump = S.bump;
    if (S.err && !st->led.error) st->led.error = S.err;
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

// the reverse of k_import_scatter: site x's tensor -> dst + dst_elem (16 B per thread and step
// when both ends are 16 B aligned: pool blocks are, the destination is when dst_elem is even)
__global__ void k_export_gather(const uint8_t* __restrict__ slab, const ExportEntry* __restrict__ ent,
                                float2* __restrict__ dst) {
  const ExportEntry e = ent[blockIdx.x];
  const float2* s = reinterpret_cast<const float2*>(slab + e.src_off);
  float2* o = dst + e.dst_elem;
  const int64_t stride = (int64_t)gridDim.y * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (((e.dst_elem | e.elems) & 1) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(s);
    float4* o4 = reinterpret_cast<float4*>(o);
    for (int64_t x = t0; x < e.elems / 2; x += stride) o4[x] = s4[x];
  } else {
    for (int64_t x = t0; x < e.elems; x += stride) o[x] = s[x];
  }
}

}  // namespace

void launch_export(const uint8_t* slab, const ExportEntry* d_ent, int count, int split, float2* dst, cudaStream_t s) {
  if (count <= 0) return;
  k_export_gather<<<dim3(count, split), 256, 0, s>>>(slab, d_ent, dst);
}

void launch_import(uint8_t* slab, DevState* st, ImportEntry* d_ent, int count, const float2* src, int d,
                   cudaStream_t s) {
  if (count <= 0) return;
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(k_import_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CommitSmem));
  }
  k_import_batch<<<1, kCommitThreads, sizeof(CommitSmem), s>>>(slab, st, d_ent, count);
  k_import_scatter<<<count, 256, 0, s>>>(slab, d_ent, src, d);
}

void launch_select(GateDesc* d_desc, int G, uint8_t* slab, DevState* st, Record* d_rec, int parallel, cudaStream_t s) {
  if (G <= 0) return;
  if (parallel)
    k_select_parallel<<<(G + 7) / 8, 256, 0, s>>>(d_desc, G, slab, st);
  else
    k_select_sequential<<<1, 32, 0, s>>>(d_desc, G, slab, st);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(k_commit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(CommitSmem));
  }
  k_commit<<<1, kCommitThreads, sizeof(CommitSmem), s>>>(d_desc, G, slab, st, d_rec);
}
// a layer of single-site gates (disjoint sites; NEXT-3's one-qubit layers): gate g acts on
// sites[g] with U = Us + g D^2. grid (blocks, count).
template <int D>
__global__ void k_gate1_layer(uint8_t* slab, const DevState* st, const int32_t* __restrict__ sites,
                              const float2* __restrict__ Us) {
  const int g = blockIdx.y;
  const SiteEntry e = reinterpret_cast<const SiteEntry*>(slab + st->sites_off)[sites[g]];
  const float2* U = Us + (int64_t)g * D * D;
  float2* B = reinterpret_cast<float2*>(slab + e.off);
  const int64_t tot = (int64_t)e.chl * e.chr;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = x / e.chr, c = x % e.chr;
    float2 in[D];
#pragma unroll
    for (int s = 0; s < D; ++s) in[s] = B[(a * D + s) * e.chr + c];
#pragma unroll
    for (int s = 0; s < D; ++s) {
      float2 o = make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < D; ++t) {
        const float2 u = U[s * D + t];
        o.x += u.x * in[t].x - u.y * in[t].y;
        o.y += u.x * in[t].y + u.y * in[t].x;
      }
      B[(a * D + s) * e.chr + c] = o;
    }
  }
}

void launch_gate1_layer(uint8_t* slab, DevState* st, int count, const int32_t* d_sites, const float2* d_us, int d,
                        cudaStream_t s) {
  if (count <= 0) return;
  const dim3 grid(16, count);
  if (d == 2) k_gate1_layer<2><<<grid, 256, 0, s>>>(slab, st, d_sites, d_us);
  else k_gate1_layer<4><<<grid, 256, 0, s>>>(slab, st, d_sites, d_us);
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
