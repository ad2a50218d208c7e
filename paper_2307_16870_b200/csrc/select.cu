// select.cu -- step a4: target, rank selection and ledger, plus the device-side
// pool allocator of the site store (north-star: "a per-site HBM tensor store with variable chi
// and a device-side pool allocator").
//
// One warp walks the wave's gates in canonical order (ascending site; reading 5):
//   log t_j  (E14; strategies PAPER.md:153/158 in log space, DESIGN reading 6)
//     naive   : log F_min / n
//     global  : min(0, (log F_min - log E) / R)                R = n - j
//     nearest : min(0, log F_min - log E - (R - 1) log F_min / n)
//     fixed   : log f_fixed (config-2 microbench)
//   tau = 1 - t (pure / ratio) or 1 - t^2 (wang)      (E10/E11 readings 1-2)
//   k = min{k >= 1 : T_k <= tau P}  ("as close to but not lower than f_t")
//       -- a 32-ary warp search over the non-increasing tails T
//   k <= min(m, n); k > chi_cap -> k = chi_cap, guarantee lost
//   f = 1 - T_k/P (pure/ratio) or sqrt(1 - T_k/P) (wang); log E += log f   (E12)
// then frees the old blocks of B_i, B_{i+1}, lambda_i (deferred to the next launch, when the
// reabsorb that reads the workspace -- never the old blocks -- has finished) and allocates the
// new ones from power-of-two size classes (free lists threaded through the free blocks + bump).
#include "eamps_internal.cuh"

namespace eamps {

namespace {

__device__ uint64_t pool_alloc(uint8_t* slab, DevState* st, uint64_t bytes, int* cls_out) {
  DevPool& P = st->pool;
  int c = size_class(bytes);
  *cls_out = c;
  uint64_t off = P.free_head[c];
  if (off) {
    P.free_head[c] = *reinterpret_cast<uint64_t*>(slab + off);
    return off;
  }
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
  *reinterpret_cast<uint64_t*>(slab + off) = st->pool.free_head[cls];
  st->pool.free_head[cls] = off;
}

__device__ void pool_defer(uint8_t* slab, DevState* st, uint64_t off, int cls) {
  if (!off) return;
  DevPool& P = st->pool;
  int64_t* pend = reinterpret_cast<int64_t*>(slab + P.pending_off);
  if (P.npending < P.pending_cap) {
    pend[2 * P.npending] = (int64_t)off;
    pend[2 * P.npending + 1] = cls;
    ++P.npending;
  } else {
    if (st->led.error == 0) st->led.error = -3;
  }
}

__device__ double target_log(const DevLedger& L, bool* bad) {
  *bad = false;
  double lt;
  if (L.strategy == 3) {
    lt = L.log_ffixed;
  } else {
    if (L.j >= L.n_planned) { *bad = true; return 0.0; }
    double R = (double)(L.n_planned - L.j);
    if (L.strategy == 0) lt = L.log_fmin / (double)L.n_planned;
    else if (L.strategy == 2) lt = (L.log_fmin - L.logE) / R;
    else lt = L.log_fmin - L.logE - (R - 1.0) * L.log_fmin / (double)L.n_planned;
  }
  return lt < 0.0 ? lt : 0.0;
}

__global__ void k_select(GateDesc* desc, int G, uint8_t* slab, DevState* st, Record* rec) {
  const int lane = threadIdx.x;
  if (lane == 0) {
    DevPool& P = st->pool;
    const int64_t* pend = reinterpret_cast<const int64_t*>(slab + P.pending_off);
    for (int64_t x = 0; x < P.npending; ++x) pool_free_now(slab, st, (uint64_t)pend[2 * x], (int)pend[2 * x + 1]);
    P.npending = 0;
  }
  __syncwarp();
  SiteEntry* sites = reinterpret_cast<SiteEntry*>(slab + st->sites_off);
  BondEntry* bonds = reinterpret_cast<BondEntry*>(slab + st->bonds_off);
  const int d = st->d;
  for (int g = 0; g < G; ++g) {
    GateDesc& gd = desc[g];
    if (st->led.error != 0) {  // sticky error: leave the rest of the wave untouched
      if (lane == 0) gd.k = 0;
      continue;
    }
    const double* T = reinterpret_cast<const double*>(slab + gd.ws_T);
    const double* s2 = reinterpret_cast<const double*>(slab + gd.ws_sig2);
    const int n = gd.n;
    const double P = T[0];
    bool bad = false;
    const double lt = target_log(st->led, &bad);
    if (bad) {
      if (lane == 0) { st->led.error = -8; gd.k = 0; }
      __syncwarp();
      continue;
    }
    const int rule = st->led.rule;
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
    if (st->led.chi_cap > 0 && k > st->led.chi_cap) { k = st->led.chi_cap; capped = 1; }
    // nu^2 = kept weight, deterministic lane-strided FP64 sum + xor tree
    double kw = 0.0;
    for (int j = lane; j < k; j += 32) kw += s2[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kw += __shfl_xor_sync(0xffffffffu, kw, o);
    if (lane == 0) {
      const double r = P > 0.0 ? T[k] / P : 0.0;
      double f, dl;
      if (rule == 1) { f = sqrt(1.0 - r); dl = 0.5 * log1p(-r); }
      else { f = 1.0 - r; dl = log1p(-r); }
      DevLedger& L = st->led;
      Record& R = rec[g];
      R.gate_index = L.j; R.bond = gd.site; R.chi_before = gd.mid; R.chi_after = k; R.capped = capped;
      R.target_f = exp(lt); R.achieved_f = f; R.discarded_weight = r;
      L.logE += dl;
      L.j += 1;
      if (capped) L.guarantee = 0;
      // site store: defer-free the old blocks, allocate the new ones
      const int i = gd.site;
      pool_defer(slab, st, (uint64_t)sites[i].off, sites[i].cls);
      pool_defer(slab, st, (uint64_t)sites[i + 1].off, sites[i + 1].cls);
      pool_defer(slab, st, (uint64_t)bonds[i + 1].off, bonds[i + 1].cls);
      int cL, cR, cLam;
      uint64_t oL = pool_alloc(slab, st, (uint64_t)gd.l * d * k * 8, &cL);
      uint64_t oR = pool_alloc(slab, st, (uint64_t)k * d * gd.r * 8, &cR);
      uint64_t oLam = pool_alloc(slab, st, (uint64_t)k * 4, &cLam);
      if (!oL || !oR || !oLam) {
        gd.k = 0;
      } else {
        sites[i].off = (int64_t)oL; sites[i].chr = k; sites[i].cls = cL;
        sites[i + 1].off = (int64_t)oR; sites[i + 1].chl = k; sites[i + 1].cls = cR;
        bonds[i + 1].off = (int64_t)oLam; bonds[i + 1].len = k; bonds[i + 1].cls = cLam;
        gd.k = k; gd.capped = capped;
        gd.off_newL = (int64_t)oL; gd.off_newR = (int64_t)oR; gd.off_newLam = (int64_t)oLam;
        gd.nu = sqrt(kw); gd.f = f; gd.t = exp(lt);
      }
    }
    __syncwarp();
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

void launch_select(GateDesc* d_desc, int G, uint8_t* slab, DevState* st, Record* d_rec, cudaStream_t s) {
  if (G <= 0) return;
  k_select<<<1, 32, 0, s>>>(d_desc, G, slab, st, d_rec);
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
