// pool.cuh -- the device-side pool allocator of the site store, batched over one CTA.
//
// Blocks are size classes of 2^k and 1.5 x 2^k bytes (>= 256 B, class_bytes) carved from the slab: per-class free stacks plus a bump
// pointer. A batch of requests (in canonical order) is resolved in parallel and
// deterministically: the rank of a request among the batch's requests of its class comes from a
// CTA-wide exclusive scan; the first cnt[c] requests of class c pop the stack, the rest take bump
// space whose offsets are an exclusive scan of their sizes in canonical order. Frees push in
// canonical order the same way. No global memory load sits on a sequential dependency chain.
#pragma once
#include "eamps_internal.cuh"

namespace eamps {

__host__ __device__ inline int size_class_fast(uint64_t bytes) {
#ifdef __CUDA_ARCH__
  if (bytes <= 256) return kMinClass;
  const int k = 64 - __clzll(bytes - 1);      // smallest k with 2^k >= bytes (k >= 9)
  if (k - 1 >= 9 && bytes <= (3ull << (k - 2))) return 2 * k - 1;
  return 2 * k;
#else
  return size_class(bytes);
#endif
}

// CTA-wide exclusive scan of one value per thread (blockDim.x <= 1024); returns the exclusive
// prefix, *total = sum over the CTA. `ws` = shared scratch of 32 T.
template <typename T>
__device__ inline T cta_exclusive_scan(T v, T* ws, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nw ? ws[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) ws[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const T before = warp > 0 ? ws[warp - 1] : T(0);
  *total = ws[nw - 1];
  __syncthreads();
  return before + x - v;
}

// Scan of `n` items held in shared memory, ITEMS per thread contiguous: out[i] = sum_{j<i} in[j].
template <typename T>
__device__ inline T cta_scan_array(const T* in, T* out, int n, T* ws) {
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int b = threadIdx.x * per, e = min(n, b + per);
  T s = T(0);
  for (int i = b; i < e; ++i) s += in[i];
  T tot;
  T pre = cta_exclusive_scan<T>(s, ws, &tot);
  for (int i = b; i < e; ++i) {
    T v = in[i];
    out[i] = pre;
    pre += v;
  }
  __syncthreads();
  return tot;
}

struct PoolBatch {  // shared-memory scratch for a batch of up to `cap` requests
  int32_t* cls;     // [cap]
  int32_t* rank;    // [cap]  rank within class / scan scratch
  uint64_t* val;    // [cap]  in: bytes or offset;  out: offset
  uint64_t* tmp;    // [cap]
  int32_t* cnt;     // [kMaxClasses] shared copy of the stack depths
  int32_t* iws;     // [32]
  uint64_t* uws;    // [32]
};

// Rank of each request within its class (requests with cls < 0 are ignored): one scan per class
// present in the batch (typically 2-3 classes).
__device__ inline void batch_class_ranks(PoolBatch& B, int n, int32_t* present /*[kMaxClasses] shared*/) {
  for (int c = threadIdx.x; c < kMaxClasses; c += blockDim.x) present[c] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (B.cls[i] >= 0) present[B.cls[i]] = 1;
  __syncthreads();
  for (int c = 0; c < kMaxClasses; ++c) {
    if (!present[c]) continue;
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int b = threadIdx.x * per, e = min(n, b + per);
    int32_t s = 0;
    for (int i = b; i < e; ++i) s += (B.cls[i] == c);
    int32_t tot;
    int32_t pre = cta_exclusive_scan<int32_t>(s, B.iws, &tot);
    for (int i = b; i < e; ++i)
      if (B.cls[i] == c) B.rank[i] = pre++;
    present[c] = tot;  // count of class c in the batch (same value written by every thread)
    __syncthreads();
  }
}

// Free a batch: val[i] = offset (0 = skip), cls[i] = class. Stack depths in B.cnt are updated.
__device__ inline bool pool_batch_free(PoolBatch& B, int n, uint8_t* slab, const DevPool& P, int32_t* present) {
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (!B.val[i]) B.cls[i] = -1;
  __syncthreads();
  batch_class_ranks(B, n, present);
  int64_t* stk = reinterpret_cast<int64_t*>(slab + P.stack_off);
  bool ok = true;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int c = B.cls[i];
    if (c < 0) continue;
    const int64_t slot = (int64_t)B.cnt[c] + B.rank[i];
    if (slot >= P.stack_cap) { ok = false; continue; }
    stk[(int64_t)c * P.stack_cap + slot] = (int64_t)B.val[i];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < kMaxClasses; c += blockDim.x) B.cnt[c] += present[c];
  __syncthreads();
  return __syncthreads_and(ok) != 0;
}

// Allocate a batch: in val[i] = bytes (0 = no request), out val[i] = slab offset.
// *bump is advanced; returns false if the ceiling would be crossed (nothing is then allocated).
__device__ inline bool pool_batch_alloc(PoolBatch& B, int n, uint8_t* slab, const DevPool& P, uint64_t* bump,
                                        uint64_t ceiling, int32_t* present) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) B.cls[i] = B.val[i] ? size_class_fast(B.val[i]) : -1;
  __syncthreads();
  batch_class_ranks(B, n, present);
  // pops for the first cnt[c] requests of each class, bump sizes for the rest
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int c = B.cls[i];
    B.tmp[i] = (c >= 0 && B.rank[i] >= B.cnt[c]) ? class_bytes(c) : 0ull;
  }
  __syncthreads();
  const uint64_t total = cta_scan_array<uint64_t>(B.tmp, B.tmp, n, B.uws);  // exclusive offsets in tmp
  const uint64_t b0 = (*bump + 255ull) & ~255ull;
  if (b0 + total > ceiling) return false;
  const int64_t* stk = reinterpret_cast<const int64_t*>(slab + P.stack_off);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int c = B.cls[i];
    if (c < 0) { B.val[i] = 0; continue; }
    if (B.rank[i] < B.cnt[c]) B.val[i] = (uint64_t)stk[(int64_t)c * P.stack_cap + (B.cnt[c] - 1 - B.rank[i])];
    else B.val[i] = b0 + B.tmp[i];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < kMaxClasses; c += blockDim.x) B.cnt[c] -= min(B.cnt[c], present[c]);
  if (threadIdx.x == 0) *bump = b0 + total;
  __syncthreads();
  return true;
}

}  // namespace eamps
