// sort_tails.cuh -- step a3: singular values "in decreasing order"
// and the tail weights T_k = sum_{j>=k} sigma_j^2 that the truncation fidelities E10/E11 need
// ("depends only on the actual truncated singular values").
// CTA-wide bitonic sort of (sigma^2, index) in shared memory (descending; ties: lower index
// first), then a deterministic FP64 suffix scan (tails summed from the small end so that
// 1 - t ~ 1e-5 budgets keep their significant digits).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace eamps {

// keys[npow2], idx[npow2] in shared memory; entries >= n are padding (key -1).
__device__ inline void cta_sort_desc(double* keys, int32_t* idx, int npow2) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int size = 2; size <= npow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < npow2 / 2; i += nt) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool desc_block = ((lo & size) == 0);  // descending overall
        double ka = keys[lo], kb = keys[hi];
        int32_t ia = idx[lo], ib = idx[hi];
        // "a before b" in descending order with ties broken by lower index
        bool a_first = (ka > kb) || (ka == kb && ia < ib);
        bool swap = desc_block ? !a_first : a_first;
        if (swap) {
          keys[lo] = kb; keys[hi] = ka;
          idx[lo] = ib; idx[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
}

// sorted keys (n) -> T (n+1): T[k] = sum_{j>=k} keys[j]; deterministic chunked suffix scan.
// `part` is scratch shared memory of blockDim.x doubles.
__device__ inline void cta_tails(const double* keys, int n, double* T_out /*global*/, double* part) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int chunk = (n + nt - 1) / nt;
  const int b = tid * chunk, e = min(n, b + chunk);
  double s = 0.0;
  for (int j = e - 1; j >= b; --j) s += keys[j];
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    double acc = 0.0;
    for (int t = nt - 1; t >= 0; --t) {
      double v = part[t];
      part[t] = acc;  // exclusive suffix: sum of chunks after t
      acc += v;
    }
  }
  __syncthreads();
  double acc = part[tid];
  for (int j = e - 1; j >= b; --j) {
    acc += keys[j];
    T_out[j] = acc;
  }
  if (tid == 0) T_out[n] = 0.0;
}

}  // namespace eamps
