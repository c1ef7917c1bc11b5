// attn_common.cuh — suffix-row bookkeeping shared by the K/V append, the attention kernels
// and the synthetic Q/K/V helper.
#pragma once
#include <cuda_bf16.h>

#include "il_internal.cuh"

namespace il {

// request owning suffix row r: largest i with cu_q[i] <= r (cu_q non-decreasing, B+1 entries)
__device__ __forceinline__ uint32_t row_owner(const int32_t* __restrict__ cu_q, uint32_t B, uint32_t r) {
  uint32_t lo = 0, hi = B;          // invariant: cu_q[lo] <= r < cu_q[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((uint32_t)cu_q[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

}  // namespace il
