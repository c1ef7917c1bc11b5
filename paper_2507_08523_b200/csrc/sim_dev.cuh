// sim_dev.cuh — exact candidate ordering and warp top-k merge shared by the two a1-a2 kernels
// (k_sim_topk: per-query pool scan for small pools; k_sim_inv: inverted-index accumulation for
// large pools).  Scores are exact fractions num / den compared by cross-multiplication (Z6).
#pragma once
#include "il_internal.cuh"

namespace il {

struct Cand {
  uint64_t num, den;
  uint32_t idx;
};
__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {   // a ranks before b
  const uint64_t l = a.num * b.den, r = b.num * a.den;                   // < 2^48: exact in u64
  return l > r || (l == r && a.idx < b.idx);
}
// k rounds of warp argmax over the lanes' sorted lists (get(q) = the lane's q-th best, n of
// them); the winning lane pops its head.  `better` is a strict total order (index breaks score
// ties), so the result does not depend on lane order.  Picks go to out[0..n) best first.
template <class Get>
__device__ __forceinline__ uint32_t warp_merge(Get get, uint32_t n, uint32_t k, uint32_t lane, Cand* out) {
  uint32_t head = 0, npick = 0;
  for (uint32_t r = 0; r < k; ++r) {
    Cand w;
    uint32_t wl = NONE32;
    if (head < n) { w = get(head); wl = lane; } else { w.num = 0; w.den = 1; w.idx = NONE32; }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      Cand o_;
      o_.num = __shfl_xor_sync(~0u, w.num, o); o_.den = __shfl_xor_sync(~0u, w.den, o);
      o_.idx = __shfl_xor_sync(~0u, w.idx, o);
      const uint32_t ol = __shfl_xor_sync(~0u, wl, o);
      if (ol != NONE32 && (wl == NONE32 || better(o_, w))) { w = o_; wl = ol; }
    }
    if (wl == NONE32) break;                             // (uniform: every lane holds the winner)
    if (lane == 0) out[r] = w;
    if (lane == wl) ++head;
    ++npick;
  }
  return npick;
}
}  // namespace il
