// attn_sm100.cuh — tcgen05/TMA prefill attention (placeholder until the kernel lands).
#pragma once
#include "il_internal.cuh"

namespace il {
static inline bool attn_sm100_supported(const Ctx*) { return false; }
static inline il_status attn_sm100_launch(Ctx*, uint32_t, const int32_t*, const int32_t*, const int32_t*,
                                          const il_bf16*, il_bf16*, il_bf16*, il_bf16*, float*, float,
                                          cudaStream_t) {
  return IL_ERR_INTERNAL;
}
}  // namespace il
