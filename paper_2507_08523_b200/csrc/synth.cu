// synth.cu — il_synth_qkv (bench / test helper, not the method): bf16 Q, K, V of suffix rows
// from the counter-based generator of DESIGN.md Z28:
//   u = mix(mix(mix(seed_t ^ token) ^ position) ^ (head * 256 + dim)),
//   x = (int(u >> 40) - 2^23) / 2^23 * scale, rounded to bf16 (RNE),
// seed_t = mix((seed << 8) ^ salt), salt = 'Q' / 'K' / 'V'.
#include <cuda_bf16.h>

#include "attn_common.cuh"
#include "il_internal.cuh"

namespace il {

__device__ __forceinline__ __nv_bfloat16 synth_val(uint64_t seed_t, uint32_t tok, uint32_t pos, uint32_t hd, float mul) {
  const uint64_t u = mix64(mix64(mix64(seed_t ^ (uint64_t)tok) ^ (uint64_t)pos) ^ (uint64_t)hd);
  const float x = (float)((int32_t)(u >> 40) - (1 << 23)) * mul;
  return __float2bfloat16_rn(x);
}

__global__ void __launch_bounds__(256) k_synth(Ctx c, uint32_t B, const uint32_t* __restrict__ prompt_tok,
                                               const int32_t* __restrict__ cu_q, const int32_t* __restrict__ prefix_len,
                                               uint64_t sq, uint64_t sk, uint64_t sv, float qmul, float kvmul,
                                               __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ kn,
                                               __nv_bfloat16* __restrict__ vn) {
  const uint32_t Hq = c.cfg.n_q_heads, Hkv = c.cfg.n_kv_heads, d = c.cfg.head_dim;
  const uint32_t total = (uint32_t)cu_q[B];
  const uint32_t per_row = (Hq + 2 * Hkv) * d;
  for (uint32_t r = blockIdx.x; r < total; r += gridDim.x) {
    const uint32_t i = row_owner(cu_q, B, r);
    const uint32_t pos = (uint32_t)prefix_len[i] + r - (uint32_t)cu_q[i];
    const uint32_t tok = prompt_tok[(size_t)i * c.cfg.max_prompt_tokens + pos];
    for (uint32_t e = threadIdx.x; e < per_row; e += blockDim.x) {
      const uint32_t h = e / d, x = e % d;
      if (h < Hq) {
        q[((size_t)r * Hq + h) * d + x] = synth_val(sq, tok, pos, h * 256 + x, qmul);
      } else if (h < Hq + Hkv) {
        const uint32_t hk = h - Hq;
        kn[((size_t)r * Hkv + hk) * d + x] = synth_val(sk, tok, pos, hk * 256 + x, kvmul);
      } else {
        const uint32_t hv = h - Hq - Hkv;
        vn[((size_t)r * Hkv + hv) * d + x] = synth_val(sv, tok, pos, hv * 256 + x, kvmul);
      }
    }
  }
}

}  // namespace il

using namespace il;

extern "C" il_status il_synth_qkv(il_ctx* c, uint32_t B, const uint32_t* prompt_tok, const int32_t* cu_q,
                                  const int32_t* prefix_len, uint64_t seed, float q_scale, il_bf16* q,
                                  il_bf16* k_new, il_bf16* v_new, il_stream s) {
  if (B == 0) return IL_OK;
  auto tseed = [&](uint64_t salt) { return mix64((seed << 8) ^ salt); };
  const float unit = 1.0f / 8388608.0f;
  k_synth<<<c->num_sms * 16, 256, 0, (cudaStream_t)s>>>(*c, B, prompt_tok, cu_q, prefix_len, tseed(0x51),
                                                        tseed(0x4B), tseed(0x56), q_scale * unit, unit,
                                                        (__nv_bfloat16*)q, (__nv_bfloat16*)k_new,
                                                        (__nv_bfloat16*)v_new);
  IL_LAUNCH_CHECK("k_synth");
  c->launches += 1;
  return IL_OK;
}
