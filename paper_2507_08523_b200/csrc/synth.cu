// synth.cu — il_synth_qkv (bench / test helper, not the method): bf16 Q, K, V of suffix rows
// from the counter-based generator of DESIGN.md Z28:
//   row key r = mix(mix(seed_t ^ token) ^ position)                     (64-bit, once per row)
//   v = fmix32((lo32(r) ^ e * 0x9E3779B9) + hi32(r)), e = head * 64 + dim / 4  (one per 4 dims)
//   u = byte (dim % 4) of v, f = 1 + u / 256 (built from bits), x = (f - 1.5) * (2 * scale)
//   in fp32 (no contraction) -- exact in bf16: (u - 128) / 128 * scale,
// seed_t = mix((seed << 8) ^ salt), salt = 'Q' / 'K' / 'V'.
#include <cuda_bf16.h>

#include "attn_common.cuh"
#include "il_internal.cuh"

namespace il {

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; return h ^ (h >> 16);
}
// the four elements (dims 4e .. 4e+3) of one mix, as two packed bf16 pairs.  (u - 128) / 256 * mul
// is formed as ((2^23 + u) - (2^23 + 128)) * (mul / 256): both differences are exact, and the one
// rounded product equals the generator's (f - 1.5) * mul with f = 1 + u / 256 (the same real number,
// mul / 256 exact); 2^23 + u is one byte permute of v into 0x4B0000uu.
__device__ __forceinline__ void synth_quad(uint64_t row_key, uint32_t e, float mul256, uint32_t& w0, uint32_t& w1) {
  const uint32_t v = fmix32(((uint32_t)row_key ^ (e * 0x9E3779B9u)) + (uint32_t)(row_key >> 32));
  uint32_t b[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)                           // {0x4B, 0x00, 0x00, byte j of v}
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(b[j]) : "r"(v), "r"(0x4B000000u), "r"(0x7650u | (uint32_t)j));
  float x[4];
#pragma unroll
  for (int j = 0; j < 4; j += 2)
    asm("{ .reg .b64 a, c, m; mov.b64 a, {%2, %3}; mov.b64 c, {%4, %4}; add.rn.f32x2 a, a, c;\n\t"
        "mov.b64 m, {%5, %5}; mul.rn.f32x2 a, a, m; mov.b64 {%0, %1}, a; }"
        : "=f"(x[j]), "=f"(x[j + 1]) : "f"(__uint_as_float(b[j])), "f"(__uint_as_float(b[j + 1])), "f"(-8388736.0f),
          "f"(mul256));
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w0) : "f"(x[1]), "f"(x[0]));   // low half = dim 4e
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(w1) : "f"(x[3]), "f"(x[2]));
}

// One warp per suffix row (grid-stride): the two (token, position) mixes are computed once per
// row and tensor; each group of 4 elements then costs one mix.  Lanes write 8 consecutive bf16 (16 B).
// PAGED: K and V go straight into the request's KV pages ([C][Hkv][16][d], page =
// block_table[i][pos / 16], slot pos % 16) -- the projection's epilogue writing the paged cache, so
// il_prefill_attn needs no separate append pass.
template <int D, bool PAGED>
__global__ void __launch_bounds__(256) k_synth(Ctx c, uint32_t B, const uint32_t* __restrict__ prompt_tok,
                                               const int32_t* __restrict__ cu_q, const int32_t* __restrict__ prefix_len,
                                               const int32_t* __restrict__ block_table,
                                               uint64_t sq, uint64_t sk, uint64_t sv, float qmul, float kvmul,
                                               __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ kn,
                                               __nv_bfloat16* __restrict__ vn, uint32_t h_begin, uint32_t h_end) {
  const uint32_t Hq = c.cfg.n_q_heads, Hkv = c.cfg.n_kv_heads;
  const uint32_t total = (uint32_t)cu_q[B];
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  constexpr uint32_t VPH = D / 8;                       // 16-byte vectors per head
  for (uint32_t r = gw; r < total; r += nw) {
    const uint32_t i = row_owner(cu_q, B, r);
    const uint32_t pos = (uint32_t)prefix_len[i] + r - (uint32_t)cu_q[i];
    const uint32_t tok = prompt_tok[(size_t)i * c.cfg.max_prompt_tokens + pos];
    const uint64_t kq = mix64(mix64(sq ^ (uint64_t)tok) ^ (uint64_t)pos);
    const uint64_t kk = mix64(mix64(sk ^ (uint64_t)tok) ^ (uint64_t)pos);
    const uint64_t kv = mix64(mix64(sv ^ (uint64_t)tok) ^ (uint64_t)pos);
    // head rows [h_begin, h_end) of Q | K | V, one 16-byte vector (8 dims) per lane and step; the
    // three tensors in separate loops (no per-vector branching: the destination of vector e of a
    // tensor is its row base + e * 8, with head = e / VPH)
    const size_t page_row = PAGED ? (size_t)(uint32_t)block_table[(size_t)i * c.max_blocks + pos / BS] * Hkv : 0;
    const size_t slot = PAGED ? (page_row * BS + pos % BS) * D : 0;
    auto quads = [&](uint64_t key, float mul256, uint32_t e) -> uint4 {
      const uint32_t hh = e / VPH, eg = hh * 64 + (e % VPH) * 2;   // generator index of the first 4 dims
      uint4 w;
      synth_quad(key, eg, mul256, w.x, w.y);
      synth_quad(key, eg + 1, mul256, w.z, w.w);
      return w;
    };
    if (h_begin < Hq) {
      uint4* dq = reinterpret_cast<uint4*>(q + (size_t)r * Hq * D);
      for (uint32_t e = h_begin * VPH + lane; e < min(h_end, Hq) * VPH; e += 32) dq[e] = quads(kq, qmul * (1.f / 256.f), e);
    }
    if (h_end > Hq) {
      const uint32_t nkv = Hkv * VPH;
      uint4* dk = reinterpret_cast<uint4*>(kn + (PAGED ? slot : (size_t)r * Hkv * D));
      uint4* dv = reinterpret_cast<uint4*>(vn + (PAGED ? slot : (size_t)r * Hkv * D));
      // paged: head hh of the row lives BS * D elements after head hh - 1 ([page][Hkv][16][d])
      const uint32_t hstride = PAGED ? BS * VPH : VPH;
      for (uint32_t e = lane; e < nkv; e += 32) {
        const uint32_t at = (e / VPH) * hstride + e % VPH;
        dk[at] = quads(kk, kvmul * (1.f / 256.f), e);
        dv[at] = quads(kv, kvmul * (1.f / 256.f), e);
      }
    }
  }
}

}  // namespace il

using namespace il;

template <bool PAGED>
static il_status synth_launch(il_ctx* c, uint32_t B, const uint32_t* prompt_tok, const int32_t* cu_q,
                              const int32_t* prefix_len, const int32_t* block_table, uint64_t seed, float q_scale,
                              il_bf16* q, il_bf16* kd, il_bf16* vd, il_stream s) {
  if (B == 0) return IL_OK;
  if (!kd != !vd) { set_error("k and v: both or neither"); return IL_ERR_ARG; }
  if (!q && !kd) return IL_OK;
  auto tseed = [&](uint64_t salt) { return mix64((seed << 8) ^ salt); };
  const float unit = 2.0f;                             // x = (f - 1.5) * 2 * scale
  const uint32_t d = c->cfg.head_dim, Hq = c->cfg.n_q_heads, Hkv = c->cfg.n_kv_heads;
  // a NULL q skips the Q heads, NULL k / v the K and V heads (Q of the next batch may be written
  // while this batch's attention still reads the pages the next batch's K / V will overwrite)
  const uint32_t h0 = q ? 0u : Hq, h1 = kd ? Hq + 2 * Hkv : Hq;
  if (d == 128)
    k_synth<128, PAGED><<<c->num_sms * 8, 256, 0, (cudaStream_t)s>>>(*c, B, prompt_tok, cu_q, prefix_len, block_table,
        tseed(0x51), tseed(0x4B), tseed(0x56), q_scale * unit, unit, (__nv_bfloat16*)q, (__nv_bfloat16*)kd,
        (__nv_bfloat16*)vd, h0, h1);
  else
    k_synth<64, PAGED><<<c->num_sms * 8, 256, 0, (cudaStream_t)s>>>(*c, B, prompt_tok, cu_q, prefix_len, block_table,
        tseed(0x51), tseed(0x4B), tseed(0x56), q_scale * unit, unit, (__nv_bfloat16*)q, (__nv_bfloat16*)kd,
        (__nv_bfloat16*)vd, h0, h1);
  IL_LAUNCH_CHECK("k_synth");
  c->launches += 1;
  return IL_OK;
}

extern "C" il_status il_synth_qkv(il_ctx* c, uint32_t B, const uint32_t* prompt_tok, const int32_t* cu_q,
                                  const int32_t* prefix_len, uint64_t seed, float q_scale, il_bf16* q,
                                  il_bf16* k_new, il_bf16* v_new, il_stream s) {
  return synth_launch<false>(c, B, prompt_tok, cu_q, prefix_len, nullptr, seed, q_scale, q, k_new, v_new, s);
}

extern "C" il_status il_synth_qkv_paged(il_ctx* c, uint32_t B, const uint32_t* prompt_tok, const int32_t* cu_q,
                                        const int32_t* prefix_len, const int32_t* block_table, uint64_t seed,
                                        float q_scale, il_bf16* q, il_bf16* k_pages, il_bf16* v_pages, il_stream s) {
  if (!c->matched) { set_error("il_synth_qkv_paged before il_prefix_match"); return IL_ERR_STATE; }
  return synth_launch<true>(c, B, prompt_tok, cu_q, prefix_len, block_table, seed, q_scale, q, k_pages, v_pages, s);
}
