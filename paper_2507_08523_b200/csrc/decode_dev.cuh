// decode_dev.cuh — the per-request part of paged decode attention on CUDA cores (il_decode_attn,
// SURVEY §8(f) NEXT-4).  One query row per request (g q-heads per kv head) against its own keys
// [NC * 128, pos]: a dot-product stream, HBM-bound (every key's K and V read once), where an M=128
// tensor tile would be 97% padding.  The keys below NC * 128 (the batch-shared prefix) are left to
// the tensor kernel's dense phase 1, which starts each row from the partial written here.
#pragma once

#include <cuda_bf16.h>

#include "il_internal.cuh"

namespace il {

// One CTA of DEC_WARPS warps per (request i, kv head kh); warp w takes key chunks w, w + DEC_WARPS,
// ... (split-K), and the warps' partial softmax states are merged through shared memory at the
// end.  Within a warp, lane l holds dims [l * DPL, l * DPL + DPL) of the g query heads and of their
// accumulators.  A chunk is KC = 32 / G2 keys (G2 = g rounded up to a power of two): the K and V
// rows of all its keys are loaded first (2 KC loads in flight per lane, coalesced 2 D bytes per
// row), each lane forms its partial dot products for all KC x G2 (key, head) pairs over its dims,
// one 31-shuffle transpose-reduction leaves lane l with the full score of (key l / G2, head l % G2),
// an online softmax per head (log2 domain, exact running max), then O += p V.  Output: with a
// shared prefix (NC > 0) the phase-2 partial (out = O / l, attn_ml = m + log2 l) that phase 1
// merges; without, the final row and its natural-log LSE.
constexpr uint32_t DEC_WARPS = 4;
#ifndef DEC_KEYS_IN_FLIGHT
#define DEC_KEYS_IN_FLIGHT 8      // (16: 5.94 ms per 16 c3 decode steps vs 5.11: registers cost more occupancy than the loads gain)
#endif

__device__ __forceinline__ void bf16x4(const uint2 u, float* f) {
  f[0] = __uint_as_float(u.x << 16); f[1] = __uint_as_float(u.x & 0xFFFF0000u);
  f[2] = __uint_as_float(u.y << 16); f[3] = __uint_as_float(u.y & 0xFFFF0000u);
}
__device__ __forceinline__ void bf16x2(const uint32_t u, float* f) {
  f[0] = __uint_as_float(u << 16); f[1] = __uint_as_float(u & 0xFFFF0000u);
}

template <uint32_t D, uint32_t G2>
__global__ void __launch_bounds__(DEC_WARPS * 32) k_decode_own(Ctx c, uint32_t B, const int32_t* __restrict__ pos,
                                                               const int32_t* __restrict__ block_table,
                                                               const __nv_bfloat16* __restrict__ q,
                                                               const __nv_bfloat16* __restrict__ k_pages,
                                                               const __nv_bfloat16* __restrict__ v_pages,
                                                               __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                                                               float scale_log2) {
  constexpr uint32_t DPL = D / 32;                       // dims per lane: 4 (D = 128) or 2 (D = 64)
  constexpr uint32_t KC = 32 / G2;                       // keys per chunk
  __shared__ float s_m[DEC_WARPS][G2], s_l[DEC_WARPS][G2];
  __shared__ float s_acc[DEC_WARPS][G2][D];
  const uint32_t Hq = c.cfg.n_q_heads, Hkv = c.cfg.n_kv_heads, g = Hq / Hkv;   // g <= G2
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t i = blockIdx.x / Hkv, kh = blockIdx.x % Hkv;
  if (i >= B) return;
  const uint32_t NC = c.sc->shared_blk / 8;
  const int32_t p = pos[i];
  const int32_t k0 = (int32_t)(NC * 128);                // (k_shared_scan: NC * 128 <= pos)
  const int32_t* bt = block_table + (size_t)i * c.max_blocks;
  // q slice of every head, pre-scaled to the log2 domain (heads g..G2-1: zero, masked below)
  float qv[G2][DPL];
#pragma unroll
  for (uint32_t h = 0; h < G2; ++h) {
#pragma unroll
    for (uint32_t e = 0; e < DPL; ++e) qv[h][e] = 0.f;
    if (h < g) {
      const __nv_bfloat16* qr = q + ((size_t)i * Hq + kh * g + h) * D + lane * DPL;
#pragma unroll
      for (uint32_t e = 0; e < DPL; ++e) qv[h][e] = __bfloat162float(qr[e]) * scale_log2;
    }
  }
  float acc[G2][DPL];
#pragma unroll
  for (uint32_t h = 0; h < G2; ++h)
#pragma unroll
    for (uint32_t e = 0; e < DPL; ++e) acc[h][e] = 0.f;
  const uint32_t my_h = lane % G2;
  float m = -INFINITY, l = 0.f;                          // running max / sum of head my_h (replicated)
  const size_t head_off = (size_t)kh * BS * D + lane * DPL;
  // NSUB chunks per iteration: their K and V rows (this lane's dims) are all loaded first, so
  // 2 x NSUB x KC loads per lane are in flight together (the kernel is bound by HBM latency x
  // bytes in flight), then the chunks are processed one by one
  constexpr uint32_t NSUB = KC >= DEC_KEYS_IN_FLIGHT ? 1 : DEC_KEYS_IN_FLIGHT / KC;
  for (int32_t kb0 = k0 + (int32_t)(warp * NSUB * KC); kb0 <= p; kb0 += (int32_t)(DEC_WARPS * NSUB * KC)) {
    uint32_t kraw_all[NSUB][KC][DPL / 2], vraw_all[NSUB][KC][DPL / 2];
#pragma unroll
    for (uint32_t sub = 0; sub < NSUB; ++sub)
#pragma unroll
    for (uint32_t kk = 0; kk < KC; ++kk) {
      const int32_t key = min(kb0 + (int32_t)(sub * KC + kk), p);   // (past p: a duplicate load, masked)
      const uint32_t page = (uint32_t)__ldg(bt + key / BS);
      const size_t off = (size_t)page * Hkv * BS * D + head_off + (size_t)(key % BS) * D;
      if (DPL == 4) {
        const uint2 a = __ldg(reinterpret_cast<const uint2*>(k_pages + off));
        const uint2 b = __ldg(reinterpret_cast<const uint2*>(v_pages + off));
        kraw_all[sub][kk][0] = a.x; kraw_all[sub][kk][DPL / 2 - 1] = a.y;
        vraw_all[sub][kk][0] = b.x; vraw_all[sub][kk][DPL / 2 - 1] = b.y;
      } else {
        kraw_all[sub][kk][0] = __ldg(reinterpret_cast<const uint32_t*>(k_pages + off));
        vraw_all[sub][kk][0] = __ldg(reinterpret_cast<const uint32_t*>(v_pages + off));
      }
    }
#pragma unroll
    for (uint32_t sub = 0; sub < NSUB; ++sub) {
    const int32_t kb = kb0 + (int32_t)(sub * KC);
    if (kb > p) break;
    const auto& kraw = kraw_all[sub];
    const auto& vraw = vraw_all[sub];
    // partial dots: vals[kk * G2 + h] over this lane's dims
    float vals[32];
#pragma unroll
    for (uint32_t kk = 0; kk < KC; ++kk) {
      float kf[DPL];
      if (DPL == 4) bf16x4(make_uint2(kraw[kk][0], kraw[kk][DPL / 2 - 1]), kf); else bf16x2(kraw[kk][0], kf);
#pragma unroll
      for (uint32_t h = 0; h < G2; ++h) {
        float sc = 0.f;
#pragma unroll
        for (uint32_t e = 0; e < DPL; ++e) sc = fmaf(qv[h][e], kf[e], sc);
        vals[kk * G2 + h] = sc;
      }
    }
    // transpose-reduce: after the step with offset o the lane keeps the half of the indices whose
    // bit o equals its own bit o; at the end vals[0] on lane l is the total of index l
#pragma unroll
    for (uint32_t o = 16; o >= 1; o >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (uint32_t x = 0; x < o; ++x) {
        const float send = up ? vals[x] : vals[x + o];
        const float keep = up ? vals[x + o] : vals[x];
        vals[x] = keep + __shfl_xor_sync(~0u, send, o);
      }
    }
    const int32_t my_key = kb + (int32_t)(lane / G2);
    const float sc = (my_key <= p && my_h < g) ? vals[0] : -INFINITY;
    // online softmax of head my_h over the lanes with the same head (xor over the key bits)
    float cm = sc;
#pragma unroll
    for (uint32_t o = G2; o < 32; o <<= 1) cm = fmaxf(cm, __shfl_xor_sync(~0u, cm, o));
    const float m_new = fmaxf(m, cm);
    const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - m_new);
    const float pk = (sc == -INFINITY) ? 0.f : exp2f(sc - m_new);
    float ps = pk;
#pragma unroll
    for (uint32_t o = G2; o < 32; o <<= 1) ps += __shfl_xor_sync(~0u, ps, o);
    l = l * alpha + ps;
    m = m_new;
#pragma unroll
    for (uint32_t h = 0; h < G2; ++h) {
      const float a = __shfl_sync(~0u, alpha, h);
#pragma unroll
      for (uint32_t e = 0; e < DPL; ++e) acc[h][e] *= a;
    }
    // O += p V (keys past p have p = 0)
#pragma unroll
    for (uint32_t kk = 0; kk < KC; ++kk) {
      float vf[DPL];
      if (DPL == 4) bf16x4(make_uint2(vraw[kk][0], vraw[kk][DPL / 2 - 1]), vf); else bf16x2(vraw[kk][0], vf);
#pragma unroll
      for (uint32_t h = 0; h < G2; ++h) {
        const float ph = __shfl_sync(~0u, pk, kk * G2 + h);
#pragma unroll
        for (uint32_t e = 0; e < DPL; ++e) acc[h][e] = fmaf(ph, vf[e], acc[h][e]);
      }
    }
    }
  }
  // merge the warps' states: M = max_w m_w, L = sum_w l_w 2^(m_w - M), O = sum_w O_w 2^(m_w - M)
#pragma unroll
  for (uint32_t h = 0; h < G2; ++h) {
#pragma unroll
    for (uint32_t e = 0; e < DPL; ++e) s_acc[warp][h][lane * DPL + e] = acc[h][e];
  }
  if (lane < G2) { s_m[warp][lane] = m; s_l[warp][lane] = l; }
  __syncthreads();
  const bool cascade = NC > 0;
  for (uint32_t x = threadIdx.x; x < g * D; x += DEC_WARPS * 32) {
    const uint32_t h = x / D, dd = x % D;
    float M = -INFINITY;
#pragma unroll
    for (uint32_t w = 0; w < DEC_WARPS; ++w) M = fmaxf(M, s_m[w][h]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (uint32_t w = 0; w < DEC_WARPS; ++w) {
      const float f = s_m[w][h] == -INFINITY ? 0.f : exp2f(s_m[w][h] - M);
      L += s_l[w][h] * f;
      O += s_acc[w][h][dd] * f;
    }
    const size_t orow = (size_t)i * Hq + kh * g + h;
    out[orow * D + dd] = __float2bfloat16_rn(O / L);
    if (dd == 0) {
      if (cascade) c.attn_ml[orow] = M + __log2f(L);
      else if (lse) lse[orow] = (M + __log2f(L)) * 0.69314718055994531f;
    }
  }
}

}  // namespace il
