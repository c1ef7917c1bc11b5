// attn.cu — il_prefill_attn: K7a suffix K/V append into pages, then prefill attention over
// the paged cached prefix + the causal suffix.  Dispatches to the
// tcgen05/TMA kernel (attn_sm100.cuh) for head_dim 128; the CUDA-core kernel below is the
// bring-up path (head_dim 64 and parity cross-checks).
#include <cuda_bf16.h>

#include "attn_common.cuh"
#include "il_internal.cuh"

namespace il {

// K7a: suffix row r of request i at absolute position p goes to page block_table[i][p/16],
// slot p%16, for every kv head: pages are [C][Hkv][16][d].  One warp per suffix row (the row's
// owner and page are looked up once); lanes move 16-byte vectors of K and V.
__global__ void __launch_bounds__(256) k_kv_append(Ctx c, uint32_t B, const int32_t* __restrict__ cu_q,
                                                   const int32_t* __restrict__ prefix_len,
                                                   const int32_t* __restrict__ block_table,
                                                   const uint4* __restrict__ k_new, const uint4* __restrict__ v_new,
                                                   uint4* __restrict__ k_pages, uint4* __restrict__ v_pages) {
  const uint32_t Hkv = c.cfg.n_kv_heads, vph = c.cfg.head_dim / 8;   // uint4 = 8 bf16
  const uint32_t vec_per_row = Hkv * vph;
  const uint32_t total = (uint32_t)cu_q[B], lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = gw; r < total; r += nw) {
    const uint32_t i = row_owner(cu_q, B, r);
    const uint32_t p = (uint32_t)prefix_len[i] + r - (uint32_t)cu_q[i];
    const uint32_t page = (uint32_t)block_table[(size_t)i * c.max_blocks + p / BS];
    const size_t src0 = (size_t)r * vec_per_row;
    for (uint32_t v = lane; v < vec_per_row; v += 32) {
      const uint32_t h = v / vph, x = v % vph;
      const size_t dst = (((size_t)page * Hkv + h) * BS + (p % BS)) * vph + x;
      const uint4 kk = k_new[src0 + v], vv = v_new[src0 + v];
      k_pages[dst] = kk;
      v_pages[dst] = vv;
    }
  }
}

// one CTA: tiles_i = ceil(S_i / tq); exclusive scan into tile_off; total into sc->n_tiles
// (+ cascade bookkeeping: suffix rows, dense M-tiles, shared-block bound = request 0's hits)
__global__ void __launch_bounds__(1024) k_tile_scan(Ctx c, uint32_t B, const int32_t* __restrict__ cu_q,
                                                    const int32_t* __restrict__ prefix_len, uint32_t tq,
                                                    uint32_t cascade) {
  __shared__ uint32_t s_w[32];
  const uint32_t tid = threadIdx.x, per = cdiv(B, 1024);
  uint32_t n = 0;
  for (uint32_t i = tid * per; i < min(B, (tid + 1) * per); ++i) n += cdiv((uint32_t)(cu_q[i + 1] - cu_q[i]), tq);
  uint32_t total;
  uint32_t acc = block_scan(n, s_w, &total);
  for (uint32_t i = tid * per; i < min(B, (tid + 1) * per); ++i) {
    c.tile_off[i] = acc;
    const uint32_t nt = cdiv((uint32_t)(cu_q[i + 1] - cu_q[i]), tq);
    for (uint32_t t = 0; t < nt; ++t) c.tile_req[acc + t] = i;
    acc += nt;
  }
  if (tid == 1023) {
    c.tile_off[B] = total; c.sc->n_tiles = total;
    const uint32_t tot = (uint32_t)cu_q[B];
    c.sc->q_total = tot;
    c.sc->n_dense = cdiv(tot, tq);
    c.sc->shared_blk = cascade ? (uint32_t)prefix_len[0] / BS : 0u;
  }
}

__device__ __forceinline__ uint32_t tile_owner(const uint32_t* __restrict__ tile_off, uint32_t B, uint32_t t) {
  uint32_t lo = 0, hi = B;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (tile_off[mid] <= t) lo = mid; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------------------
// Bring-up attention on CUDA cores (fp32 math, online softmax).  Work item = (request,
// kv head, tile of 16 suffix tokens); rows = 16 tokens x g q-heads (GQA packed).  K/V are
// streamed 32 keys at a time through shared memory.  Never benchmarked.
// ---------------------------------------------------------------------------------------
constexpr uint32_t SIMPLE_TQ = 16;
constexpr uint32_t SIMPLE_KC = 32;

template <int D>
__global__ void __launch_bounds__(256) k_attn_simple(Ctx c, uint32_t B, const int32_t* __restrict__ cu_q,
                                                     const int32_t* __restrict__ prefix_len,
                                                     const int32_t* __restrict__ block_table,
                                                     const __nv_bfloat16* __restrict__ q,
                                                     const __nv_bfloat16* __restrict__ k_pages,
                                                     const __nv_bfloat16* __restrict__ v_pages,
                                                     __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                                                     float scale) {
  constexpr int PER = D / 32;
  extern __shared__ float smem[];
  const uint32_t Hq = c.cfg.n_q_heads, Hkv = c.cfg.n_kv_heads, g = Hq / Hkv;
  const uint32_t R = SIMPLE_TQ * g;                    // rows of a work item (<= 128)
  float* sQ = smem;                                    // [R][D]
  float* sK = sQ + R * D;                              // [KC][D+1]
  float* sV = sK + SIMPLE_KC * (D + 1);                // [KC][D]
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const uint32_t n_items = c.sc->n_tiles * Hkv;
  for (uint32_t w = blockIdx.x; w < n_items; w += gridDim.x) {
    const uint32_t t = w / Hkv, kh = w % Hkv;
    const uint32_t i = tile_owner(c.tile_off, B, t);
    const uint32_t tt = t - c.tile_off[i];
    const uint32_t r0 = (uint32_t)cu_q[i] + tt * SIMPLE_TQ;
    const uint32_t S = (uint32_t)(cu_q[i + 1] - cu_q[i]);
    const uint32_t ntok = min(SIMPLE_TQ, S - tt * SIMPLE_TQ);
    const uint32_t P = (uint32_t)prefix_len[i];
    const uint32_t p0 = P + tt * SIMPLE_TQ;          // absolute position of the tile's first token
    const uint32_t p_last = p0 + ntok - 1;
    __syncthreads();
    // rows: row = tok * g + hh  (q head = kh * g + hh)
    for (uint32_t e = threadIdx.x; e < R * D; e += blockDim.x) {
      const uint32_t row = e / D, x = e % D, tok = row / g, hh = row % g;
      float v = 0.f;
      if (tok < ntok) v = __bfloat162float(q[((size_t)(r0 + tok) * Hq + kh * g + hh) * D + x]);
      sQ[e] = v;
    }
    float m[16], l[16], o[16][PER];
    const uint32_t rows_per_warp = cdiv(R, nw);
#pragma unroll
    for (int a = 0; a < 16; ++a) {
      m[a] = -INFINITY; l[a] = 0.f;
#pragma unroll
      for (int x = 0; x < PER; ++x) o[a][x] = 0.f;
    }
    const int32_t* bt = block_table + (size_t)i * c.max_blocks;
    for (uint32_t k0 = 0; k0 <= p_last; k0 += SIMPLE_KC) {
      __syncthreads();
      for (uint32_t e = threadIdx.x; e < SIMPLE_KC * D; e += blockDim.x) {
        const uint32_t j = e / D, x = e % D, pos = k0 + j;
        float kv = 0.f, vv = 0.f;
        if (pos <= p_last) {
          const uint32_t page = (uint32_t)bt[pos / BS];
          const size_t off = (((size_t)page * Hkv + kh) * BS + pos % BS) * D + x;
          kv = __bfloat162float(k_pages[off]);
          vv = __bfloat162float(v_pages[off]);
        }
        sK[j * (D + 1) + x] = kv;
        sV[j * D + x] = vv;
      }
      __syncthreads();
#pragma unroll
      for (int a = 0; a < 16; ++a) {
        const uint32_t row = warp * rows_per_warp + a;
        if ((uint32_t)a >= rows_per_warp || row >= R) continue;
        const uint32_t tok = row / g;
        if (tok >= ntok) continue;
        const uint32_t pos_q = p0 + tok, key = k0 + lane;
        float sc = 0.f;
        for (uint32_t x = 0; x < D; ++x) sc += sQ[row * D + x] * sK[lane * (D + 1) + x];
        sc = (key <= pos_q) ? sc * scale : -INFINITY;
        float mx = sc;
        for (int of = 16; of; of >>= 1) mx = fmaxf(mx, __shfl_xor_sync(~0u, mx, of));
        const float m_new = fmaxf(m[a], mx);
        const float corr = __expf(m[a] - m_new);
        const float pj = (key <= pos_q) ? __expf(sc - m_new) : 0.f;
        float ps = pj;
        for (int of = 16; of; of >>= 1) ps += __shfl_xor_sync(~0u, ps, of);
        l[a] = l[a] * corr + ps;
        m[a] = m_new;
#pragma unroll
        for (int x = 0; x < PER; ++x) o[a][x] *= corr;
        for (uint32_t j = 0; j < SIMPLE_KC; ++j) {
          const float pjj = __shfl_sync(~0u, pj, j);
#pragma unroll
          for (int x = 0; x < PER; ++x) o[a][x] += pjj * sV[j * D + lane + 32 * x];
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 16; ++a) {
      const uint32_t row = warp * rows_per_warp + a;
      if ((uint32_t)a >= rows_per_warp || row >= R) continue;
      const uint32_t tok = row / g, hh = row % g;
      if (tok >= ntok) continue;
      const float inv = 1.f / l[a];
      const size_t base = ((size_t)(r0 + tok) * Hq + kh * g + hh) * D;
#pragma unroll
      for (int x = 0; x < PER; ++x) out[base + lane + 32 * x] = __float2bfloat16_rn(o[a][x] * inv);
      if (lse && lane == 0) lse[(size_t)(r0 + tok) * Hq + kh * g + hh] = m[a] + __logf(l[a]);
    }
  }
}

}  // namespace il

#include "attn_sm100.cuh"

using namespace il;

extern "C" il_status il_prefill_attn(il_ctx* c, uint32_t B, const int32_t* cu_q, const int32_t* prefix_len,
                                     const int32_t* block_table, const il_bf16* q, const il_bf16* k_new,
                                     const il_bf16* v_new, il_bf16* k_pages, il_bf16* v_pages, il_bf16* out,
                                     float* lse, float scale, il_stream s) {
  if (!c->matched) { set_error("il_prefill_attn before il_prefix_match"); return IL_ERR_STATE; }
  if (B == 0) return IL_OK;
  cudaStream_t st = (cudaStream_t)s;
  const uint32_t d = c->cfg.head_dim, g = c->cfg.n_q_heads / c->cfg.n_kv_heads;
  k_kv_append<<<c->num_sms * 8, 256, 0, st>>>(*c, B, cu_q, prefix_len, block_table, (const uint4*)k_new,
                                              (const uint4*)v_new, (uint4*)k_pages, (uint4*)v_pages);
  IL_LAUNCH_CHECK("k_kv_append");
  c->launches += 1;
  if (attn_sm100_supported(c)) {
    return attn_sm100_launch(c, B, cu_q, prefix_len, block_table, q, k_pages, v_pages, out, lse, scale, st);
  }
  if (g * SIMPLE_TQ > 128) { set_error("bring-up attention: Hq/Hkv > 8 unsupported"); return IL_ERR_ARG; }
  k_tile_scan<<<1, 1024, 0, st>>>(*c, B, cu_q, prefix_len, SIMPLE_TQ, 0u);
  const uint32_t R = SIMPLE_TQ * g;
  const size_t smem = ((size_t)R * d + SIMPLE_KC * (d + 1) + SIMPLE_KC * d) * sizeof(float);
  if (d == 128) {
    static bool a = false;
    if (!a) { IL_CUDA(cudaFuncSetAttribute(k_attn_simple<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); a = true; }
    k_attn_simple<128><<<c->num_sms * 4, 256, smem, st>>>(*c, B, cu_q, prefix_len, block_table,
        (const __nv_bfloat16*)q, (const __nv_bfloat16*)k_pages, (const __nv_bfloat16*)v_pages,
        (__nv_bfloat16*)out, lse, scale);
  } else {
    static bool a = false;
    if (!a) { IL_CUDA(cudaFuncSetAttribute(k_attn_simple<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); a = true; }
    k_attn_simple<64><<<c->num_sms * 4, 256, smem, st>>>(*c, B, cu_q, prefix_len, block_table,
        (const __nv_bfloat16*)q, (const __nv_bfloat16*)k_pages, (const __nv_bfloat16*)v_pages,
        (__nv_bfloat16*)out, lse, scale);
  }
  IL_LAUNCH_CHECK("k_attn_simple");
  c->launches += 2;
  return IL_OK;
}

#ifdef IL_ATTN_TRACE
extern "C" il_status il_debug_trace(unsigned long long* out_h) {
  IL_CUDA(cudaDeviceSynchronize());
  IL_CUDA(cudaMemcpyFromSymbol(out_h, il::sm100::g_trace, sizeof(il::sm100::g_trace)));
  IL_CUDA(cudaMemcpyFromSymbol(out_h + 16 * 4096, il::sm100::g_trace_item, sizeof(il::sm100::g_trace_item)));
  return IL_OK;
}
#endif
