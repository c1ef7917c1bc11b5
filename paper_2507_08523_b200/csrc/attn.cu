// attn.cu — il_prefill_attn: K7a suffix K/V append into pages, then prefill attention over
// the paged cached prefix + the causal suffix on the tcgen05/TMA kernel
// (attn_sm100.cuh; head_dim 64 or 128, Hq/Hkv in 1..8 -- validate() rejects anything else at
// il_create, so there is no other attention kernel).
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
    const uint32_t S = (uint32_t)(cu_q[i + 1] - cu_q[i]), nt = cdiv(S, tq);
    const uint32_t P = (uint32_t)prefix_len[i], r0 = (uint32_t)cu_q[i], nblk = cdiv(P + S, BS);
    for (uint32_t t = 0; t < nt; ++t) {
      c.tile_req[acc + t] = i;
      // (one 16-byte load decodes a tile in the phase-2 kernel: no dependent loads at item switches)
      c.tile_desc[acc + t] = make_uint4(i, P + t * tq, r0 + t * tq, min(tq, S - t * tq) | (nblk << 8));
    }
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

}  // namespace il

#include "decode_dev.cuh"
#include "attn_sm100.cuh"

using namespace il;

extern "C" il_status il_prefill_attn(il_ctx* c, uint32_t B, const int32_t* cu_q, const int32_t* prefix_len,
                                     const int32_t* block_table, const il_bf16* q, const il_bf16* k_new,
                                     const il_bf16* v_new, il_bf16* k_pages, il_bf16* v_pages, il_bf16* out,
                                     float* lse, float scale, il_stream s) {
  if (!c->matched) { set_error("il_prefill_attn before il_prefix_match"); return IL_ERR_STATE; }
  if (B == 0) return IL_OK;
  cudaStream_t st = (cudaStream_t)s;
  if (k_new || v_new) {                                 // (both NULL: the suffix K / V are already in the pages)
    if (!k_new || !v_new) { set_error("k_new and v_new: both or neither"); return IL_ERR_ARG; }
    k_kv_append<<<c->num_sms * 8, 256, 0, st>>>(*c, B, cu_q, prefix_len, block_table, (const uint4*)k_new,
                                                (const uint4*)v_new, (uint4*)k_pages, (uint4*)v_pages);
    IL_LAUNCH_CHECK("k_kv_append");
    c->launches += 1;
  }
  return attn_sm100_launch(c, B, cu_q, prefix_len, block_table, q, k_pages, v_pages, out, lse, scale, st);
}

extern "C" il_status il_decode_attn(il_ctx* c, uint32_t B, const int32_t* pos, const int32_t* block_table,
                                    const il_bf16* q, const il_bf16* k_new, const il_bf16* v_new, il_bf16* k_pages,
                                    il_bf16* v_pages, il_bf16* out, float* lse, float scale, il_stream s) {
  if (!c->matched) { set_error("il_decode_attn before il_prefix_match"); return IL_ERR_STATE; }
  if (B > c->cfg.max_batch) { set_error("B > max_batch"); return IL_ERR_ARG; }
  if (B == 0) return IL_OK;
  cudaStream_t st = (cudaStream_t)s;
  const int32_t* cu = reinterpret_cast<const int32_t*>(c->dec_cu);    // 0, 1, .., max_batch
  if (k_new || v_new) {
    if (!k_new || !v_new) { set_error("k_new and v_new: both or neither"); return IL_ERR_ARG; }
    k_kv_append<<<c->num_sms * 8, 256, 0, st>>>(*c, B, cu, pos, block_table, (const uint4*)k_new,
                                                (const uint4*)v_new, (uint4*)k_pages, (uint4*)v_pages);
    IL_LAUNCH_CHECK("k_kv_append");
    c->launches += 1;
  }
  return attn_sm100_launch(c, B, cu, pos, block_table, q, k_pages, v_pages, out, lse, scale, st, true);
}

// one-time per-context setup of the attention kernels (il_create, current device)
il_status il::attn_setup(Ctx*) {
  IL_CUDA(cudaFuncSetAttribute(sm100::k_attn_sm100<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               sm100::smem_bytes(128)));
  IL_CUDA(cudaFuncSetAttribute(sm100::k_attn_sm100<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               sm100::smem_bytes(64)));
  IL_CUDA(cudaFuncSetAttribute(sm100::d2::k_attn_dense2<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm100::d2::SMEM));
  using sm100::p2::k_attn_p2;
  IL_CUDA(cudaFuncSetAttribute(k_attn_p2<128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm100::p2::smem_bytes2<128>));
  IL_CUDA(cudaFuncSetAttribute(k_attn_p2<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm100::p2::smem_bytes2<64>));
  IL_CUDA(cudaFuncSetAttribute(k_attn_p2<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm100::p2::smem_bytes2<128>));
  IL_CUDA(cudaFuncSetAttribute(k_attn_p2<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm100::p2::smem_bytes2<64>));
  // the phase-2 kernel's setmaxnreg split assumes the launch register count (a smaller pool
  // would leave setmaxnreg.inc waiting forever): refuse to run otherwise
  for (const void* f : {(const void*)k_attn_p2<128, false>, (const void*)k_attn_p2<64, false>,
                        (const void*)k_attn_p2<128, true>, (const void*)k_attn_p2<64, true>}) {
    cudaFuncAttributes a;
    IL_CUDA(cudaFuncGetAttributes(&a, f));
    if (a.numRegs != sm100::p2::REGS2_LAUNCH) {
      set_error("k_attn_p2 compiled with an unexpected register count (setmaxnreg pool)");
      return IL_ERR_CUDA;
    }
  }
  return IL_OK;
}

#ifdef IL_ATTN_TRACE
extern "C" il_status il_debug_trace_reset() {
  IL_CUDA(cudaDeviceSynchronize());
  static unsigned long long zero[16 * 4096];
  IL_CUDA(cudaMemcpyToSymbol(il::sm100::g_trace, zero, sizeof(zero)));
  return IL_OK;
}
extern "C" il_status il_debug_trace(unsigned long long* out_h) {
  IL_CUDA(cudaDeviceSynchronize());
  IL_CUDA(cudaMemcpyFromSymbol(out_h, il::sm100::g_trace, sizeof(il::sm100::g_trace)));
  IL_CUDA(cudaMemcpyFromSymbol(out_h + 16 * 4096, il::sm100::g_trace_item, sizeof(il::sm100::g_trace_item)));
  return IL_OK;
}
#endif
