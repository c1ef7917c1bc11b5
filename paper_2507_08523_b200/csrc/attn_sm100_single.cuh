// attn_sm100_single.cuh — variant of the tcgen05 prefill attention with ONE M-tile per work
// item: 128-key KV tiles (N = 128 QK MMAs), S and O double-buffered in TMEM, two softmax
// warpgroups splitting each tile's key columns.  Selected with IL_ATTN_KERNEL=single.
#pragma once
#include "attn_sm100.cuh"

namespace il {
namespace sm100s {
using namespace il::sm100;



constexpr uint32_t D = 128;              // head dim handled by this kernel
constexpr uint32_t BM = 128, BN = 128;   // rows per M-tile, keys per KV tile
constexpr uint32_t CB = 16384;           // one 64-column block of a 128-row bf16 tile
constexpr uint32_t TILE = 2 * CB;        // 128 x 128 bf16 = 32 KB
constexpr uint32_t NST = 3;              // K and V ring depth (each)
constexpr uint32_t OFF_Q = 0;
constexpr uint32_t OFF_K = TILE;                 // K[s] = OFF_K + s * TILE
constexpr uint32_t OFF_V = (1 + NST) * TILE;     // V[s] = OFF_V + s * TILE
constexpr uint32_t OFF_RED = (1 + 2 * NST) * TILE;   // float red[2 tiles][2 WGs][128 rows]
constexpr uint32_t OFF_BAR = OFF_RED + 2 * 2 * 128 * 4;
constexpr uint32_t NBAR = 32;
constexpr uint32_t SMEM_BYTES = OFF_BAR + NBAR * 8 + 16;
constexpr int THREADS = 384;
constexpr uint32_t SM_THREADS = 256;     // two softmax warpgroups

enum Bar { Q_FULL = 0, Q_FREE = 1, K_FULL = 2, K_FREE = 5, V_FULL = 8, V_FREE = 11, S_FULL = 14, P_FULL = 16,
           PV_DONE = 18, O_FULL = 20, O_FREE = 22 };

constexpr uint32_t IDESC_QK = (1u << 4) | (1u << 7) | (1u << 10) | ((BN >> 3) << 17) | ((BM >> 4) << 24);
constexpr uint32_t IDESC_PV = IDESC_QK | (1u << 16);

struct Item {
  uint32_t i, kh, mt, P, S, r0, ntok, n_kv, nblk;
};
__device__ __forceinline__ Item decode_item(const Ctx& c, uint32_t B, const int32_t* __restrict__ cu_q,
                                            const int32_t* __restrict__ prefix_len, uint32_t w, uint32_t Hkv,
                                            uint32_t TQ) {
  Item it;
  const uint32_t t = w / Hkv;
  it.kh = w % Hkv;
  const uint32_t lo = c.tile_req[t];
  it.i = lo;
  it.mt = t - c.tile_off[lo];
  it.P = (uint32_t)prefix_len[lo];
  it.r0 = (uint32_t)cu_q[lo];
  it.S = (uint32_t)cu_q[lo + 1] - it.r0;
  it.ntok = min(TQ, it.S - it.mt * TQ);
  const uint32_t p_last = it.P + it.mt * TQ + it.ntok - 1;
  it.n_kv = p_last / BN + 1;
  it.nblk = cdiv(it.P + it.S, BS);
  return it;
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    k_attn_sm100s(Ctx c, uint32_t B, const int32_t* __restrict__ cu_q, const int32_t* __restrict__ prefix_len,
                 const int32_t* __restrict__ block_table, __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                 float scale_log2, uint32_t g, uint32_t TQ, const __grid_constant__ CUtensorMap tm_q,
                 const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023) != 0) __trap();          // swizzle atoms need 1024-byte alignment
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + OFF_BAR;
  auto bar = [&](uint32_t idx) { return bar0 + 8 * idx; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + NBAR * 8);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t Hq = c.cfg.n_q_heads, Hkv = c.cfg.n_kv_heads;
  const uint32_t n_items = c.sc->n_tiles * Hkv;

  if (threadIdx.x == 0) {
    mbar_init(bar(Q_FULL), 1); mbar_init(bar(Q_FREE), 1);
    for (uint32_t s = 0; s < NST; ++s) {
      mbar_init(bar(K_FULL + s), 1); mbar_init(bar(K_FREE + s), 1);
      mbar_init(bar(V_FULL + s), 1); mbar_init(bar(V_FREE + s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bar(S_FULL + b), 1); mbar_init(bar(P_FULL + b), SM_THREADS); mbar_init(bar(PV_DONE + b), 1);
      mbar_init(bar(O_FULL + b), 1); mbar_init(bar(O_FREE + b), SM_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm_q) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm_k) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm_v) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: S[0] = [0,128), S[1] = [128,256) (P of a tile overwrites the first 64
  // columns of its S as packed bf16), O[0] = [256,384), O[1] = [384,512).

  if (warp == 0 || warp == 3) {
    // ================= TMA producers: warp 0 = Q + K tiles, warp 3 = V tiles =================
    // The whole warp fetches the 8 page ids of a KV tile in parallel (one tile ahead); lane 0
    // issues the TMA boxes.
    const bool is_k = warp == 0;
    const CUtensorMap* tm = is_k ? &tm_k : &tm_v;
    const uint32_t full0 = is_k ? K_FULL : V_FULL, free0 = is_k ? K_FREE : V_FREE;
    const uint32_t ring = sbase + (is_k ? OFF_K : OFF_V);
    uint32_t kt = 0, it = 0;
    for (uint32_t w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
      const Item I = decode_item(c, B, cu_q, prefix_len, w, Hkv, TQ);
      const int32_t* bt = block_table + (size_t)I.i * c.max_blocks;
      auto page_of = [&](uint32_t n) -> int32_t {   // lane's page: lane & 7
        const uint32_t blk = n * 8 + (lane & 7);
        return blk < I.nblk ? __ldg(bt + blk) : __ldg(bt);
      };
      int32_t nxt = page_of(0);
      if (is_k && lane == 0) {
        if (it >= 1) mbar_wait(bar(Q_FREE), (it - 1) & 1);
        mbar_expect_tx(bar(Q_FULL), 2 * 128 * g * TQ);
        const int qrow = (int)(I.r0 + I.mt * TQ);
        tma_load_3d(sbase + OFF_Q, &tm_q, 0, (int)(I.kh * g), qrow, bar(Q_FULL));
        tma_load_3d(sbase + OFF_Q + CB, &tm_q, 64, (int)(I.kh * g), qrow, bar(Q_FULL));
      }
      for (uint32_t n = 0; n < I.n_kv; ++n, ++kt) {
        const int32_t cur = nxt;
        if (n + 1 < I.n_kv) nxt = page_of(n + 1);
        const uint32_t s = kt % NST, u = kt / NST;
        if (lane == 0) {
          if (kt >= NST) mbar_wait(bar(free0 + s), (u - 1) & 1);
          if (0) IL_TRACE(is_k ? 0 : 1, kt);
          mbar_expect_tx(bar(full0 + s), TILE);
        }
        const uint32_t dst = ring + s * TILE;
        __syncwarp();
        if (lane < 16) {                                 // lane = (page, column half)
          const uint32_t p = lane & 7, h = lane >> 3;
          const int row = (int)(((uint32_t)cur * Hkv + I.kh) * BS);
          tma_load_2d(dst + h * CB + p * 2048, tm, (int)(64 * h), row, bar(full0 + s));
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer: warp-uniform loop, one elected lane issues ==============
    const uint64_t dq = sdesc(sbase + OFF_Q, 16, 1024);
    const uint64_t dk0 = sdesc(sbase + OFF_K, 16, 1024), dv0 = sdesc(sbase + OFF_V, CB, 1024);
    uint32_t kt = 0, it = 0;
    for (uint32_t w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
      const Item I = decode_item(c, B, cu_q, prefix_len, w, Hkv, TQ);
      const uint32_t ob = it & 1;
      const uint32_t o_tmem = tmem + 256 + ob * 128;
      mbar_wait(bar(Q_FULL), it & 1);
      if (it >= 2) mbar_wait(bar(O_FREE + ob), ((it - 2) >> 1) & 1);
      tc_fence_after();
      auto pv = [&](uint32_t tt, bool first) {
        const uint32_t b = tt & 1, s = tt % NST;
        mbar_wait(bar(P_FULL + b), (tt >> 1) & 1);
        mbar_wait(bar(V_FULL + s), (tt / NST) & 1);
        tc_fence_after();
        const uint64_t dv = dv0 + (uint64_t)((s * TILE) >> 4);
        const uint32_t p_tmem = tmem + b * 128;
#pragma unroll
        for (uint32_t k = 0; k < 8; ++k)
          mma_ts_w<IDESC_PV>(o_tmem, p_tmem + k * 8, dv + (uint64_t)((k * 2048) >> 4), (first && k == 0) ? 0u : 1u);
        commit_w(bar(PV_DONE + b));
        commit_w(bar(V_FREE + s));
      };
      for (uint32_t n = 0; n < I.n_kv; ++n, ++kt) {
        const uint32_t s = kt % NST, b = kt & 1;
        mbar_wait(bar(K_FULL + s), (kt / NST) & 1);
        tc_fence_after();
        const uint64_t dk = dk0 + (uint64_t)((s * TILE) >> 4);
#pragma unroll
        for (uint32_t k = 0; k < 8; ++k)
          mma_ss_w<IDESC_QK>(tmem + b * 128, dq + (uint64_t)(((k >> 2) * CB + (k & 3) * 32) >> 4),
                             dk + (uint64_t)(((k >> 2) * CB + (k & 3) * 32) >> 4), k ? 1u : 0u);
        commit_w(bar(S_FULL + b));
        commit_w(bar(K_FREE + s));
        if (n + 1 == I.n_kv) commit_w(bar(Q_FREE));
        if (n >= 1) pv(kt - 1, n == 1);
      }
      pv(kt - 1, I.n_kv == 1);
      commit_w(bar(O_FULL + ob));
    }
  } else if (warp >= 4) {
    // ================= softmax + epilogue: 2 warpgroups x 128 threads, thread = row =========
    // WG w owns key columns [64w, 64w+64) of every S tile and O columns [64w, 64w+64); the row
    // max is combined through shared memory, so both WGs exponentiate against the same max.
    const uint32_t sm_t = threadIdx.x - 128, wg = sm_t >> 7, r = sm_t & 127, q4 = warp & 3;
    const uint32_t lane_addr = (32 * q4) << 16;
    float* red = reinterpret_cast<float*>(smem + OFF_RED);
    uint32_t kt = 0, it = 0;
    for (uint32_t w = blockIdx.x; w < n_items; w += gridDim.x, ++it) {
      const Item I = decode_item(c, B, cu_q, prefix_len, w, Hkv, TQ);
      const uint32_t t = r / g, hh = r % g;
      const bool valid = (r < g * TQ) && (t < I.ntok);
      const uint32_t pos_q = I.P + I.mt * TQ + min(t, I.ntok - 1);
      const uint32_t ob = it & 1;
      const uint32_t o_tmem = tmem + lane_addr + 256 + ob * 128 + 64 * wg;
      float m_used = -INFINITY, l = 0.f;
      for (uint32_t n = 0; n < I.n_kv; ++n, ++kt) {
        const uint32_t b = kt & 1;
        const uint32_t s_tmem = tmem + lane_addr + b * 128;
        mbar_wait(bar(S_FULL + b), (kt >> 1) & 1);
        if (sm_t == 0) if (0) IL_TRACE(4, kt);
        tc_fence_after();
        float sv[64];
        tmem_ld32(s_tmem + 64 * wg, *reinterpret_cast<float(*)[32]>(&sv[0]));
        tmem_ld32(s_tmem + 64 * wg + 32, *reinterpret_cast<float(*)[32]>(&sv[32]));
        tmem_wait_ld();
        const uint32_t key0 = n * BN + 64 * wg;
        if (key0 + 63 > pos_q) {
#pragma unroll
          for (int j = 0; j < 64; ++j)
            if (key0 + j > pos_q) sv[j] = -INFINITY;
        }
        float mxa[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) mxa[a] = sv[a];
#pragma unroll
        for (int j = 8; j < 64; ++j) mxa[j & 7] = fmaxf(mxa[j & 7], sv[j]);
        float* rb = red + b * 256;
        rb[wg * 128 + r] = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                                 fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
        named_bar_sync(1, SM_THREADS);
        if (sm_t == 0) if (0) IL_TRACE(5, kt);
        const float mx2 = fmaxf(rb[r], rb[128 + r]) * scale_log2;
        bool need = false;
        float factor = 1.f;
        if (n == 0) {
          m_used = mx2;
        } else if (mx2 > m_used + 8.f) {
          need = true;
          factor = ex2(m_used - mx2);
          m_used = mx2;
          l *= factor;
        }
        if (__any_sync(~0u, need)) {
          // lazy rescale of this warp's rows of its O half once PV of the previous tile landed
          mbar_wait(bar(PV_DONE + ((kt - 1) & 1)), ((kt - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            float ov[32];
            tmem_ld32(o_tmem + 32 * q, ov);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] *= factor;
            tmem_st32(o_tmem + 32 * q, ov);
          }
          tmem_wait_st();
        }
        const float negm = -m_used;
        float rsa[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
          const float p0 = ex2(fmaf(sv[j], scale_log2, negm));
          const float p1 = ex2(fmaf(sv[j + 1], scale_log2, negm));
          rsa[(j >> 1) & 3] += p0 + p1;
          pk[j >> 1] = pack_bf16(p0, p1);
        }
        l += (rsa[0] + rsa[1]) + (rsa[2] + rsa[3]);
        // P (bf16 pairs) of keys [64wg, 64wg+64) -> TMEM columns [32wg, 32wg+32) of this S
        tmem_st32u(s_tmem + 32 * wg, pk);
        tmem_wait_st();
        tc_fence_before();
        if (r == 0) if (0) IL_TRACE(6 + wg, kt);
        mbar_arrive(bar(P_FULL + b));
      }
      // epilogue: combine the two row-sum halves, O / l -> bf16, natural-log LSE
      float* lb = red + ((kt & 1) * 256);              // the buffer the next tile writes last
      lb[wg * 128 + r] = l;
      mbar_wait(bar(O_FULL + ob), (it >> 1) & 1);
      tc_fence_after();
      named_bar_sync(1, SM_THREADS);
      const float lt = lb[r] + lb[128 + r];
      named_bar_sync(1, SM_THREADS);
      const float inv = 1.f / lt;
      const size_t orow = ((size_t)(I.r0 + I.mt * TQ + t) * Hq + I.kh * g + hh);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float ov[32];
        tmem_ld32(o_tmem + 32 * q, ov);
        tmem_wait_ld();
        if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(out + orow * D + 64 * wg + 32 * q);
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            uint4 v;
            v.x = pack_bf16(ov[8 * ch + 0] * inv, ov[8 * ch + 1] * inv);
            v.y = pack_bf16(ov[8 * ch + 2] * inv, ov[8 * ch + 3] * inv);
            v.z = pack_bf16(ov[8 * ch + 4] * inv, ov[8 * ch + 5] * inv);
            v.w = pack_bf16(ov[8 * ch + 6] * inv, ov[8 * ch + 7] * inv);
            dst[ch] = v;
          }
        }
      }
      if (valid && lse && wg == 0) lse[orow] = (m_used + __log2f(lt)) * 0.69314718055994531f;
      tc_fence_before();
      mbar_arrive(bar(O_FREE + ob));
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

}  // namespace sm100s

static inline il_status attn_sm100s_launch(Ctx* c, uint32_t B, const int32_t* cu_q, const int32_t* prefix_len,
                                           const int32_t* block_table, const il_bf16* q, il_bf16* k_pages,
                                           il_bf16* v_pages, il_bf16* out, float* lse, float scale, cudaStream_t st) {
  namespace S = sm100s;
  const uint32_t Hq = c->cfg.n_q_heads, Hkv = c->cfg.n_kv_heads, g = Hq / Hkv, TQ = S::BM / g;
  auto enc = encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return IL_ERR_CUDA; }
  CUtensorMap tq, tk, tv;
  {
    cuuint64_t dims[3] = {S::D, Hq, c->cfg.max_suffix_tokens};
    cuuint64_t strides[2] = {S::D * 2, (cuuint64_t)Hq * S::D * 2};
    cuuint32_t box[3] = {64, g, TQ};
    cuuint32_t es[3] = {1, 1, 1};
    if (enc(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)q, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("tensor map (q) encode failed"); return IL_ERR_CUDA;
    }
  }
  for (int which = 0; which < 2; ++which) {
    cuuint64_t dims[2] = {S::D, (cuuint64_t)c->cfg.kv_pages * Hkv * BS};
    cuuint64_t strides[1] = {S::D * 2};
    cuuint32_t box[2] = {64, BS};
    cuuint32_t es[2] = {1, 1};
    if (enc(which ? &tv : &tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, which ? (void*)v_pages : (void*)k_pages, dims,
            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      set_error("tensor map (kv) encode failed"); return IL_ERR_CUDA;
    }
  }
  k_tile_scan<<<1, 1024, 0, st>>>(*c, B, cu_q, prefix_len, TQ, 0u);
  static bool attr = false;
  if (!attr) {
    IL_CUDA(cudaFuncSetAttribute(S::k_attn_sm100s, cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM_BYTES));
    attr = true;
  }
  S::k_attn_sm100s<<<c->num_sms, S::THREADS, S::SMEM_BYTES, st>>>(*c, B, cu_q, prefix_len, block_table, (__nv_bfloat16*)out,
                                                          lse, scale * 1.4426950408889634f, g, TQ, tq, tk, tv);
  IL_LAUNCH_CHECK("S::k_attn_sm100s");
  c->launches += 2;
  return IL_OK;
}

}  // namespace il
