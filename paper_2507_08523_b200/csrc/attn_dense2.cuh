// attn_dense2.cuh — the cascade's dense pass (every suffix row of the batch over the batch-shared
// prefix, P:182 / P:188-198) on a CTA PAIR: tcgen05.mma.cta_group::2, M = 256.
// A/B variant behind IL_DENSE2=1 (head dim 128); the default dense pass is k_attn_sm100 phase 3.
// Parity green (test_parity_attn_direct), but measured SLOWER: 781 vs 512 us at c3 -- every step
// hands off four times across the pair (S read and P, per tile, through cluster-scope mbarrier
// arrives after a named barrier) and the leader's issuer waits on each in turn.
//
// Why.  On one CTA the per-tile chain S -> softmax -> P (over S in TMEM) -> PV + next
// QK bounds the pass (tensor pipe ~46% busy): the next QK of a tile may only overwrite S once P is
// out of it.  Here P goes to shared memory instead (two 64-key K-major halves per tile), so S is
// free as soon as the softmax has loaded it into registers and QK(n + 1) runs during the softmax
// of step n.  Alone that would be shared-memory bound (the SS PV MMA re-reads P, the softmax writes
// it); the CTA pair halves each SM's K / V operand reads and TMA writes: each CTA holds 64 of a KV
// tile's 128 keys of K (the QK's N split) and 64 of V's 128 head dims (the PV's N split).
//
// Pair: rank 0 (leader) issues every MMA for both CTAs; each CTA keeps its own 128 rows of the two
// M-tiles A / B in its TMEM (S_A, S_B, O_A, O_B) and its own Q, P, K-half and V-half in its smem
// (same offsets in both: the MMA descriptors address each CTA's own copy).  Barriers the leader
// waits on (Q_FULL, K_FULL, V_FULL, S_READ, P_FULL, O_FREE) live in the leader and count one
// arrival (or one TMA transaction set) per CTA; barriers the CTAs wait on (S_FULL, PV_DONE, O_FULL,
// Q_FREE, K_FREE, V_FREE) live in each CTA and are signalled by multicast commits.
// Work: cluster item w = (quad u = w / Hkv of four dense M-tiles, kv head w % Hkv); rank r takes
// tiles 4u + 2r (A) and 4u + 2r + 1 (B).  KV steps = the NC 128-key tiles of request 0's pages.
#pragma once


namespace il {
namespace sm100 {
namespace d2 {

constexpr uint32_t NK = 3, NV = 3;                    // K / V ring stages (halves: 16 KB each at DH = 128)
constexpr uint32_t QT = 2 * CB;                       // Q tile: 128 rows x 128 dims (32 KB)
constexpr uint32_t HALF = 16384;                      // K half (64 keys x 128 dims), V half (128 keys x 64 dims), P half
constexpr uint32_t OFF_Q = 0, OFF_K = 2 * QT, OFF_V = OFF_K + NK * HALF, OFF_P = OFF_V + NV * HALF,
                   OFF_BAR = OFF_P + 4 * HALF;        // P: tile x half h at OFF_P + (2x + h) HALF
enum BarD : uint32_t {
  Q_FULL = 0, Q_FREE = 2, K_FULL = 4, K_FREE = K_FULL + NK, V_FULL = K_FREE + NK, V_FREE = V_FULL + NV,
  S_FULL = V_FREE + NV, S_READ = S_FULL + 2, P_FULL = S_READ + 2, PV_DONE = P_FULL + 4, O_FULL = PV_DONE + 4,
  O_FREE = O_FULL + 2, NBAR = O_FREE + 2
};
constexpr uint32_t SMEM = OFF_BAR + NBAR * 8 + 16;
static_assert(SMEM <= 232448, "smem");
// kind::f16, D f32, A / B bf16, M = 256 (cta_group::2), N = 128; QK: A, B K-major; PV: B MN-major
constexpr uint32_t IDESC_QK_D = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((256u >> 4) << 24);
constexpr uint32_t IDESC_PV_D = IDESC_QK_D | (1u << 16);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// the leader's (rank 0) copy of a shared address
__device__ __forceinline__ uint32_t to_leader(uint32_t a) {
  uint32_t p;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(p) : "r"(a), "r"(0));
  return p;
}
__device__ __forceinline__ void arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void expect_tx_cluster(uint32_t bar_cluster, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar_cluster),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(dst), "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void tma3d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
      : "memory");
}
// wait without a suspend-time hint: arrivals from the peer CTA (cluster scope) need not wake a
// suspended try_wait, which then sleeps out its whole hint
__device__ __forceinline__ void mbar_wait_c(uint32_t bar, uint32_t parity) {
  uint32_t done;
  const long long t0 = clock64();
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(bar), "r"(parity)
                 : "memory");
    if (!done && clock64() - t0 > (1ll << 34)) __trap();
  } while (!done);
}
template <uint32_t IDESC>
__device__ __forceinline__ void mma2_ss(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{ .reg .pred e, q; setp.ne.b32 q, %3, 0; elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %4, q; }" ::"r"(d_tmem), "l"(a), "l"(b), "r"(acc),
      "n"(IDESC)
      : "memory");
}
// commit to the same barrier offset in both CTAs of the pair
__device__ __forceinline__ void commit2(uint32_t bar) {
  asm volatile(
      "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1; }" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}

template <uint32_t DH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_attn_dense2(Ctx c, const int32_t* __restrict__ block_table, __nv_bfloat16* __restrict__ out, float scale_log2,
                  uint32_t g, uint32_t TQ, const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v) {
  static_assert(DH == 128, "the pair kernel is written for head dim 128");
  constexpr uint32_t D = DH;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023) != 0) __trap();
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + OFF_BAR;
  auto bar = [&](uint32_t i) { return bar0 + 8 * i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + NBAR * 8);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const uint32_t Hq = c.cfg.n_q_heads, Hkv = c.cfg.n_kv_heads;
  const uint32_t NC = c.sc->shared_blk / 8;
  const uint32_t q_total = c.sc->q_total, n_dense = c.sc->n_dense;
  const uint32_t n_items = NC ? cdiv(n_dense, 4) * Hkv : 0u;
  const uint32_t cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (uint32_t x = 0; x < 2; ++x) {
      mbar_init(bar(Q_FULL + x), 2); mbar_init(bar(Q_FREE + x), 1);
      mbar_init(bar(S_FULL + x), 1); mbar_init(bar(S_READ + x), 2);
      mbar_init(bar(O_FULL + x), 1); mbar_init(bar(O_FREE + x), 2);
      for (uint32_t h = 0; h < 2; ++h) { mbar_init(bar(P_FULL + 2 * x + h), 2); mbar_init(bar(PV_DONE + 2 * x + h), 1); }
    }
    for (uint32_t s = 0; s < NK; ++s) { mbar_init(bar(K_FULL + s), 2); mbar_init(bar(K_FREE + s), 1); }
    for (uint32_t s = 0; s < NV; ++s) { mbar_init(bar(V_FULL + s), 2); mbar_init(bar(V_FREE + s), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm_q) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm_k) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm_v) : "memory");
  }
  // each CTA allocates its TMEM for pair MMAs (cta_group::2); the same columns in both
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM (each CTA, its 128 rows): S_A [0, 128), S_B [128, 256), O_A [256, 384), O_B [384, 512)

  if (warp == 0) {
    // ============ K / V producer: this CTA's halves (K: keys 64 rank .. of the tile = pages 4 rank ..
    // 4 rank + 3, both 64-dim blocks; V: dims 64 rank .. of all 8 pages), into the leader's barriers
    IL_REGS_DEC();
    const int32_t* bt = block_table;                   // request 0's row: the batch-shared prefix
    uint32_t lc = 0;
    for (uint32_t w = cl; w < n_items; w += ncl) {
      const uint32_t kh = w % Hkv;
      for (uint32_t n = 0; n < NC; ++n, ++lc) {
        const uint32_t ks = lc % NK, vs = lc % NV;
        // lanes 0-7: K box (page 4 rank + (lane & 3), block lane >> 2); lanes 8-15: V box (page lane - 8)
        const uint32_t kp = 8 * n + 4 * rank + (lane & 3), vp = 8 * n + (lane & 7);
        const int32_t page = __ldg(bt + (lane < 8 ? kp : vp));
        const int row = (int)(((uint32_t)page * Hkv + kh) * BS);
        if (lane == 0) {
          if (lc >= NK) mbar_wait_c(bar(K_FREE + ks), (lc / NK - 1) & 1);
          expect_tx_cluster(to_leader(bar(K_FULL + ks)), HALF);
          if (lc >= NV) mbar_wait_c(bar(V_FREE + vs), (lc / NV - 1) & 1);
          expect_tx_cluster(to_leader(bar(V_FULL + vs)), HALF);
        }
        __syncwarp();
        if (lane < 8) {                                // K half: [block][4 pages x 16 keys][64 dims]
          const uint32_t p = lane & 3, h = lane >> 2;
          tma2d_pair(sbase + OFF_K + ks * HALF + h * 8192 + p * 2048, &tm_k, (int)(64 * h), row,
                     to_leader(bar(K_FULL + ks)));
        } else if (lane < 16) {                        // V half: [8 pages x 16 keys][64 dims of block rank]
          tma2d_pair(sbase + OFF_V + vs * HALF + (lane - 8) * 2048, &tm_v, (int)(64 * rank), row,
                     to_leader(bar(V_FULL + vs)));
        }
      }
    }
  } else if (warp == 2) {
    // ============ Q producer: lane x loads this CTA's M-tile x of each item
    IL_REGS_DEC();
    if (lane < 2) {
      const uint32_t x = lane;
      uint32_t ix = 0;
      for (uint32_t w = cl; w < n_items; w += ncl, ++ix) {
        const uint32_t t = 4 * (w / Hkv) + 2 * rank + x;
        if (ix >= 1) mbar_wait_c(bar(Q_FREE + x), (ix - 1) & 1);
        expect_tx_cluster(to_leader(bar(Q_FULL + x)), QT);
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h)
          tma3d_pair(sbase + OFF_Q + x * QT + h * CB, &tm_q, (int)(64 * h), (int)((w % Hkv) * g), (int)(t * TQ),
                     to_leader(bar(Q_FULL + x)));
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================= MMA issuer (leader only) =================
    IL_REGS_DEC();
    if (rank == 0) {
      const uint64_t dq0 = sdesc(sbase + OFF_Q, 16, 1024), dk0 = sdesc(sbase + OFF_K, 16, 1024);
      const uint64_t dp0 = sdesc(sbase + OFF_P, 16, 1024), dv0 = sdesc(sbase + OFF_V, 16, 1024);
      uint32_t lc = 0, st = 0, ix = 0;                   // KV loads, tile steps (per tile), items
      // PV of tile x for step s (load l): both 64-key halves of P (A from smem), V half (B)
      auto pv = [&](uint32_t x, uint32_t s, uint32_t l, bool first, bool last, uint32_t it) {
        const uint32_t vs = l % NV;
        if (first && it > 0) mbar_wait_c(bar(O_FREE + x), (it - 1) & 1);
        mbar_wait_c(bar(V_FULL + vs), (l / NV) & 1);
        const uint32_t o_tmem = tmem + 256 + 128 * x;
        mbar_wait_c(bar(P_FULL + 2 * x), s & 1);        // both P halves of the tile (one hand-off)
        tc_fence_after();
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
          const uint64_t dp = dp0 + (uint64_t)(((2 * x + h) * HALF) >> 4);
          const uint64_t dv = dv0 + (uint64_t)((vs * HALF + h * 4 * 2048) >> 4);
#pragma unroll
          for (uint32_t k = 0; k < 4; ++k)             // 16 keys per MMA: P +32 B, V +2 KB
            mma2_ss<IDESC_PV_D>(o_tmem, dp + (uint64_t)((k * 32) >> 4), dv + (uint64_t)((k * 2048) >> 4),
                                (first && h == 0 && k == 0) ? 0u : 1u);
          commit2(bar(PV_DONE + 2 * x + h));
        }
        if (last) commit2(bar(O_FULL + x));
      };
      for (uint32_t w = cl; w < n_items; w += ncl, ++ix) {
        for (uint32_t n = 0; n < NC; ++n, ++lc, ++st) {
          const uint32_t ks = lc % NK;
          mbar_wait_c(bar(K_FULL + ks), (lc / NK) & 1);
#pragma unroll
          for (uint32_t x = 0; x < 2; ++x) {
            if (n == 0) mbar_wait_c(bar(Q_FULL + x), ix & 1);
            if (st > 0) mbar_wait_c(bar(S_READ + x), (st - 1) & 1);   // S of the previous step is in registers
            tc_fence_after();
            const uint64_t dq = dq0 + (uint64_t)((x * QT) >> 4), dk = dk0 + (uint64_t)((ks * HALF) >> 4);
#pragma unroll
            for (uint32_t k = 0; k < D / 16; ++k)
              mma2_ss<IDESC_QK_D>(tmem + 128 * x, dq + (uint64_t)(((k >> 2) * CB + (k & 3) * 32) >> 4),
                                  dk + (uint64_t)(((k >> 2) * 8192 + (k & 3) * 32) >> 4), k ? 1u : 0u);
            commit2(bar(S_FULL + x));
            if (n + 1 == NC) commit2(bar(Q_FREE + x));
          }
          commit2(bar(K_FREE + ks));
          if (n > 0) {                                   // PV of step n - 1 (its softmax overlapped these QKs)
#pragma unroll
            for (uint32_t x = 0; x < 2; ++x) pv(x, st - 1, lc - 1, n == 1, false, ix);
            commit2(bar(V_FREE + (lc - 1) % NV));
          }
          if (n + 1 == NC) {                             // the item's last PV
#pragma unroll
            for (uint32_t x = 0; x < 2; ++x) pv(x, st, lc, NC == 1, true, ix);
            commit2(bar(V_FREE + lc % NV));
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    IL_REGS_DEC();                                      // (no role: its registers go to the softmax warps)
  } else if (warp >= 4) {
    // ====== softmax + epilogue: warpgroup x = this CTA's M-tile x, thread = row r ======
    IL_REGS_INC();
    const uint32_t sm_t = threadIdx.x - 128, xo = sm_t >> 7, r = sm_t & 127, q4 = warp & 3;
    const uint32_t lane_addr = (32 * q4) << 16;
    const uint32_t s_tmem = tmem + lane_addr + 128 * xo, o_tmem = tmem + lane_addr + 256 + 128 * xo;
    const uint32_t t = r / g, hh = r % g;
    const uint32_t p_row = sbase + OFF_P + 2 * xo * HALF + r * 128;   // this row's 128 B in each P half
    uint32_t st = 0, it = 0;
    for (uint32_t w = cl; w < n_items; w += ncl, ++it) {
      const uint32_t tile = 4 * (w / Hkv) + 2 * rank + xo, kh = w % Hkv;
      const uint32_t r0 = tile * TQ, ntok = r0 < q_total ? min(TQ, q_total - r0) : 0u;
      const bool valid = (r < g * TQ) && (t < ntok);
      const size_t orow = (size_t)(r0 + t) * Hq + kh * g + hh;
      float m_used = -INFINITY, l = 0.f;
      for (uint32_t n = 0; n < NC; ++n, ++st) {
        mbar_wait_c(bar(S_FULL + xo), st & 1);
        tc_fence_after();
        float a[128];
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_ld32(s_tmem + 32 * q, *reinterpret_cast<float(*)[32]>(&a[32 * q]));
        tmem_wait_ld();
        tc_fence_before();
        // S is in registers: the leader may compute the next step's S into these columns
        __syncwarp(); asm volatile("barrier.sync %0, 128;" ::"r"(1 + xo) : "memory");
        if (r == 0) arrive_cluster(to_leader(bar(S_READ + xo)));
        float mxa[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mxa[q] = a[q];
#pragma unroll
        for (int j = 8; j < 128; ++j) mxa[j & 7] = fmaxf(mxa[j & 7], a[j]);
        const float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                               fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
        const float mx2 = mx * scale_log2;
        bool need = false;
        float factor = 1.f;
        if (m_used == -INFINITY) {
          m_used = mx2;
        } else if (mx2 > m_used + 8.f) {
          need = true;
          factor = ex2(m_used - mx2);
          m_used = mx2;
          l *= factor;
        }
        if (__any_sync(~0u, need)) {
          // rescale O once the previous step's PV (both halves) has landed
          mbar_wait_c(bar(PV_DONE + 2 * xo + 1), (st - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int q = 0; q < (int)(D / 32); ++q) {
            float ov[32];
            tmem_ld32(o_tmem + 32 * q, ov);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] *= factor;
            tmem_st32(o_tmem + 32 * q, ov);
          }
          tmem_wait_st();
          tc_fence_before();
        }
        const float negm = -m_used;
        float rsa[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t pk[32];
#pragma unroll
          for (int jj = 0; jj < 64; jj += 2) {
            const int j = 64 * h + jj;
            float x0, x1;
            ffma2(x0, x1, a[j], a[j + 1], scale_log2, negm);
            const float p0 = ex2(x0), p1 = ex2(x1);
            fadd2(rsa[(j >> 1) & 2], rsa[((j >> 1) & 2) + 1], p0, p1);
            pk[jj >> 1] = pack_bf16(p0, p1);
          }
          // the previous step's PV of this half has read its P: overwrite it (K-major, 128 B swizzle:
          // 16-byte chunk q of row r at q ^ (r & 7))
          if (st > 0) mbar_wait_c(bar(PV_DONE + 2 * xo + h), (st - 1) & 1);
          const uint32_t dst = p_row + h * HALF;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst + ((q ^ (r & 7)) << 4)), "r"(pk[4 * q]),
                         "r"(pk[4 * q + 1]), "r"(pk[4 * q + 2]), "r"(pk[4 * q + 3])
                         : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");     // generic-proxy writes -> the tensor core
        __syncwarp(); asm volatile("barrier.sync %0, 128;" ::"r"(1 + xo) : "memory");
        if (r == 0) arrive_cluster(to_leader(bar(P_FULL + 2 * xo)));
        l += (rsa[0] + rsa[1]) + (rsa[2] + rsa[3]);
      }
      // epilogue: O / l (bf16) and m + log2 l: the partial k_attn_p2 merges
      mbar_wait_c(bar(O_FULL + xo), it & 1);
      tc_fence_after();
      {
        const float inv = 1.f / l;
#pragma unroll
        for (int q = 0; q < (int)(D / 32); ++q) {
          float ov[32];
          tmem_ld32(o_tmem + 32 * q, ov);
          tmem_wait_ld();
          if (valid) store_row32(out + orow * D + 32 * q, ov, inv);
        }
        if (valid) c.attn_ml[orow] = m_used + __log2f(l);
      }
      tc_fence_before();
      __syncwarp(); asm volatile("barrier.sync %0, 128;" ::"r"(1 + xo) : "memory");
      if (r == 0) arrive_cluster(to_leader(bar(O_FREE + xo)));
    }
  }
  tc_fence_before();
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

}  // namespace d2
}  // namespace sm100
}  // namespace il
