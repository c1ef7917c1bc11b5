// attn_p2.cuh — cascade phase 2 of the prefill attention (each request's own KV range past the
// batch-shared prefix: its cached demonstrations, then its own suffix keys under the causal
// mask) on 64-key KV steps with a DOUBLE-BUFFERED S per Q tile.  It runs
// after the dense pass over the shared prefix (k_attn_sm100 phase 3) and merges that pass's
// partial (O / l, m + log2 l) into each row in its epilogue, writing the result and the LSE.
//
// Why a kernel of its own.  Phase 2 items are short (~2.4 128-key tiles per
// M-tile at c3), so the per-tile chain of the shared kernel -- QK -> softmax -> (P aliases S)
// PV -> next QK -> ... -- is the whole story there: with one S buffer per tile the next QK can
// only be issued after the softmax has released P, and the tensor pipe idles (~20% busy).  Here
// each Q tile owns two 64-column S buffers (TMEM: S0, S1, O per tile = 64 + 64 + 128 columns,
// two tiles = 512), so QK of step n+1 runs while the softmax of step n does; P of step n is
// written over the first 32 columns of its buffer and PV(n) must be issued before QK(n+2)
// overwrites that buffer (tcgen05 ops of one thread execute in order).  64-key steps also halve
// the keys computed past the causal diagonal.  (The QK MMA at N = 64 runs at 2/3 of the N = 128
// rate -- SS mode reads Q's 4 KB per MMA from smem either way -- which phase 1, tensor bound,
// could not afford; phase 2 is chain bound.)
//
// Work: the two Q tiles of a CTA are two independent PIPELINES (streams) x = 0 / 1, each with
// its own Q buffer, K / V rings, TMA producer warp and MMA issuer warp; they share only the tensor
// pipe and the SM's issue slots.  Stream x takes items w = blockIdx.x + k gridDim.x; item w = M-tile
// tile_of(w, x) (the x-th of pair w / Hkv, pairs walked from the last one: IL_P2_REV) with kv head
// w % Hkv; a tile is decoded from one 16-byte k_tile_scan descriptor read one item ahead.  Warp
// roles: warp 2x = producer of stream x (Q, K and V TMAs; warp 2 also allocates TMEM), warp 2x + 1
// = MMA issuer of stream x, warps 4-7 / 8-11 = softmax of stream 0 / 1, warps 12-15 / 16-19 =
// epilogue of stream 0 / 1 (l and m handed over through smem; O read into registers and released
// before the dense pass's partial is read and merged).  The issuer's order per step s of an item is
// QK(s), then PV(s - 1) (so the softmax of step s - 1 overlaps QK(s)), and PV(last) right after the
// item's last QK; QK(s) overwrites the S buffer of step s - 2, whose PV precedes it.
// DENSE = true (an A / B variant, IL_DENSE_P2=1) runs the dense pass itself on this design.
#pragma once
// (included from attn_sm100.cuh after namespace sm100: uses its PTX wrappers, Tile and decode_tile)

namespace il {
namespace sm100 {
namespace p2 {

constexpr uint32_t BN2 = 64;                      // keys per KV step
#ifndef IL_P2_REV
#define IL_P2_REV 1
#endif
#ifndef IL_P2_SKIP_PAD
#define IL_P2_SKIP_PAD 0                          // (1: measured slower, 245 -> 255 us; also with P = 0 stored)
#endif
constexpr uint32_t KCB2 = BN2 * 128;              // one 64-column block of a 64-key K / V tile (8 KB)
// per-stream K / V ring depths (64-key tiles): head dim 128 fills 224 KB with (2, 3)
#ifndef IL_P2_NSTK
#define IL_P2_NSTK 2
#endif
#ifndef IL_P2_NSTV
#define IL_P2_NSTV 3
#endif
// bit (j / 2) % 8 set: exponential pair j of a row computed by the cubic on the FMA pipe (the two
// streams' softmax warps share each SMSP's MUFU)
#ifndef IL_P2_EMU
#define IL_P2_EMU 0
#endif
template <uint32_t DH> constexpr uint32_t NK2 = DH == 128 ? IL_P2_NSTK : 2 * IL_P2_NSTK;
template <uint32_t DH> constexpr uint32_t NV2 = DH == 128 ? IL_P2_NSTV : 2 * IL_P2_NSTV;
// smem per stream (NCB = DH / 64): Q NCB x 16 KB | K ring | V ring (NCB x 8 KB per 64-key tile); barriers after both
template <uint32_t DH> constexpr uint32_t stream_bytes2 = (CB + (NK2<DH> + NV2<DH>) * KCB2) * (DH / 64);
// per stream: Q_FULL, Q_FREE, S_FULL x 2, P_FULL x 2, PV_DONE, O_FULL, O_FREE, K_FULL / K_FREE, V_FULL / V_FREE
enum Bar2 : uint32_t { Q_FULL2 = 0, Q_FREE2, S_FULL2, P_FULL2 = S_FULL2 + 2, PV_DONE2 = P_FULL2 + 2, O_FULL2, O_FREE2, L_READY2,
                       K_RING2 };
template <uint32_t DH> constexpr uint32_t nbar2 = K_RING2 + 2 * (NK2<DH> + NV2<DH>);
// + the row sums / maxima the softmax warps hand to the epilogue warps (2 streams x 128 float2)
template <uint32_t DH> constexpr uint32_t smem_bytes2 = 2 * stream_bytes2<DH> + 2 * nbar2<DH> * 8 + 64 + 2048;
// warps 0-3 producers / issuers, 4-11 softmax, 12-19 epilogue (stream x: 12 + 4x .. 15 + 4x)
constexpr int THREADS2 = 640;
// register split (setmaxnreg, per warpgroup): the launch gives every thread REGS2_LAUNCH (ptxas'
// cap for 640 threads; attn_setup checks the compiled count, since setmaxnreg.inc waits for the
// CTA's pool to hold the request), producers / issuers and epilogue warps give some back, the
// softmax warps (a 64-key row + its P) take it
constexpr int REGS2_LAUNCH = 96, REGS2_PROD = 56, REGS2_EPI = 96, REGS2_SM = 112;   // (EPI = LAUNCH: no setmaxnreg)
static_assert(4 * REGS2_PROD + 8 * REGS2_EPI + 8 * REGS2_SM <= 20 * REGS2_LAUNCH, "register split exceeds the pool");

// S = Q K^T at N = 64 keys; O += P V as in k_attn_sm100 (K = 16 keys per MMA, 4 per step)
constexpr uint32_t IDESC_QK2 = (1u << 4) | (1u << 7) | (1u << 10) | ((BN2 >> 3) << 17) | ((BM >> 4) << 24);

// A phase-2 M-tile from its k_tile_scan descriptor {request, position of its first suffix token,
// its first suffix row, ntok | nblk << 8}: one 16-byte load, no dependent loads.
struct TD {
  uint32_t i, pos0, row0, ntok, nblk;
};
__device__ __forceinline__ TD unpack(uint4 d) { return TD{d.x, d.y, d.z, d.w & 0xFFu, d.w >> 8}; }
// 64-key steps of a tile: key tiles 2 NC .. (position of its last row) / 64
__device__ __forceinline__ uint32_t n_steps(uint4 d, uint32_t NC) { return (d.y + (d.w & 0xFFu) - 1) / BN2 + 1 - 2 * NC; }

// DENSE = false: phase 2 (each request's own M-tiles over its keys past the shared prefix, merging
// the dense pass's partial).  DENSE = true: the dense pass itself (phase 3) -- M-tiles of TQ
// consecutive suffix rows of the batch (rows of several requests) over the batch-shared prefix
// (request 0's pages, 2 NC 64-key steps, no causal mask: every suffix position lies past it),
// writing the partial (O / l, m + log2 l).  There the two streams process M-tiles 2u and 2u + 1
// of the same kv head, i.e. the SAME K / V tiles: one producer warp fills K / V rings both issuers
// read (twice as deep; each slot is released by both), warp 2 loads both Q tiles.
template <uint32_t DH, bool DENSE>
__global__ void __launch_bounds__(THREADS2, 1)
    k_attn_p2(Ctx c, uint32_t B, const int32_t* __restrict__ block_table, __nv_bfloat16* __restrict__ out,
              float* __restrict__ lse, float scale_log2, uint32_t g, uint32_t TQ, const __grid_constant__ CUtensorMap tm_q,
              const __grid_constant__ CUtensorMap tm_o, const __grid_constant__ CUtensorMap tm_k,
              const __grid_constant__ CUtensorMap tm_v) {
  constexpr uint32_t D = DH, NCB = DH / 64, NB = nbar2<DH>;
  // ring depths: per stream, or (DENSE) one pair of rings twice as deep shared by both streams
  constexpr uint32_t NK = DENSE ? 2 * NK2<DH> : NK2<DH>, NV = DENSE ? 2 * NV2<DH> : NV2<DH>;
  constexpr uint32_t RB = 2 * (NK2<DH> + NV2<DH>);                // ring barriers per stream block
  constexpr uint32_t QTILE = NCB * CB, KVT = NCB * KCB2, SB = stream_bytes2<DH>;
  constexpr uint32_t OFF_K = QTILE, OFF_V = OFF_K + NK2<DH> * KVT;      // within a stream's region
  static_assert(DH == 64 || DH == 128, "head dim");
  static_assert(OFF_V + NV2<DH> * KVT == SB && smem_bytes2<DH> <= 232448, "smem map");
  static_assert(!DENSE || 2 * QTILE + (NK + NV) * KVT == 2 * SB, "DENSE smem map");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023) != 0) __trap();
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + 2 * SB;
  // barrier idx of stream x
  auto bar = [&](uint32_t x, uint32_t idx) { return bar0 + 8 * (x * NB + idx); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 2 * SB + 2 * NB * 8);
  float2* s_lm = reinterpret_cast<float2*>(smem + 2 * SB + 2 * NB * 8 + 64);   // [stream][row] (l, m)

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t Hq = c.cfg.n_q_heads, Hkv = c.cfg.n_kv_heads;
  const uint32_t NC = c.sc->shared_blk / 8;             // 128-key tiles of the batch-shared prefix
  const uint32_t q_total = c.sc->q_total;
  // M-tiles: phase-2 tiles, or (DENSE) the dense tiles rounded up to an even count (a padding tile
  // has no rows: its outputs are never written)
  const uint32_t ntl = DENSE ? cdiv(c.sc->n_dense, 2) * 2 : c.sc->n_tiles;
  // (DENSE with no batch-shared prefix, NC = 0: nothing to do -- every item would have no steps)
  const uint32_t n_items = DENSE && NC == 0 ? 0u : cdiv(ntl, 2) * Hkv;
  const uint4* desc = c.tile_desc;
  const bool merge = !DENSE && NC > 0;                  // the dense pass (phase 3) left a partial of every row
  const uint32_t kt0 = DENSE ? 0u : 2 * NC;             // first 64-key tile
  // tile t's descriptor {request, first position, first suffix row, ntok | nblk << 8}; the dense
  // tiles' rows lie past the shared prefix whatever their request (position 2^30: no mask)
  auto tdesc = [&](uint32_t t) -> uint4 {
    if (DENSE) {
      const uint32_t r0 = t * TQ, nt = r0 < q_total ? min(TQ, q_total - r0) : 0u;
      return make_uint4(0u, 1u << 30, r0, nt | ((8 * NC) << 8));
    }
    IL_CHECK(t < c.sc->n_tiles);
    return __ldg(desc + t);
  };
  auto nsteps = [&](const uint4& dd) -> uint32_t { return DENSE ? 2 * NC : n_steps(dd, NC); };
  // item ww of stream x -> M-tile: pair ww / Hkv, walked from the LAST pair when IL_P2_REV (phase 2:
  // the dense pass wrote its last rows' partials last, so they are still in L2 when this starts)
  // (stream x's tiles are x, x + 2, ..: nx = (ntl + 1 - x) / 2 of them; reversed, u -> nx - 1 - u, so
  // that the items past the end stay the last ones and the streams' loops can stop at the first)
  auto tile_of = [&](uint32_t ww, uint32_t x) -> uint32_t {
    const uint32_t u = ww / Hkv, nx = (ntl + 1 - x) / 2;
    return (IL_P2_REV && !DENSE) ? (u < nx ? 2 * (nx - 1 - u) + x : ntl) : 2 * u + x;
  };
  // ring barrier i: the stream's own block, or (DENSE) both streams' blocks as one
  auto rbar = [&](uint32_t x, uint32_t i) {
    return DENSE ? (i < RB ? bar(0, K_RING2 + i) : bar(1, K_RING2 + i - RB)) : bar(x, K_RING2 + i);
  };
  static_assert(!DENSE || 2 * (NK + NV) == 2 * RB, "shared rings use both streams' barrier blocks");
  constexpr uint32_t phase = 2;                         // (IL_TRACE: trace builds with IL_TRACE_PHASE=2)
  (void)phase;

  if (threadIdx.x == 0) {
    for (uint32_t x = 0; x < 2; ++x) {
      mbar_init(bar(x, Q_FULL2), 1); mbar_init(bar(x, Q_FREE2), 1);
      mbar_init(bar(x, PV_DONE2), 1); mbar_init(bar(x, O_FULL2), 1); mbar_init(bar(x, O_FREE2), 128);
      mbar_init(bar(x, L_READY2), 128);
      for (uint32_t b = 0; b < 2; ++b) { mbar_init(bar(x, S_FULL2 + b), 1); mbar_init(bar(x, P_FULL2 + b), 128); }
      for (uint32_t i = 0; i < RB; ++i) mbar_init(bar(x, K_RING2 + i), 1);
    }
    if (DENSE)                                          // shared K_FREE / V_FREE: released by both issuers
      for (uint32_t i = 0; i < NK + NV; ++i) {
        const uint32_t j = i < NK ? NK + i : 2 * NK + NV + (i - NK);
        const uint32_t b = j < RB ? bar(0, K_RING2 + j) : bar(1, K_RING2 + j - RB);
        mbar_init(b, 2);
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
  // TMEM columns of stream x: S0 [256x, +64), S1 [256x + 64, +64), O [256x + 128, +128)

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGS2_PROD));
    const uint32_t x = warp >> 1;                       // this warp's stream
    // smem: Q of stream x, its K / V rings (DENSE: Q0 | Q1 | the shared K ring | the shared V ring)
    const uint32_t sq = DENSE ? sbase + x * QTILE : sbase + x * SB;
    const uint32_t sk = DENSE ? sbase + 2 * QTILE : sq + OFF_K, sv = DENSE ? sk + NK * KVT : sq + OFF_V;
    // ring barriers: K_FULL [0, NK), K_FREE [NK, 2NK), V_FULL, V_FREE
    auto kfull = [&](uint32_t i) { return rbar(x, i); };
    auto kfree = [&](uint32_t i) { return rbar(x, NK + i); };
    auto vfull = [&](uint32_t i) { return rbar(x, 2 * NK + i); };
    auto vfree = [&](uint32_t i) { return rbar(x, 2 * NK + NV + i); };
    auto ok = [&](uint32_t ww) { return ww < n_items && tile_of(ww, x) < ntl; };
    auto ld = [&](uint32_t ww) { return tdesc(tile_of(ww, x)); };
    uint32_t w = blockIdx.x;
    uint4 d = ok(w) ? ld(w) : make_uint4(0, 0, 0, 0);
    if (DENSE && warp == 2) {
      // ============ (DENSE) Q producer: lane xq loads stream xq's Q tile of each item
      if (lane < 2) {
        const uint32_t xq = lane, qbytes = 2 * D * g * TQ, sqx = sbase + xq * QTILE;
        auto okq = [&](uint32_t ww) { return ww < n_items && tile_of(ww, xq) < ntl; };
        uint32_t ix = 0, wq = blockIdx.x;
        uint4 dl = okq(wq) ? tdesc(tile_of(wq, xq)) : make_uint4(0, 0, 0, 0);
        for (; okq(wq); wq += gridDim.x, ++ix) {
          const uint32_t wn = wq + gridDim.x;
          const uint4 dn = okq(wn) ? tdesc(tile_of(wn, xq)) : dl;
          if (ix >= 1) mbar_wait(bar(xq, Q_FREE2), (ix - 1) & 1);
          mbar_expect_tx(bar(xq, Q_FULL2), qbytes);
#pragma unroll
          for (uint32_t h = 0; h < NCB; ++h)
            tma_load_3d(sqx + h * CB, &tm_q, (int)(64 * h), (int)((wq % Hkv) * g), (int)dl.z, bar(xq, Q_FULL2));
          if (okq(wn)) {
#pragma unroll
            for (uint32_t h = 0; h < NCB; ++h) tma_prefetch_3d(&tm_q, (int)(64 * h), (int)((wn % Hkv) * g), (int)dn.z);
          }
          dl = dn;
        }
      }
      __syncwarp();
    } else if ((warp & 1) == 0) {
      // ============ producer of stream x: Q of each item, then its K / V tiles (64 keys = 4 pages);
      // (DENSE: warp 0, K / V only, for both streams -- their items share kv head and pages).
      // The page ids of an item's first 8 steps are read one item ahead, lane l holding step
      // l / 4's page l % 4 (the block tables are written by il_prefix_match and are usually out of
      // L2 by now: a per-step read sat on the critical path); descriptors are read two items ahead.
      const uint32_t qbytes = 2 * D * g * TQ;
      auto page_at = [&](const uint4& dd, uint32_t kt, uint32_t p) -> int32_t {
        const uint32_t blk = kt * 4 + p;
#ifdef IL_P2_SAME_PAGES
        return __ldg(block_table + (blk < (dd.w >> 8) ? blk : 0u));   // profiling variant: every tile reads request 0's pages
#else
        IL_CHECK(dd.x < B && (dd.w >> 8) <= c.max_blocks);
        const int32_t pg = __ldg(block_table + (size_t)dd.x * c.max_blocks + (blk < (dd.w >> 8) ? blk : 0u));
        IL_CHECK(pg >= 0 && (uint32_t)pg < c.cfg.kv_pages);
        return pg;
#endif
      };
      auto pages_of = [&](const uint4& dd) -> int32_t {
        return (lane >> 2) < nsteps(dd) ? page_at(dd, kt0 + (lane >> 2), lane & 3) : 0;
      };
      uint32_t s = 0, ix = 0;
      uint4 dn = ok(w + gridDim.x) ? ld(w + gridDim.x) : d;
      int32_t pg = ok(w) ? pages_of(d) : 0;
      while (ok(w)) {
        const uint32_t wn = w + gridDim.x;
        const uint4 dnn = ok(wn + gridDim.x) ? ld(wn + gridDim.x) : dn;
        const int32_t pgn = ok(wn) ? pages_of(dn) : 0;
        const uint32_t kh = w % Hkv, nst = nsteps(d);
        if (!DENSE && lane == 0) {
          if (ix >= 1) mbar_wait(bar(x, Q_FREE2), (ix - 1) & 1);
          mbar_expect_tx(bar(x, Q_FULL2), qbytes);
          IL_TRACE(12 + x, ix & 4095);
#pragma unroll
          for (uint32_t h = 0; h < NCB; ++h)
            tma_load_3d(sq + h * CB, &tm_q, (int)(64 * h), (int)(kh * g), (int)d.z, bar(x, Q_FULL2));
          if (ok(wn)) {                                 // the next item's Q (and the partial it merges) into L2
#pragma unroll
            for (uint32_t h = 0; h < NCB; ++h) {
              tma_prefetch_3d(&tm_q, (int)(64 * h), (int)((wn % Hkv) * g), (int)dn.z);
              if (merge) tma_prefetch_3d(&tm_o, (int)(64 * h), (int)((wn % Hkv) * g), (int)dn.z);
            }
          }
        }
        for (uint32_t j = 0; j < nst; ++j, ++s) {
          const int32_t page = j < 8 ? __shfl_sync(~0u, pg, 4 * j + (lane & 3)) : page_at(d, kt0 + j, lane & 3);
          const int row = (int)(((uint32_t)page * Hkv + kh) * BS);
          const uint32_t ks = s % NK, vs = s % NV;
          if (lane == 0) {
            if (s >= NK) mbar_wait(kfree(ks), (s / NK - 1) & 1);
#ifndef IL_P2_TRACE_SM
            IL_TRACE(2 * x, s & 4095);
#endif
#ifdef IL_P2_NO_KV
            mbar_arrive(kfull(ks));                    // profiling variant: no K / V loads
#else
            mbar_expect_tx(kfull(ks), KVT);
#endif
          }
          __syncwarp();
#ifndef IL_P2_NO_KV
          if (lane < 4 * NCB)                          // lane = (page, 64-column block)
            tma_load_2d(sk + ks * KVT + (lane >> 2) * KCB2 + (lane & 3) * 2048, &tm_k, (int)(64 * (lane >> 2)), row,
                        kfull(ks));
#endif
          if (lane == 0) {
            if (s >= NV) mbar_wait(vfree(vs), (s / NV - 1) & 1);
#ifndef IL_P2_TRACE_SM
            IL_TRACE(2 * x + 1, s & 4095);
#endif
#ifdef IL_P2_NO_KV
            mbar_arrive(vfull(vs));
#else
            mbar_expect_tx(vfull(vs), KVT);
#endif
          }
          __syncwarp();
#ifndef IL_P2_NO_KV
          if (lane < 4 * NCB)
            tma_load_2d(sv + vs * KVT + (lane >> 2) * KCB2 + (lane & 3) * 2048, &tm_v, (int)(64 * (lane >> 2)), row,
                        vfull(vs));
#endif
        }
        ++ix;
        w = wn;
        d = dn;
        dn = dnn;
        pg = pgn;
      }
    } else {
      // ================= MMA issuer of stream x (warp-uniform, one elected lane issues) ==========
      const uint64_t dq = sdesc(sq, 16, 1024);
      const uint64_t dk0 = sdesc(sk, 16, 1024), dv0 = sdesc(sv, KCB2, 1024);
      const uint32_t o_tmem = tmem + 256 * x + 128;
      uint32_t s = 0, it = 0;
      // PV of step p (first / last: its item's first / last step; the item's index it_p)
      auto pv = [&](uint32_t p, bool first, bool last, uint32_t it_p) {
        const uint32_t vs = p % NV;
        if (first && it_p > 0) mbar_wait(bar(x, O_FREE2), (it_p - 1) & 1);   // previous epilogue read O
        mbar_wait(bar(x, P_FULL2 + (p & 1)), (p >> 1) & 1);
        mbar_wait(vfull(vs), (p / NV) & 1);
        tc_fence_after();
        if (lane == 0) IL_TRACE(8 + x, p & 4095);
        const uint64_t dv = dv0 + (uint64_t)((vs * KVT) >> 4);
        const uint32_t p_tmem = tmem + 256 * x + 64 * (p & 1);
#pragma unroll
        for (uint32_t k = 0; k < BN2 / 16; ++k)
          mma_ts_w<IDESC_PV_T<DH>>(o_tmem, p_tmem + 8 * k, dv + (uint64_t)((k * 2048) >> 4), (first && k == 0) ? 0u : 1u);
        commit_w(bar(x, PV_DONE2));
        if (last) commit_w(bar(x, O_FULL2));
        commit_w(vfree(vs));
      };
      while (ok(w)) {
        const uint32_t wn = w + gridDim.x;
        const uint4 dn = ok(wn) ? ld(wn) : d;
        const uint32_t nst = nsteps(d);
        for (uint32_t j = 0; j < nst; ++j, ++s) {
          if (j == 0) mbar_wait(bar(x, Q_FULL2), it & 1);
          const uint32_t ks = s % NK, b = s & 1;
          mbar_wait(kfull(ks), (s / NK) & 1);
          tc_fence_after();
          if (lane == 0) IL_TRACE(6 + x, s & 4095);
          const uint64_t dk = dk0 + (uint64_t)((ks * KVT) >> 4);
#pragma unroll
          for (uint32_t k = 0; k < D / 16; ++k)
            mma_ss_w<IDESC_QK2>(tmem + 256 * x + 64 * b, dq + (uint64_t)(((k >> 2) * CB + (k & 3) * 32) >> 4),
                                dk + (uint64_t)(((k >> 2) * KCB2 + (k & 3) * 32) >> 4), k ? 1u : 0u);
          commit_w(bar(x, S_FULL2 + b));
          commit_w(kfree(ks));
          if (j + 1 == nst) commit_w(bar(x, Q_FREE2));  // the item's last QK has read Q
          if (j >= 1) pv(s - 1, j == 1, false, it);      // the softmax of step s - 1 overlapped QK(s)
          if (j + 1 == nst) pv(s, nst == 1, true, it);   // the item's last PV: its epilogue may start
        }
        ++it;
        w = wn;
        d = dn;
      }
    }
  } else if (warp >= 12) {
    // ====== epilogue of stream xe (warps 12 + 4 xe .. 15 + 4 xe): thread = row r, TMEM lane r.
    // merged O / L -> bf16 row of `out` and the LSE.  The softmax warps
    // hand l and m over through smem and go on with the next item; O is released (O_FREE) for the
    // next item's first PV once read.
    const uint32_t xe = (warp - 12) >> 2, q4 = warp & 3, r = 32 * q4 + lane;
    const uint32_t o_tmem = tmem + ((32 * q4) << 16) + 256 * xe + 128;
    const uint32_t t = r / g, hh = r % g;
    auto ok = [&](uint32_t ww) { return ww < n_items && tile_of(ww, xe) < ntl; };
    auto ld = [&](uint32_t ww) { return tdesc(tile_of(ww, xe)); };
    uint32_t w = blockIdx.x, it = 0;
    uint4 dcur = ok(w) ? ld(w) : make_uint4(0, 0, 0, 0);
    while (ok(w)) {
      const uint32_t wn = w + gridDim.x;
      const uint4 dn = ok(wn) ? ld(wn) : dcur;
      const TD T = unpack(dcur);
      const bool valid = (r < g * TQ) && (t < T.ntok);
      const size_t orow = (size_t)(T.row0 + t) * Hq + (w % Hkv) * g + hh;
      mbar_wait(bar(xe, L_READY2), it & 1);
      const float2 lm = s_lm[128 * xe + r];             // (l, m) of this row's own part
      // merge with the dense pass's partial (O1 / l1 in `out`, m1 + log2 l1 in attn_ml):
      // M = max(m, ml1), O = (O2 2^(m - M) + O1n 2^(ml1 - M)) / (l 2^(m - M) + 2^(ml1 - M))
      const float ml1 = merge && valid ? c.attn_ml[orow] : -INFINITY;
      const float mm = fmaxf(lm.y, ml1), a2 = ex2(lm.y - mm), a1 = ex2(ml1 - mm);
      const float L = lm.x * a2 + a1, inv = 1.f / L;
      const __nv_bfloat16* prow = out + orow * D;
      const bool mv = merge && valid;
      // O (scaled, as bf16 pairs) into registers, then O is released for the next item's first PV
      // before the partial is read and added: the merge's loads stay off the stream's chain
      uint32_t ob[D / 2];
      mbar_wait(bar(xe, O_FULL2), it & 1);
      tc_fence_after();
      const float s2 = a2 * inv, s1 = a1 * inv;
#pragma unroll
      for (int q = 0; q < (int)(D / 32); ++q) {
        float ov[32];
        tmem_ld32(o_tmem + 32 * q, ov);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) ob[16 * q + j] = pack_bf16(ov[2 * j] * s2, ov[2 * j + 1] * s2);
      }
      tc_fence_before();
      if (r == 0) IL_TRACE(14 + xe, it & 4095);
      mbar_arrive(bar(xe, O_FREE2));
#pragma unroll
      for (int h = 0; h < (int)(D / 16); ++h) {         // 16 columns = one 256-bit access
        uint32_t w8[8];
        if (mv) {
          uint32_t pc[8];
          ld_v8_nv(prow + 16 * h, pc);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t u = ob[8 * h + e];
            w8[e] = pack_bf16(__uint_as_float(u << 16) + __uint_as_float(pc[e] << 16) * s1,
                              __uint_as_float(u & 0xFFFF0000u) + __uint_as_float(pc[e] & 0xFFFF0000u) * s1);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) w8[e] = ob[8 * h + e];
        }
#ifdef IL_P2_NO_EPI
        if (valid && w8[0] == 12345u)                  // profiling variant: no output stores
#else
        if (valid)
#endif
        {
          IL_CHECK(orow < (size_t)q_total * Hq && T.row0 + T.ntok <= q_total);
          st_v8(out + orow * D + 16 * h, w8);
        }
      }
      if (valid) {
        if (DENSE) c.attn_ml[orow] = mm + __log2f(L);    // the partial the phase-2 kernel merges
        else if (lse) lse[orow] = (mm + __log2f(L)) * 0.69314718055994531f;
      }
      ++it;
      w = wn;
      dcur = dn;
    }
  } else {
    // ====== softmax, one warpgroup per stream: thread = row r of its Q tile ======
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS2_SM));
    const uint32_t sm_t = threadIdx.x - 128, xo = sm_t >> 7, r = sm_t & 127, q4 = warp & 3;
    const uint32_t lane_addr = (32 * q4) << 16;
    const uint32_t s_tmem = tmem + lane_addr + 256 * xo, o_tmem = s_tmem + 128;
    const uint32_t t = r / g;
    uint32_t it = 0, cs = 0;
    auto ok = [&](uint32_t ww) { return ww < n_items && tile_of(ww, xo) < ntl; };
    auto ld = [&](uint32_t ww) { return tdesc(tile_of(ww, xo)); };
    uint32_t w = blockIdx.x;
    uint4 dcur = ok(w) ? ld(w) : make_uint4(0, 0, 0, 0);
    while (ok(w)) {
      const uint32_t wn = w + gridDim.x;
      const uint4 dn = ok(wn) ? ld(wn) : dcur;         // (used at the next item: the load runs meanwhile)
      const TD T = unpack(dcur);
      const uint32_t pos_q = T.pos0 + min(t, T.ntok - 1);
      const uint32_t nst = nsteps(dcur);
      float m_used = -INFINITY, l = 0.f;
#if IL_P2_SKIP_PAD
      const bool pad_warp = 32 * q4 >= g * T.ntok;         // (warp-uniform)
#endif
      for (uint32_t n = 0; n < nst; ++n, ++cs) {
        const uint32_t b = cs & 1u, sb = s_tmem + 64 * b;
        mbar_wait(bar(xo, S_FULL2 + b), (cs >> 1) & 1);
        tc_fence_after();
        if (r == 0) IL_TRACE(4 + xo, cs & 4095);
#if IL_P2_SKIP_PAD
        if (pad_warp) {
          // every row of this warp is padding (rows >= g ntok): its P only feeds output rows nobody
          // writes, so the warp skips the softmax (the other stream's warps get the SMSP's MUFU)
          mbar_arrive(bar(xo, P_FULL2 + b));
          continue;
        }
#endif
#ifdef IL_P2_NO_SM
        {   // profiling variant: P = 0 without touching S
          uint32_t z[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) z[j] = 0u;
          tmem_st32u(sb, z);
          tmem_wait_st();
          tc_fence_before();
          if (r == 0) IL_TRACE(10 + xo, cs & 4095);
          mbar_arrive(bar(xo, P_FULL2 + b));
          l = 1.f; m_used = 0.f;
          continue;
        }
#endif
        float a[64];
        tmem_ld32(sb, *reinterpret_cast<float(*)[32]>(&a[0]));
        tmem_ld32(sb + 32, *reinterpret_cast<float(*)[32]>(&a[32]));
        tmem_wait_ld();
#ifdef IL_P2_TRACE_SM
        if (r == 0 && xo == 0) IL_TRACE(0, cs & 4095);
#endif
        // causal mask: keys key0 + j with j >= nv lie in this row's future (32-key chunks valid
        // for the whole warp need no select)
        const int nv = (int)pos_q - (int)((kt0 + n) * BN2) + 1;
        if (__any_sync(~0u, nv < (int)BN2)) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (__all_sync(~0u, 32 * q + 32 <= nv)) continue;
#pragma unroll
            for (int j = 0; j < 32; ++j) a[32 * q + j] = 32 * q + j < nv ? a[32 * q + j] : -INFINITY;
          }
        }
        float mxa[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mxa[q] = a[q];
#pragma unroll
        for (int j = 8; j < 64; ++j) mxa[j & 7] = fmaxf(mxa[j & 7], a[j]);
        const float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                               fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
        const float mx2 = mx * scale_log2;
#ifdef IL_P2_TRACE_SM
        if (r == 0 && xo == 0) IL_TRACE(1, cs & 4095);
#endif
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
        const float negm = m_used == -INFINITY ? 0.f : -m_used;
        float rsa[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
          float x0, x1;
          ffma2(x0, x1, a[j], a[j + 1], scale_log2, negm);
          float p0, p1;
          if ((IL_P2_EMU >> ((j >> 1) & 7)) & 1) {
            ex2_poly2(x0, x1, p0, p1);                 // this pair on the FMA pipe
          } else {
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          fadd2(rsa[(j >> 1) & 2], rsa[((j >> 1) & 2) + 1], p0, p1);
          pk[j >> 1] = pack_bf16(p0, p1);
        }
#ifdef IL_P2_TRACE_SM
        if (r == 0 && xo == 0) IL_TRACE(2, cs & 4095);
#endif
        tmem_st32u(sb, pk);                            // P (bf16 pairs) over the first 32 columns of S
        l += (rsa[0] + rsa[1]) + (rsa[2] + rsa[3]);
        tmem_wait_st();
#ifdef IL_P2_TRACE_SM
        if (r == 0 && xo == 0) IL_TRACE(3, cs & 4095);
#endif
        // (the O rescale comes after the exponentials, when S is no longer live: fewer registers;
        // PV(cs) is only issued after P_FULL below, so it accumulates onto the rescaled O)
        if (__any_sync(~0u, need)) {
          // lazy rescale of O once PV(cs - 1) has landed (PV(cs - 2) was issued before QK(cs), so
          // it completed before S(cs) was signalled)
          mbar_wait(bar(xo, PV_DONE2), (cs - 1) & 1);
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
        }

        tc_fence_before();
        if (r == 0) IL_TRACE(10 + xo, cs & 4095);
        mbar_arrive(bar(xo, P_FULL2 + b));
      }
      // hand l and m to the epilogue warps (single buffer: the previous item's epilogue has read
      // it once it released O)
      if (it >= 1) mbar_wait(bar(xo, O_FREE2), (it - 1) & 1);
      s_lm[128 * xo + r] = make_float2(l, m_used);
      mbar_arrive(bar(xo, L_READY2));
      ++it;
      w = wn;
      dcur = dn;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

}  // namespace p2
}  // namespace sm100
}  // namespace il
