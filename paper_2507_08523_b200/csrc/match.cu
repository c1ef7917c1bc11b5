// match.cu — il_prefix_match: K5 chained block hash + longest cached prefix + touch/pin,
// K6 page accounting, LRU eviction (grid-wide radix select) and block-table build.
#include <cooperative_groups.h>

#include "il_internal.cuh"
#include "match_dev.cuh"

namespace cg = cooperative_groups;

namespace il {

// NEXT-1 in-batch dedup (IL_F_DEDUP; Z22b, oracle run_batch_dp).  The batch's table
// of computed blocks: hash -> the lowest admission index presenting it at a position >= its own
// snapshot hit count.  A later request's leading run continues from its snapshot hits through
// blocks owned by an earlier request at the same depth with equal tokens (capped as Z20); those
// blocks' pages are the owner's.  Only the snapshot hits were touched and pinned (k_hash_match).
__device__ __forceinline__ uint32_t bd_slot0(const Ctx& c, uint64_t H) {
  return (uint32_t)((H >> 17) ^ (H >> 40)) & c.bd_mask;    // (bits other than the index table's)
}
__device__ __forceinline__ uint32_t bd_find(const Ctx& c, uint64_t H) {
  for (uint32_t s = bd_slot0(c, H);; s = (s + 1) & c.bd_mask) {
    const uint64_t k = c.bd_key[s];
    if (k == H) return ~c.bd_owner[s];
    if (k == 0) return NONE32;
  }
}
// (k_hash_match, per block j >= h_i of request i) owner <- min(owner, i); a slot taken for the
// first time this batch goes on bd_list, which k_alloc_commit clears after the last lookup
__device__ __forceinline__ void bd_insert(const Ctx& c, uint64_t H, uint32_t i) {
  uint32_t s = bd_slot0(c, H);
  while (true) {
    const uint64_t k = c.bd_key[s];
    if (k == H) break;
    if (k == 0) {
      const uint64_t old = atomicCAS((unsigned long long*)&c.bd_key[s], 0ull, (unsigned long long)H);
      if (old == 0) { c.bd_list[atomicAdd(&c.sc->bd_n, 1u)] = s; break; }
      if (old == H) break;
    }
    s = (s + 1) & c.bd_mask;
  }
  atomicMax(&c.bd_owner[s], ~i);
}

// K5: one warp per request.  Hashes every full block (block_hash row), finds the capped
// leading run of resident + verified blocks in the snapshot index, writes the hit pages to
// the block table, and touches + pins them: stamp <- max(stamp, (b, i)) (Z21).
__global__ void __launch_bounds__(256) k_hash_match(Ctx c, uint32_t B, const uint32_t* __restrict__ prompt_tok,
                                                    const uint32_t* __restrict__ prompt_len,
                                                    uint64_t* __restrict__ block_hash, uint32_t* __restrict__ hit,
                                                    int32_t* __restrict__ block_table, uint32_t dedup) {
  const uint64_t b_cur = c.sc->batch_done + 1;     // device batch counter (graph-replay safe)
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= B) return;
  const uint32_t L = prompt_len[i];
  const uint32_t* row = prompt_tok + (size_t)i * c.cfg.max_prompt_tokens;
  int32_t* bt = block_table + (size_t)i * c.max_blocks;
  const uint32_t h = warp_hash_match(c, row, L, block_hash + (size_t)i * c.max_blocks, bt, false);
  __syncwarp();
  if (dedup)                                        // the blocks this request computes -> dedup table
    for (uint32_t j = h + lane; j < L / BS; j += 32) bd_insert(c, block_hash[(size_t)i * c.max_blocks + j], i);
  const uint64_t st = stamp_of(b_cur, i);
  const uint32_t epoch = (uint32_t)b_cur;
  uint32_t newly = 0;
  // instruction blocks are touched once per batch by k_alloc_scan
  for (uint32_t j = min(c.n_instr_blocks, h) + lane; j < h; j += 32) {
    const uint32_t p = (uint32_t)bt[j];
    atomicMax((unsigned long long*)&c.pg_stamp[p], (unsigned long long)st);
    newly += atomicExch(&c.pg_pin[p], epoch) != epoch;
  }
  for (int o = 16; o; o >>= 1) newly += __shfl_xor_sync(~0u, newly, o);
  // multi-GPU: box-level hits = this rank's leading run, continued through blocks the residency
  // map says some rank holds (hash only), capped as Z20 (records.cu, il.h il_commit_apply)
  uint32_t box = h;
  if (c.map_active) {
    const uint32_t F = L / BS, cap = L ? (L - 1) / BS : 0;
    const uint64_t* bh = block_hash + (size_t)i * c.max_blocks;
    for (uint32_t base = h; base < min(F, cap); base += 32) {
      const uint32_t j = base + lane;
      bool ok = false;
      if (j < F) ok = map_has(c, bh[j]);
      const uint32_t m = __ballot_sync(~0u, ok);
      const uint32_t lead = (m == ~0u) ? 32u : (uint32_t)(__ffs(~m) - 1);
      box += lead;
      if (lead < 32) break;
    }
    box = min(box, cap);
    if (lane == 0) c.box_hit[i] = box;
  }
  if (lane == 0) {
    hit[i] = h;
    c.hit_local[i] = h;
    if (newly) atomicAdd(&c.sc->pinned, newly);
    atomicAdd(&c.sc->hit_sum, h);
    atomicAdd(&c.sc->full_sum, L / BS);
    atomicAdd(&c.sc->box_hit_sum, box);
  }
}

// K6a (one CTA): per-request pages needed (ceil(L/16) - h), suffix lengths, exclusive scans
// -> need_off, cu_q, prefix_len; how many blocks must be evicted.
__global__ void __launch_bounds__(1024) k_alloc_scan(Ctx c, uint32_t B, const uint32_t* __restrict__ prompt_len,
                                                     const uint32_t* __restrict__ hit,
                                                     int32_t* __restrict__ prefix_len, int32_t* __restrict__ cu_q,
                                                     uint64_t) {
  const uint64_t b_cur = c.sc->batch_done + 1;     // device batch counter (graph-replay safe)
  __shared__ uint32_t s_w[32];
  __shared__ int32_t s_top[1025];
  const uint32_t tid = threadIdx.x, per = cdiv(B, 1024);
  // Touch + pin the instruction's hit blocks once: block j gets stamp (b, max{i : h_i > j}).
  const uint32_t nI = min(c.n_instr_blocks, 1024u);
  for (uint32_t x = tid; x <= nI; x += 1024) s_top[x] = -1;
  __syncthreads();
  for (uint32_t i = tid; i < B; i += 1024) atomicMax(&s_top[min(c.hit_local[i], nI)], (int32_t)i);
  __syncthreads();
  // suffix max: s_top[c] = max over c' >= c (a block max-scan over the reversed entries)
  if (nI < 1024) {
    const int32_t v = tid <= nI ? s_top[nI - tid] : -1;
    const int32_t r = block_scan_max(v, reinterpret_cast<int32_t*>(s_w));
    if (tid <= nI) s_top[nI - tid] = r;
  } else if (tid == 0) {
    for (int x = (int)nI - 1; x >= 0; --x) s_top[x] = max(s_top[x], s_top[x + 1]);
  }
  __syncthreads();
  {
    uint32_t newly = 0;
    for (uint32_t j = tid; j < nI; j += 1024) {
      const int32_t who = s_top[j + 1];                 // max i with min(h_i, nI) > j
      if (who < 0) continue;
      const uint32_t p = (uint32_t)c.instr_pages[j];
      atomicMax((unsigned long long*)&c.pg_stamp[p], (unsigned long long)stamp_of(b_cur, (uint32_t)who));
      newly += atomicExch(&c.pg_pin[p], (uint32_t)b_cur) != (uint32_t)b_cur;
    }
    if (newly) atomicAdd(&c.sc->pinned, newly);
  }
  __syncthreads();
  uint32_t n = 0, sfx = 0;
  for (uint32_t i = tid * per; i < min(B, (tid + 1) * per); ++i) {
    const uint32_t L = prompt_len[i], h = hit[i];
    n += cdiv(L + c.cfg.max_decode_tokens, BS) - h;    // prompt pages (+ the decode reserve)
    sfx += L - BS * h;
  }
  uint32_t need, suf;
  uint32_t an = block_scan(n, s_w, &need);
  uint32_t as = block_scan(sfx, s_w, &suf);
  // More suffix rows than the caller's Q / K_new / V_new / out buffers hold: latch the capacity
  // error and publish an EMPTY suffix (cu_q = 0), so that k_synth, k_kv_append, k_tile_scan and
  // the attention kernel, which all loop up to cu_q[B], touch nothing outside the caller's buffers.
  const bool sfx_over = suf > c.cfg.max_suffix_tokens;
  for (uint32_t i = tid * per; i < min(B, (tid + 1) * per); ++i) {
    const uint32_t L = prompt_len[i], h = hit[i];
    c.need_off[i] = an; cu_q[i] = sfx_over ? 0 : (int32_t)as; prefix_len[i] = (int32_t)(BS * h);
    an += cdiv(L + c.cfg.max_decode_tokens, BS) - h;
    as += L - BS * h;
  }
  if (tid == 1023) {
    if (sfx_over) suf = 0;
    c.need_off[B] = need; cu_q[B] = (int32_t)suf;
    DevScalars* sc = c.sc;
    sc->need_total = need;
    sc->suffix_total = suf;
    sc->evicted = 0;
    uint32_t m = need > sc->n_free ? need - sc->n_free : 0;
    const uint32_t cand = sc->resident - sc->pinned;
    if (m > cand) { latch(sc, IL_ERR_CAPACITY); m = 0; sc->need_total = 0; }
    if (sfx_over) latch(sc, IL_ERR_CAPACITY);
    sc->evict_m = m;
    sc->cand = cand;
    sc->stamp_min = ~0ull;
  }
}

// K6b: LRU eviction as one cooperative grid.  Candidates are resident, unpinned pages.
// Order (Z21): stamp ascending, depth descending (hash ascending never decides: one stamp
// (b, i) belongs to one request's chain, whose depths are distinct).  The key
//   key = (b - b_min) << 25 | i << 12 | (4095 - depth)
// is unique per candidate; an 11-bit-digit radix select over the grid finds the m-th
// smallest key, then every candidate with key <= it is evicted: its slot becomes a
// tombstone and its page returns to the free stack.
constexpr int EV_THREADS = 512;
constexpr uint32_t EV_BINS = 2048;

__device__ __forceinline__ bool ev_cand(const Ctx& c, uint32_t p, uint32_t epoch) {
  return c.pg_state[p] == 1 && c.pg_pin[p] != epoch;
}
__device__ __forceinline__ uint64_t ev_key(const Ctx& c, uint32_t p, uint64_t b_min) {
  const uint64_t st = c.pg_stamp[p];
  return (((st >> 32) - b_min) << 25) | ((st & 0x1FFFull) << 12) | (uint64_t)(4095u - min(c.pg_depth[p], 4095u));
}

__global__ void __launch_bounds__(EV_THREADS) k_evict(Ctx c, uint64_t) {
  const uint64_t b_cur = c.sc->batch_done + 1;     // device batch counter (graph-replay safe)
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t s_hist[EV_BINS];
  __shared__ uint64_t s_red;
  __shared__ uint32_t s_wsum[EV_THREADS / 32];
  DevScalars* sc = c.sc;
  const uint32_t m = sc->evict_m;
  const uint32_t epoch = (uint32_t)b_cur, C = c.cfg.kv_pages;
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  if (m == 0) return;                                   // uniform across the grid
  // pass 0: b_min over candidates
  if (threadIdx.x == 0) s_red = ~0ull;
  __syncthreads();
  uint64_t bmin = ~0ull;
  for (uint32_t p = gtid; p < C; p += gstride)
    if (ev_cand(c, p, epoch)) bmin = min(bmin, c.pg_stamp[p] >> 32);
  for (int o = 16; o; o >>= 1) bmin = min(bmin, __shfl_xor_sync(~0u, bmin, o));
  if ((threadIdx.x & 31) == 0) atomicMin((unsigned long long*)&s_red, (unsigned long long)bmin);
  __syncthreads();
  if (threadIdx.x == 0) atomicMin((unsigned long long*)&sc->stamp_min, (unsigned long long)s_red);
  grid.sync();
  const uint64_t b_min = sc->stamp_min;
  const uint64_t kmax = ((b_cur - b_min) << 25) | ((1ull << 25) - 1);
  int top_bit = 63 - __clzll((long long)kmax);
  int shift = (top_bit / 11) * 11;                      // lowest bit of the top digit
  uint64_t prefix = 0;                                  // key bits above `shift` selected so far
  uint32_t remaining = m;
  for (int pass = 0; shift >= 0; ++pass, shift -= 11) {
    uint32_t* ghist = c.hist + (pass & 1) * EV_BINS;
    for (uint32_t x = threadIdx.x; x < EV_BINS; x += blockDim.x) s_hist[x] = 0;
    __syncthreads();
    for (uint32_t p = gtid; p < C; p += gstride) {
      if (!ev_cand(c, p, epoch)) continue;
      const uint64_t key = ev_key(c, p, b_min);
      const uint64_t hi = (shift + 11 >= 64) ? 0 : (key >> (shift + 11));
      if (hi != prefix) continue;
      atomicAdd(&s_hist[(key >> shift) & (EV_BINS - 1)], 1u);
    }
    __syncthreads();
    for (uint32_t x = threadIdx.x; x < EV_BINS; x += blockDim.x)
      if (s_hist[x]) atomicAdd(&ghist[x], s_hist[x]);
    grid.sync();
    // every CTA finds the bin holding the remaining-th smallest key identically: a block-wide
    // prefix sum over the 2048 bins (4 per thread; L1 bypassed: other CTAs wrote them)
    {
      constexpr uint32_t PER = EV_BINS / EV_THREADS;
      uint32_t v[PER], sum = 0;
#pragma unroll
      for (uint32_t k = 0; k < PER; ++k) { v[k] = __ldcg(&ghist[threadIdx.x * PER + k]); sum += v[k]; }
      const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
      uint32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(~0u, inc, o);
        if (lane >= (uint32_t)o) inc += y;
      }
      if (lane == 31) s_wsum[wid] = inc;
      __syncthreads();
      if (wid == 0) {
        uint32_t t = lane < EV_THREADS / 32 ? s_wsum[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(~0u, t, o);
          if (lane >= (uint32_t)o) t += y;
        }
        if (lane < EV_THREADS / 32) s_wsum[lane] = t;      // inclusive warp-total scan
      }
      __syncthreads();
      uint32_t acc = inc - sum + (wid ? s_wsum[wid - 1] : 0u);   // exclusive prefix of this thread's bins
      if (acc < remaining && remaining <= acc + sum) {
#pragma unroll
        for (uint32_t k = 0; k < PER; ++k) {
          if (acc + v[k] >= remaining) { s_red = ((uint64_t)(threadIdx.x * PER + k) << 32) | (remaining - acc); break; }
          acc += v[k];
        }
      }
    }
    __syncthreads();
    const uint32_t bin = (uint32_t)(s_red >> 32);
    remaining = (uint32_t)(s_red & 0xFFFFFFFFu);
    prefix = (prefix << 11) | bin;
    // clear the other histogram buffer for the next pass (CTA 0), ordered by the next sync
    if (blockIdx.x == 0)
      for (uint32_t x = threadIdx.x; x < EV_BINS; x += blockDim.x) c.hist[((pass + 1) & 1) * EV_BINS + x] = 0;
    grid.sync();
  }
  // both histogram buffers are dead now (every CTA read the last one before the pass's sync)
  for (uint32_t x = gtid; x < 2 * EV_BINS; x += gstride) c.hist[x] = 0;
  // prefix is now the exact m-th smallest key; evict every candidate with key <= prefix
  const uint64_t kstar = prefix;
  uint32_t ev = 0;
  for (uint32_t p = gtid; p < C; p += gstride) {
    if (!ev_cand(c, p, epoch)) continue;
    if (ev_key(c, p, b_min) > kstar) continue;
    c.pg_state[p] = 0;
    const uint32_t s = c.pg_slot[p];
    c.slot_key[s] = KEY_TOMB;
    c.slot_page[s] = NONE32;
    c.pg_slot[p] = NONE32;
    const uint32_t f = atomicAdd(&sc->n_free, 1u);
    c.free_list[f] = p;
    const uint32_t e = atomicAdd(&sc->evicted, 1u);
    c.evicted_list[e] = c.pg_hash[p];
    ++ev;
  }
  for (int o = 16; o; o >>= 1) ev += __shfl_xor_sync(~0u, ev, o);
  if ((threadIdx.x & 31) == 0 && ev) atomicSub(&sc->resident, ev);
  grid.sync();
  if (gtid == 0) {
    if (sc->evicted != m) latch(sc, IL_ERR_INTERNAL);
  }
}

// K6c: pop the batch's pages (free stack top) into the block table after the hit pages.
__global__ void __launch_bounds__(256) k_alloc_fill(Ctx c, uint32_t B, const uint32_t* __restrict__ prompt_len,
                                                    const uint32_t* __restrict__ hit, const uint64_t* __restrict__ block_hash,
                                                    int32_t* __restrict__ block_table) {
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= B) return;
  DevScalars* sc = c.sc;
  if (sc->status == IL_ERR_CAPACITY) return;
  const uint32_t base = sc->n_free - sc->need_total + c.need_off[i];
  const uint32_t h = hit[i], nb = cdiv(prompt_len[i] + c.cfg.max_decode_tokens, BS);
  int32_t* bt = block_table + (size_t)i * c.max_blocks;
  for (uint32_t j = h + lane; j < nb; j += 32) bt[j] = (int32_t)c.free_list[base + (j - h)];
  // IL_F_DEDUP: the in-batch shared run [snapshot hits, h) gets the owner's pages, popped for the
  // owner's blocks [h_o, nb_o) from the same stack (the owner's run ends before any block it owns)
  if (c.bd_key)
    for (uint32_t j = c.hit_local[i] + lane; j < h; j += 32) {
      const uint32_t o = bd_find(c, block_hash[(size_t)i * c.max_blocks + j]);
      bt[j] = (int32_t)c.free_list[sc->n_free - sc->need_total + c.need_off[o] + (j - hit[o])];
    }
}
// warp per request: extend hit[i] through blocks an earlier request computes
__global__ void __launch_bounds__(256) k_bd_resolve(Ctx c, uint32_t B, const uint32_t* __restrict__ prompt_tok,
                                                    const uint32_t* __restrict__ prompt_len,
                                                    const uint64_t* __restrict__ block_hash,
                                                    uint32_t* __restrict__ hit) {
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= B) return;
  const uint32_t L = prompt_len[i], F = L / BS, cap = L ? (L - 1) / BS : 0, lim = min(F, cap);
  const uint32_t hl = hit[i];
  const uint64_t* bh = block_hash + (size_t)i * c.max_blocks;
  const uint32_t* row = prompt_tok + (size_t)i * c.cfg.max_prompt_tokens;
  uint32_t he = hl;
  for (uint32_t base = hl; base < lim; base += 32) {
    const uint32_t j = base + lane;
    bool ok = false;
    if (j < lim) {
      const uint64_t H = bh[j];
      const uint32_t o = bd_find(c, H);
      if (o < i && block_hash[(size_t)o * c.max_blocks + j] == H) {
        const uint4* a = reinterpret_cast<const uint4*>(row + (size_t)BS * j);
        const uint4* b = reinterpret_cast<const uint4*>(prompt_tok + (size_t)o * c.cfg.max_prompt_tokens + (size_t)BS * j);
        ok = true;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 x = a[q], y = b[q];
          ok &= x.x == y.x && x.y == y.y && x.z == y.z && x.w == y.w;
        }
      }
    }
    const uint32_t m = __ballot_sync(~0u, ok);
    const uint32_t lead = (m == ~0u) ? 32u : (uint32_t)(__ffs(~m) - 1);
    he += lead;
    if (lead < 32) break;
  }
  if (lane == 0 && he > hl) {
    hit[i] = he;
    atomicAdd(&c.sc->dedup_sum, he - hl);
    atomicAdd(&c.sc->hit_sum, he - hl);
    if (!c.map_active) {                              // box-level hits include the shared run (oracle)
      atomicAdd(&c.sc->box_hit_sum, he - hl);
    } else if (he > c.box_hit[i]) {
      atomicAdd(&c.sc->box_hit_sum, he - c.box_hit[i]);
      c.box_hit[i] = he;
    }
  }
}
// (a kernel rather than a memset node: keeps the captured match graph all-kernel)
__global__ void k_match_begin(Ctx c) {
  DevScalars* sc = c.sc;
  sc->pinned = 0; sc->hit_sum = 0; sc->full_sum = 0; sc->box_hit_sum = 0; sc->inserted = 0; sc->dedup_sum = 0;
}
__global__ void __launch_bounds__(1024) k_alloc_commit(Ctx c) {
  DevScalars* sc = c.sc;
  if (c.bd_key) {                                   // the dedup table's lookups are over: clear it
    const uint32_t n = sc->bd_n;
    for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
      const uint32_t s = c.bd_list[x];
      c.bd_key[s] = 0;
      c.bd_owner[s] = 0;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (sc->status != IL_ERR_CAPACITY) sc->n_free -= sc->need_total;
    sc->bd_n = 0;
  }
}

}  // namespace il

using namespace il;

// one-time per-context setup (il_create, current device): cooperative grid size of k_evict
il_status il::match_setup(Ctx* c) {
  int per_sm = 0;
  IL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_evict, EV_THREADS, 0));
  // one CTA per SM: each of the five passes over the pages is short, the grid syncs dominate
  // (148 CTAs: 25 us per evicting c3 step; 296: 28; 74: 27; 37: 38)
  c->ev_per_sm = std::max(1, std::min(per_sm, 1));
  c->ev_blocks = c->ev_per_sm * c->num_sms;
  return IL_OK;
}

extern "C" il_status il_prefix_match(il_ctx* c, uint32_t B, const uint32_t* prompt_tok, const uint32_t* prompt_len,
                                     uint64_t* block_hash, uint32_t* hit, int32_t* block_table,
                                     int32_t* prefix_len, int32_t* cu_q, il_stream s) {
  if (!c->pool_loaded) { set_error("il_prefix_match before il_pool_load"); return IL_ERR_STATE; }
  if (B > c->cfg.max_batch) { set_error("B > max_batch"); return IL_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)s;
  const uint64_t b_cur = c->batch + 1;
  const bool dedup = (c->cfg.flags & IL_F_DEDUP) && B > 1;
  k_match_begin<<<1, 1, 0, st>>>(*c);
  k_instr_probe<<<1, 256, 0, st>>>(*c, 0u);
  if (B) k_hash_match<<<cdiv(B * 32, 256), 256, 0, st>>>(*c, B, prompt_tok, prompt_len, block_hash, hit, block_table,
                                                           dedup ? 1u : 0u);
  if (dedup) k_bd_resolve<<<cdiv(B * 32, 256), 256, 0, st>>>(*c, B, prompt_tok, prompt_len, block_hash, hit);
  k_alloc_scan<<<1, 1024, 0, st>>>(*c, B, prompt_len, hit, prefix_len, cu_q, b_cur);
  {
    Ctx cc = *c;
    uint64_t bc = b_cur;
    void* args[] = {&cc, &bc};
    IL_CUDA(cudaLaunchCooperativeKernel((void*)k_evict, dim3(c->ev_blocks), dim3(EV_THREADS), args, 0, st));
  }
  if (B) k_alloc_fill<<<cdiv(B * 32, 256), 256, 0, st>>>(*c, B, prompt_len, hit, block_hash, block_table);
  k_alloc_commit<<<1, 1024, 0, st>>>(*c);
  IL_LAUNCH_CHECK("il_prefix_match");
  c->launches += (B ? 7 : 5) + (dedup ? 1 : 0);
  c->prompt_tok = prompt_tok;
  c->prompt_len = prompt_len;
  c->block_hash = block_hash;
  c->hit = hit;
  c->block_table = block_table;
  c->matched = true;
  c->last_B = B;
  return IL_OK;
}
