// match_dev.cuh — warp-cooperative chained block hashing + prefix-index probing (K5),
// shared by il_prefix_match and the never-worse guard of il_refine_batch.
#pragma once
#include "il_internal.cuh"

namespace il {

// Hashes the full 16-token blocks of one prompt row with a single warp: lane j hashes block
// base+j (16 independent lane terms, Z17), the serial fold H_j = mix(H_{j-1}*PHI + c_j) is
// evaluated redundantly by all lanes (content broadcast by shuffle), then the 32 blocks are
// probed in parallel and a ballot gives the leading run of resident + verified blocks.
// Every prompt starts with the same instruction, so its nI full blocks are taken from
// the per-pool hashes (k_instr_hash) and the per-batch probe (k_instr_probe): an exact
// shortcut, the same keys against the same snapshot.
// Returns the hit count capped at floor((L-1)/16) (Z20).  Optionally stores every block hash
// (hash_out[j]) and the pages of the leading run (page_out[j]).  If stop_at_miss, returns as
// soon as the run ends (the guard only needs the count).  kRowReadOnly = false when `row` was
// written earlier in the calling kernel (the guard): its tokens are then read with ld.global.cg.
template <bool kRowReadOnly = true>
__device__ __forceinline__ uint32_t warp_hash_match(const Ctx& c, const uint32_t* __restrict__ row,
                                                    uint32_t L, uint64_t* hash_out, int32_t* page_out,
                                                    bool stop_at_miss) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t F = L / BS;
  const bool verify = (c.cfg.flags & IL_F_VERIFY) != 0;
  const uint32_t nI = min(c.n_instr_blocks, F);
  const uint32_t hI = min(c.sc->instr_hits, nI);
  if (hash_out)
    for (uint32_t j = lane; j < nI; j += 32) hash_out[j] = c.instr_hash[j];
  if (page_out)
    for (uint32_t j = lane; j < hI; j += 32) page_out[j] = c.instr_pages[j];
  uint64_t prev = nI ? c.instr_hash[nI - 1] : root_hash(c.cfg.hash_seed);
  uint32_t h = hI;
  bool run = hI == nI;
  const uint32_t cap = L ? (L - 1) / BS : 0;
  if (!run && stop_at_miss) return min(h, cap);
  for (uint32_t base = nI; base < F; base += 32) {
    const uint32_t j = base + lane;
    const bool active = j < F;
    uint32_t tok[16];
    uint64_t content = 0;
    if (active) content = block_content<kRowReadOnly>(row + (size_t)BS * j, tok);
    const uint64_t chunk_prev = prev;
    const uint32_t nb = min(32u, F - base);
    uint64_t H = 0;
    for (uint32_t t = 0; t < nb; ++t) {
      const uint64_t ct = __shfl_sync(~0u, content, t);
      prev = chain_step(prev, ct);
      if (lane == t) H = prev;
    }
    if (active && hash_out) hash_out[j] = H;
    if (run) {
      uint32_t page = NONE32;
      if (active) page = index_find(c.slot_key, c.slot_page, c.slot_mask, H, nullptr);
      bool ok = page != NONE32;
      const uint64_t up = __shfl_up_sync(~0u, H, 1);
      if (ok && verify) {
        const uint64_t parent = lane == 0 ? chunk_prev : up;
        ok = c.pg_parent[page] == parent;
        const uint4* pt = reinterpret_cast<const uint4*>(c.pg_tok + (size_t)page * BS);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 x = pt[q];
          ok &= x.x == tok[4 * q] && x.y == tok[4 * q + 1] && x.z == tok[4 * q + 2] && x.w == tok[4 * q + 3];
        }
      }
      const uint32_t m = __ballot_sync(~0u, ok && active);
      const uint32_t lead = (m == ~0u) ? 32u : (uint32_t)(__ffs(~m) - 1);
      if (page_out && lane < lead) page_out[j] = (int32_t)page;
      h += lead;
      if (lead < 32) run = false;
    }
    if (!run && stop_at_miss) break;
  }
  return min(h, cap);
}

// Once per batch: the leading run of the instruction's blocks resident (and verified) in the
// index snapshot, and their pages.  One CTA, one thread per block.  from_refine: il_refine_batch's
// probe (guard), which records the batch; il_prefix_match's probe then reuses it -- nothing changes
// the index between the two -- and clears the record, so a second match of the batch probes again.
static __global__ void __launch_bounds__(256) k_instr_probe(Ctx c, uint32_t from_refine) {
  __shared__ uint32_t s_first_bad;
  const uint32_t nI = c.n_instr_blocks;
  const uint32_t b_cur = (uint32_t)(c.sc->batch_done + 1);
  if (!from_refine && c.sc->probe_batch == b_cur) {    // (uniform over the CTA)
    __syncthreads();
    if (threadIdx.x == 0) c.sc->probe_batch = 0;
    return;
  }
  const bool verify = (c.cfg.flags & IL_F_VERIFY) != 0;
  if (threadIdx.x == 0) s_first_bad = nI;
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < nI; j += blockDim.x) {
    const uint64_t H = c.instr_hash[j];
    const uint32_t page = index_find(c.slot_key, c.slot_page, c.slot_mask, H, nullptr);
    bool ok = page != NONE32;
    if (ok && verify) {
      ok = c.pg_parent[page] == (j ? c.instr_hash[j - 1] : root_hash(c.cfg.hash_seed));
      for (uint32_t x = 0; x < BS; ++x) ok &= c.pg_tok[(size_t)page * BS + x] == c.instr[BS * j + x];
    }
    c.instr_pages[j] = ok ? (int32_t)page : -1;
    if (!ok) atomicMin(&s_first_bad, j);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    c.sc->instr_hits = s_first_bad;
    c.sc->probe_batch = from_refine ? b_cur : 0u;
  }
}

}  // namespace il
