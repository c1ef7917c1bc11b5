// match_dev.cuh — warp-cooperative chained block hashing + prefix-index probing (K5),
// shared by il_prefix_match and the never-worse guard of il_refine_batch.
#pragma once
#include "il_internal.cuh"

namespace il {

// Hashes the full 16-token blocks of one prompt row with a single warp: lane j hashes block
// base+j (16 independent lane terms, Z17), the serial fold H_j = mix(H_{j-1}*PHI + c_j) is
// evaluated redundantly by all lanes (content broadcast by shuffle), then the 32 blocks are
// probed in parallel and a ballot gives the leading run of resident + verified blocks.
// Returns the hit count capped at floor((L-1)/16) (Z20).  Optionally stores every block hash
// (hash_out[j]) and the pages of the leading run (page_out[j]).  If stop_at_miss, returns as
// soon as the run ends (the guard only needs the count).
__device__ __forceinline__ uint32_t warp_hash_match(const Ctx& c, const uint32_t* __restrict__ row,
                                                    uint32_t L, uint64_t* hash_out, int32_t* page_out,
                                                    bool stop_at_miss) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t F = L / BS;
  const bool verify = (c.cfg.flags & IL_F_VERIFY) != 0;
  uint64_t prev = root_hash(c.cfg.hash_seed);
  uint32_t h = 0;
  bool run = true;
  for (uint32_t base = 0; base < F; base += 32) {
    const uint32_t j = base + lane;
    const bool active = j < F;
    uint32_t tok[16];
    uint64_t content = 0;
    if (active) content = block_content(row + (size_t)BS * j, tok);
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
  const uint32_t cap = L ? (L - 1) / BS : 0;
  return min(h, cap);
}

}  // namespace il
