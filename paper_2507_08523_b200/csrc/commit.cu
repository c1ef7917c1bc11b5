#include <algorithm>
// commit.cu — il_commit (K8): prefix-index insert in admission order (first request owns the
// page, duplicates and partial pages are freed; Z22, Z23) + tombstone compaction, and the
// ICL-Table commit (keyed upsert in admission order, keep the T most recent; Z2, Z3, Z14).
#include <cooperative_groups.h>

#include "il_internal.cuh"

namespace cg = cooperative_groups;

namespace il {

constexpr uint32_t OCC_FREE = 0xFFFFFFFEu;   // the request's page is a duplicate: free it
constexpr uint32_t OCC_CAND = 0xFFFFFFFDu;   // not resident: insert candidate

__device__ __forceinline__ void push_free(const Ctx& c, uint32_t page) {
  const uint32_t f = atomicAdd(&c.sc->n_free, 1u);
  c.free_list[f] = page;
}

// Phase A: blocks j in [h_i, F_i) that are resident now (only the Z20-capped block can be)
// get their stamp refreshed and the request's page freed; the rest become insert candidates.
__global__ void __launch_bounds__(256) k_commit_probe(Ctx c, uint32_t B, uint64_t) {
  const uint64_t b_cur = c.sc->batch_done + 1;     // device batch counter (graph-replay safe)
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= B) return;
  const uint32_t L = c.prompt_len[i], h = c.hit[i], F = L / BS;
  const uint64_t st = stamp_of(b_cur, i);
  for (uint32_t j = h + lane; j < F; j += 32) {
    const uint64_t H = c.block_hash[(size_t)i * c.max_blocks + j];
    const uint32_t page = index_find(c.slot_key, c.slot_page, c.slot_mask, H, nullptr);
    if (page != NONE32) {
      atomicMax((unsigned long long*)&c.pg_stamp[page], (unsigned long long)st);
      c.occ[(size_t)i * c.max_blocks + j] = OCC_FREE;
    } else {
      c.occ[(size_t)i * c.max_blocks + j] = OCC_CAND;
    }
  }
}

// Phase B: lock-free insert-or-find of every candidate key (CAS into EMPTY slots, linear
// probing past tombstones), then claim = min admission index, cstamp = max stamp over the
// requests presenting the key (order-independent, hence deterministic).
__global__ void __launch_bounds__(256) k_commit_insert(Ctx c, uint32_t B, uint64_t) {
  const uint64_t b_cur = c.sc->batch_done + 1;     // device batch counter (graph-replay safe)
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= B) return;
  const uint32_t L = c.prompt_len[i], h = c.hit[i], F = L / BS;
  const uint64_t st = stamp_of(b_cur, i);
  uint32_t inserted = 0;
  for (uint32_t j = h + lane; j < F; j += 32) {
    uint32_t* occ = c.occ + (size_t)i * c.max_blocks + j;
    if (*occ != OCC_CAND) continue;
    const uint64_t H = c.block_hash[(size_t)i * c.max_blocks + j];
    uint32_t s = (uint32_t)(H ^ (H >> 32)) & c.slot_mask;
    while (true) {
      const uint64_t k = c.slot_key[s];
      if (k == H) break;
      if (k == KEY_EMPTY) {
        const uint64_t old = atomicCAS((unsigned long long*)&c.slot_key[s], (unsigned long long)KEY_EMPTY,
                                       (unsigned long long)H);
        if (old == KEY_EMPTY) { ++inserted; break; }
        if (old == H) break;
      }
      s = (s + 1) & c.slot_mask;
    }
    atomicMin(&c.claim[s], i);
    atomicMax((unsigned long long*)&c.cstamp[s], (unsigned long long)st);
    *occ = s;
  }
  for (int o = 16; o; o >>= 1) inserted += __shfl_xor_sync(~0u, inserted, o);
  if (lane == 0 && inserted) atomicAdd(&c.sc->used_slots, inserted);
}

// Phase C: the claimant owns the block: its page becomes resident with the block's hash,
// parent hash, tokens, depth and the max stamp.  Every other page of the batch that is not
// resident now (duplicates, the capped block, the partial trailing block) is freed.
__global__ void __launch_bounds__(256) k_commit_own(Ctx c, uint32_t B) {
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= B) return;
  const uint32_t L = c.prompt_len[i], h = c.hit[i], F = L / BS;
  const int32_t* bt = c.block_table + (size_t)i * c.max_blocks;
  const uint64_t* bh = c.block_hash + (size_t)i * c.max_blocks;
  const uint32_t* row = c.prompt_tok + (size_t)i * c.cfg.max_prompt_tokens;
  uint32_t owned = 0;
  for (uint32_t j = h + lane; j < F; j += 32) {
    const uint32_t o = c.occ[(size_t)i * c.max_blocks + j];
    const uint32_t page = (uint32_t)bt[j];
    if (o == OCC_FREE) { push_free(c, page); continue; }
    if (c.claim[o] != i) { push_free(c, page); continue; }
    c.slot_page[o] = page;
    c.pg_hash[page] = bh[j];
    c.pg_parent[page] = j ? bh[j - 1] : root_hash(c.cfg.hash_seed);
    const uint4* src = reinterpret_cast<const uint4*>(row + (size_t)BS * j);
    uint4* dst = reinterpret_cast<uint4*>(c.pg_tok + (size_t)page * BS);
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[q] = src[q];
    c.pg_depth[page] = j;
    c.pg_stamp[page] = c.cstamp[o];
    c.pg_slot[page] = o;
    c.pg_state[page] = 1;
    c.claim[o] = NONE32;
    c.cstamp[o] = 0;
    if (c.ins_list) c.ins_list[atomicAdd(&c.sc->inserted, 1u)] = bh[j];   // multi-GPU block record
    ++owned;
  }
  // the partial block (Z23) and the decode reserve's pages go back to the free stack
  for (uint32_t j = F + lane; j < cdiv(L + c.cfg.max_decode_tokens, BS); j += 32) push_free(c, (uint32_t)bt[j]);
  for (int o = 16; o; o >>= 1) owned += __shfl_xor_sync(~0u, owned, o);
  if (lane == 0 && owned) atomicAdd(&c.sc->resident, owned);
}

// Tombstone compaction: when live + tombstones exceed IL_REBUILD_PCT % of the slots, rebuild the table
// from the resident pages (one cooperative grid).
#ifndef IL_REBUILD_PCT
#define IL_REBUILD_PCT 50
#endif
__global__ void __launch_bounds__(512) k_rebuild(Ctx c) {
  cg::grid_group grid = cg::this_grid();
  DevScalars* sc = c.sc;
  // (live + tombstones) / slots above IL_REBUILD_PCT % (50 and 75 measure the same at c3): probes
  // through tombstones grow long before the table fills
  if ((uint64_t)sc->used_slots * 100 <= (uint64_t)c.n_slots * IL_REBUILD_PCT) return;   // uniform
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  for (uint32_t s = gtid; s < c.n_slots; s += gs) { c.slot_key[s] = KEY_EMPTY; c.slot_page[s] = NONE32; }
  grid.sync();
  for (uint32_t p = gtid; p < c.cfg.kv_pages; p += gs) {
    if (c.pg_state[p] != 1) continue;
    const uint64_t H = c.pg_hash[p];
    uint32_t s = (uint32_t)(H ^ (H >> 32)) & c.slot_mask;
    while (atomicCAS((unsigned long long*)&c.slot_key[s], (unsigned long long)KEY_EMPTY, (unsigned long long)H) !=
           KEY_EMPTY)
      s = (s + 1) & c.slot_mask;
    c.slot_page[s] = p;
    c.pg_slot[p] = s;
  }
  grid.sync();
  if (gtid == 0) { sc->used_slots = sc->resident; sc->rebuilds += 1; }
}

// ---------------------------------------------------------------------------------------
// ICL Table commit.
// ---------------------------------------------------------------------------------------
// k_tab_key: each request's final DS tuple -> 64-bit hash -> slot of a per-batch dedup table
// (lock-free CAS insert), and dd_max[slot] = 1 + the last admission index presenting it.
__global__ void k_tab_key(Ctx c, uint32_t B) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  uint64_t h = 0x5851F42D4C957F2Dull;
  for (uint32_t j = 0; j < c.cfg.k; ++j) h = mix64(h ^ ((uint64_t)c.final_ds[(size_t)i * c.cfg.k + j] + PHI64 * (j + 1)));
  h |= 1ull;                                           // never the EMPTY key 0
  uint32_t s = (uint32_t)(h ^ (h >> 32)) & c.dd_mask;
  while (true) {
    const uint64_t old = atomicCAS((unsigned long long*)&c.dd_key[s], 0ull, (unsigned long long)h);
    if (old == 0 || old == h) break;
    s = (s + 1) & c.dd_mask;
  }
  c.tab_slot[i] = s;
  atomicMax(&c.dd_max[s], i + 1);
}

// k_tab_find: one warp per request: whether it is the last request of the batch presenting its
// final DS (confirmed by comparing tuples: a 64-bit hash collision latches IL_ERR_INTERNAL
// instead of merging two keys), and the slot already holding the key in the table (or -1).
// Where the key can already be in the table follows from the rules: a rule-1 final DS IS the
// target's key (its slot is known); a rule-2/3 final DS cannot be in the snapshot table, since
// an entry with the same template multiset would have PMC = k and the request would be rule 1;
// only a guard-reverted request (final = DS_current, possibly an existing entry) needs a scan.
__global__ void __launch_bounds__(256) k_tab_find(Ctx c, uint32_t B) {
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= B) return;
  const uint32_t k = c.cfg.k;
  const uint32_t rep = c.dd_max[c.tab_slot[i]] - 1;
  if (rep != i) {                                      // (warp-uniform) lane q compares entry q
    const bool ne = lane < k && c.final_ds[(size_t)rep * k + lane] != c.final_ds[(size_t)i * k + lane];
    if (__any_sync(~0u, ne) && lane == 0) latch(c.sc, IL_ERR_INTERNAL);
  }
  const il_refine_info inf = c.info[i];
  int32_t found = -1;
  if (inf.rule == 1 && !inf.reverted) {
    found = inf.target_slot;
  } else if (inf.reverted) {
    // scan for DS_current: 8 slots per lane per round, stamps and first demonstrations loaded
    // together (the scan is L2-latency bound); only slots whose first demonstration matches
    // compare the rest
    const uint32_t T = c.cfg.table_capacity, f0 = c.final_ds[(size_t)i * k];
    for (uint32_t s0 = lane; s0 < T; s0 += 8 * 32) {
      uint64_t st[8];
      uint32_t d0[8];
#pragma unroll
      for (uint32_t u = 0; u < 8; ++u) {
        const uint32_t sl = s0 + 32 * u;
        st[u] = sl < T ? c.tab_stamp[sl] : 0ull;
        d0[u] = sl < T ? c.tab_ds[(size_t)sl * k] : 0u;
      }
#pragma unroll
      for (uint32_t u = 0; u < 8; ++u) {
        if (st[u] == 0 || d0[u] != f0) continue;
        const uint32_t sl = s0 + 32 * u;
        bool eq = true;
        for (uint32_t q = 1; q < k; ++q) eq &= c.tab_ds[(size_t)sl * k + q] == c.final_ds[(size_t)i * k + q];
        if (eq) found = (int32_t)sl;
      }
    }
    for (int o = 16; o; o >>= 1) found = max(found, __shfl_xor_sync(~0u, found, o));
  }
  if (lane == 0) { c.tab_find[i] = found; c.tab_last[i] = rep == i; }
}


// k_tab_commit (one CTA of 1024 threads, T <= 8192 slots, B <= 8192 requests).
// The recency order after the batch is: untouched old entries (stamps of earlier batches),
// then the batch's keys ordered by their last request.  Keep the T most recent.
__global__ void __launch_bounds__(1024) k_tab_commit(Ctx c, uint32_t B, uint64_t) {
  const uint64_t b_cur = c.sc->batch_done + 1;     // device batch counter (graph-replay safe)
  extern __shared__ uint64_t s_old[];                  // old stamps, compacted [n_old]
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_hist[256];
  __shared__ uint64_t s_pref;
  __shared__ uint32_t s_rem;
  const uint32_t tid = threadIdx.x, T = c.cfg.table_capacity, k = c.cfg.k;
  const uint32_t perB = cdiv(B, 1024), perT = cdiv(T, 1024);
  // 1. refresh keys that exist (rule 1 targets and re-appended keys)
  for (uint32_t i = tid; i < B; i += 1024)
    if (c.tab_last[i] && c.tab_find[i] >= 0) c.tab_stamp[c.tab_find[i]] = stamp_of(b_cur, i);
  __syncthreads();
  // 2. counts: old (stamp of an earlier batch), live, new keys, last requests
  uint32_t my_old = 0;
  for (uint32_t s = tid * perT; s < min(T, (tid + 1) * perT); ++s) {
    const uint64_t st = c.tab_stamp[s];
    my_old += st != 0 && (st >> 32) < b_cur;
  }
  uint32_t n_old;
  const uint32_t old_off = block_scan(my_old, s_w, &n_old);
  {
    uint32_t o = old_off;
    for (uint32_t s = tid * perT; s < min(T, (tid + 1) * perT); ++s) {
      const uint64_t st = c.tab_stamp[s];
      if (st != 0 && (st >> 32) < b_cur) s_old[o++] = st;
    }
  }
  uint32_t my_last = 0, my_new = 0;
  for (uint32_t i = tid * perB; i < min(B, (tid + 1) * perB); ++i) {
    my_last += c.tab_last[i];
    my_new += c.tab_last[i] && c.tab_find[i] < 0;
  }
  uint32_t n_last, n_new;
  const uint32_t last_off = block_scan(my_last, s_w, &n_last);
  const uint32_t new_off = block_scan(my_new, s_w, &n_new);
  const uint32_t total = n_old + n_last;                 // live entries after the batch
  const uint32_t d = total > T ? total - T : 0;          // entries to drop
  // 3. drop: the d smallest old stamps, or all old + the first (d - n_old) batch keys
  uint64_t tau = 0;                                      // drop old entries with stamp <= tau
  if (d > 0 && d <= n_old) {
    // radix select (8-bit digits, MSB first) of the d-th smallest old stamp
    if (tid == 0) { s_pref = 0; s_rem = d; }
    __syncthreads();
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (uint32_t x = tid; x < 256; x += 1024) s_hist[x] = 0;
      __syncthreads();
      const uint64_t pref = s_pref;
      for (uint32_t x = tid; x < n_old; x += 1024) {
        const uint64_t v = s_old[x];
        const uint64_t hi = shift + 8 >= 64 ? 0 : v >> (shift + 8);
        if (hi == pref) atomicAdd(&s_hist[(v >> shift) & 255], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        uint32_t acc = 0, bin = 0;
        for (bin = 0; bin < 256; ++bin) {
          if (acc + s_hist[bin] >= s_rem) break;
          acc += s_hist[bin];
        }
        s_pref = (pref << 8) | bin;
        s_rem -= acc;
      }
      __syncthreads();
    }
    tau = s_pref;
  } else if (d > n_old) {
    tau = ~0ull;                                         // every old entry goes
  }
  const uint32_t d_batch = d > n_old ? d - n_old : 0;   // batch keys dropped (earliest last-requests)
  if (d > 0) {
    for (uint32_t s = tid; s < T; s += 1024) {
      const uint64_t st = c.tab_stamp[s];
      if (st != 0 && (st >> 32) < b_cur && st <= tau) c.tab_stamp[s] = 0;
    }
  }
  __syncthreads();
  // batch keys: request i with last[i] has rank r among last requests; it survives iff r >= d_batch
  {
    uint32_t r = last_off;
    for (uint32_t i = tid * perB; i < min(B, (tid + 1) * perB); ++i) {
      if (!c.tab_last[i]) continue;
      if (r < d_batch && c.tab_find[i] >= 0) c.tab_stamp[c.tab_find[i]] = 0;
      ++r;
    }
  }
  __syncthreads();
  // 4. free slots (stamp 0) in slot order receive the surviving new keys in admission order
  uint32_t my_free = 0;
  for (uint32_t s = tid * perT; s < min(T, (tid + 1) * perT); ++s) my_free += c.tab_stamp[s] == 0;
  uint32_t n_free;
  const uint32_t free_off = block_scan(my_free, s_w, &n_free);
  // surviving new keys: new requests whose last-rank >= d_batch; their order = new rank minus
  // the number of dropped new keys before them.  Dropped batch keys are a prefix (by i) of
  // the last requests, so the surviving new keys are a suffix of the new requests.
  uint32_t my_dnew = 0;
  {
    uint32_t r = last_off;
    for (uint32_t i = tid * perB; i < min(B, (tid + 1) * perB); ++i) {
      if (!c.tab_last[i]) continue;
      if (r < d_batch && c.tab_find[i] < 0) ++my_dnew;
      ++r;
    }
  }
  uint32_t n_dnew;
  block_scan(my_dnew, s_w, &n_dnew);
  // map: j-th free slot (slot order) -> stored in s_old reuse as u32 list
  uint32_t* s_free = reinterpret_cast<uint32_t*>(s_old);
  __syncthreads();
  {
    uint32_t o = free_off;
    for (uint32_t s = tid * perT; s < min(T, (tid + 1) * perT); ++s)
      if (c.tab_stamp[s] == 0) s_free[o++] = s;
  }
  __syncthreads();
  {
    uint32_t rn = new_off, rl = last_off;
    for (uint32_t i = tid * perB; i < min(B, (tid + 1) * perB); ++i) {
      if (!c.tab_last[i]) continue;
      const bool is_new = c.tab_find[i] < 0;
      if (is_new && rl >= d_batch) {
        const uint32_t slot_rank = rn - n_dnew;
        if (slot_rank < n_free) {
          const uint32_t s = s_free[slot_rank];
          for (uint32_t j = 0; j < k; ++j) {
            const uint32_t dd = c.final_ds[(size_t)i * k + j];
            c.tab_ds[(size_t)s * k + j] = dd;
            c.tab_tpl[(size_t)j * T + s] = c.tid[dd];
          }
          c.tab_stamp[s] = stamp_of(b_cur, i);
        } else {
          latch(c.sc, IL_ERR_INTERNAL);
        }
      }
      rn += is_new;
      ++rl;
    }
  }
  if (tid == 0) c.sc->table_entries = min(total, T);
  for (uint32_t i = tid; i < B; i += 1024) {          // leave the dedup table empty
    const uint32_t sl = c.tab_slot[i];
    c.dd_key[sl] = 0;
    c.dd_max[sl] = 0;
  }
}

}  // namespace il

using namespace il;

// index half of the commit (this context's blocks), stamps of batch b_cur
static il_status commit_index(Ctx* c, cudaStream_t st, uint64_t b_cur) {
  const uint32_t B = c->last_B;
  if (B) {
    const uint32_t g = cdiv(B * 32, 256);
    k_commit_probe<<<g, 256, 0, st>>>(*c, B, b_cur);
    k_commit_insert<<<g, 256, 0, st>>>(*c, B, b_cur);
    k_commit_own<<<g, 256, 0, st>>>(*c, B);
  }
  Ctx cc = *c;
  void* args[] = {&cc};
  IL_CUDA(cudaLaunchCooperativeKernel((void*)k_rebuild, dim3(c->rb_blocks), dim3(512), args, 0, st));
  IL_LAUNCH_CHECK("il_commit (index)");
  c->launches += (B ? 3 : 0) + 1;
  return IL_OK;
}

// table half: B records (final DS + refine info) in admission order, stamps (b_cur, i)
il_status il::commit_table(Ctx* c, uint32_t B, const uint32_t* final_ds, const il_refine_info* info,
                           cudaStream_t st, uint64_t b_cur) {
  if (!B) return IL_OK;
  c->final_ds = final_ds;
  c->info = info;
  k_tab_key<<<cdiv(B, 256), 256, 0, st>>>(*c, B);
  k_tab_find<<<cdiv(B * 32, 256), 256, 0, st>>>(*c, B);
  const size_t smem = (size_t)c->cfg.table_capacity * 8;
  k_tab_commit<<<1, 1024, smem, st>>>(*c, B, b_cur);
  IL_LAUNCH_CHECK("il_commit (table)");
  c->launches += 3;
  return IL_OK;
}

__global__ void k_end_batch(Ctx c) { c.sc->batch_done += 1; }

// one-time per-context setup (il_create, current device): attributes and cooperative grid size
il_status il::commit_setup(Ctx* c) {
  IL_CUDA(cudaFuncSetAttribute(k_tab_commit, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 * 8));
  int per_sm = 0;
  IL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rebuild, 512, 0));
  c->rb_per_sm = std::max(1, std::min(per_sm, 2));
  c->rb_blocks = c->rb_per_sm * c->num_sms;
  return IL_OK;
}

il_status il::end_batch(Ctx* c, cudaStream_t st) {
  k_end_batch<<<1, 1, 0, st>>>(*c);
  IL_LAUNCH_CHECK("il_commit (end of batch)");
  c->launches += 1;
  c->batch += 1;
  c->refined = c->matched = c->index_done = c->exported = false;
  return IL_OK;
}

extern "C" il_status il_commit(il_ctx* c, il_stream s) {
  if (!c->matched || c->index_done) { set_error("il_commit before il_prefix_match"); return IL_ERR_STATE; }
  const bool pair = (c->cfg.flags & IL_F_PAIR) != 0;
  if (pair && !c->refined) { set_error("il_commit before il_refine_batch"); return IL_ERR_STATE; }
  cudaStream_t st = (cudaStream_t)s;
  const uint64_t b_cur = c->batch + 1;
  il_status r = commit_index(c, st, b_cur);
  if (r != IL_OK) return r;
  if (pair) {
    r = commit_table(c, c->last_B, c->final_ds, c->info, st, b_cur);
    if (r != IL_OK) return r;
  }
  return end_batch(c, st);
}

extern "C" il_status il_commit_index(il_ctx* c, il_stream s) {
  if (!c->matched || c->index_done) { set_error("il_commit_index before il_prefix_match"); return IL_ERR_STATE; }
  il_status r = commit_index(c, (cudaStream_t)s, c->batch + 1);
  if (r != IL_OK) return r;
  c->index_done = true;
  return IL_OK;
}

extern "C" il_status il_commit_records(il_ctx* c, uint32_t B_global, const uint32_t* final_ds_all,
                                       const il_refine_info* info_all, il_stream s) {
  if (!c->index_done) { set_error("il_commit_records before il_commit_index"); return IL_ERR_STATE; }
  if (!(c->cfg.flags & IL_F_PAIR)) { set_error("il_commit_records needs IL_F_PAIR"); return IL_ERR_STATE; }
  if (B_global > c->max_records) { set_error("B_global > max_global_batch"); return IL_ERR_ARG; }
  if (B_global && (!final_ds_all || !info_all)) { set_error("null records"); return IL_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)s;
  il_status r = commit_table(c, B_global, final_ds_all, info_all, st, c->batch + 1);
  if (r != IL_OK) return r;
  return end_batch(c, st);
}
