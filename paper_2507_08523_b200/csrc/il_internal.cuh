// il_internal.cuh — context layout and device helpers shared by the CUDA translation
// units of libinferlog_b200.so.  Nothing here is shared with the CPU checker.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/il.h"

namespace il {

constexpr uint32_t BS = 16;                 // KV block size (tokens)
constexpr uint32_t TOK_SEP = 1, TOK_TPL = 2;
constexpr uint64_t KEY_EMPTY = 0ull;
constexpr uint64_t KEY_TOMB = ~0ull;
constexpr uint32_t NONE32 = 0xFFFFFFFFu;
constexpr int MAXK = 8;
// a1-a2 for pools above this many demos use the inverted index (select_inv.cu) instead of the
// per-query pool scan; the index holds the pool in chunks of SIM_CHUNK demos (one shared-memory
// accumulator each)
constexpr uint32_t SIM_BIG_POOL = 1024;
constexpr uint32_t SIM_CHUNK = 16384;

// Device-resident scalars (one 256 B line).
struct DevScalars {
  uint32_t status;           // latched il_status
  uint32_t n_free;           // free-page stack size
  uint32_t resident;         // live index entries (== resident pages)
  uint32_t used_slots;       // live + tombstones
  uint32_t pinned;           // distinct pages pinned in the current batch
  uint32_t need_total;       // pages the current batch allocates
  uint32_t evict_m;          // blocks to evict
  uint32_t evicted;          // evicted by the current batch
  uint32_t suffix_total;     // sum of suffix lengths
  uint32_t rebuilds;
  uint32_t table_entries;
  uint32_t n_new_keys;       // ICL commit scratch
  uint32_t rebuild_flag;
  uint32_t n_tiles;          // attention work items
  uint32_t instr_hits;       // per batch: leading resident (verified) instruction blocks
  uint32_t n_dense;          // attention: dense M-tiles over all suffix rows (cascade phase 1)
  uint64_t stamp_min;        // eviction radix-select scratch
  uint64_t stamp_max;
  uint64_t sel_prefix;       // selected key prefix
  uint64_t sel_key;          // final threshold key
  uint64_t batch_done;       // committed batches (device copy: CUDA-graph replays advance it)
  uint32_t sel_remaining;
  uint32_t sel_shift;
  uint32_t cand;             // eviction candidates
  uint32_t q_total;          // attention: suffix rows of the batch (cu_q[B])
  uint32_t shared_blk;       // attention: blocks every request shares (same pages, all cached)
  uint32_t inserted;         // blocks this batch's il_commit_index made resident (records)
  uint32_t hit_sum;          // last prefix match: sum of capped hits, sum of full blocks,
  uint32_t full_sum;         //   sum of box-level hits
  uint32_t box_hit_sum;
  uint32_t map_used;         // residency-map slots holding a key
  uint32_t map_rebuilds;
  uint64_t ring_head;        // block-record FIFO (monotonic counters)
  uint64_t ring_tail;
  uint32_t dedup_sum;        // last prefix match: blocks shared in-batch (IL_F_DEDUP)
  uint32_t bd_n;             // in-batch dedup table: slots taken this batch (cleared by k_alloc_commit)
  uint32_t probe_batch;      // low bits of the batch whose instruction probe il_refine_batch ran (0 = none)
  uint32_t pad1;
};

struct Ctx {
  il_config cfg;
  uint32_t max_blocks = 0, n_slots = 0, slot_mask = 0;
  uint32_t n_demos = 0, n_instr = 0, n_instr_blocks = 0;
  bool pool_loaded = false, refined = false, matched = false, index_done = false;
  uint32_t max_records = 0;    // max(max_batch, max_global_batch): table-commit scratch size
  uint32_t last_B = 0;
  uint64_t batch = 0;        // b of the last committed batch
  // workspace carve
  DevScalars* sc = nullptr;
  // pool
  uint32_t *log_off, *log_tok, *tpl_off, *tpl_tok, *tid, *src;
  uint32_t *uniq_tok, *uniq_cnt, *uniq_n, *norm2;
  uint32_t *rend_off, *rend_tok, *rend_len;
  uint32_t *instr;
  uint64_t *instr_hash;       // chain hashes of the instruction's full blocks (pool_load)
  int32_t *instr_pages;      // per batch: pages of the instruction's leading resident blocks
  // ICL table
  uint32_t *tab_ds;          // [T][k] demo ids
  uint32_t *tab_tpl;         // [k][T] template ids (SoA: coalesced PMC scans)
  uint64_t* tab_stamp;
  // prefix index + pages
  uint64_t* slot_key;
  uint32_t* slot_page;
  uint32_t* claim;
  uint64_t* cstamp;
  uint64_t *pg_hash, *pg_parent, *pg_stamp;
  uint32_t *pg_tok, *pg_depth, *pg_slot, *pg_state, *pg_pin;
  uint32_t* free_list;
  // batch scratch
  uint32_t *need_off, *occ, *hist;
  int32_t *tab_find;         // per request: existing table slot of final_ds or -1
  uint32_t *tab_last;        // per request: last in batch with this key
  uint64_t *tab_hash;        // per request: hash of the final DS tuple
  uint32_t *tab_slot;        // per request: its slot in the dedup table
  uint64_t *dd_key;          // per-batch dedup table of final-DS hashes (cleared after use)
  uint32_t *dd_max;          // 1 + last admission index presenting the key
  uint32_t dd_mask = 0;
  uint32_t *tile_off;        // attention work decomposition
  uint32_t *tile_req;        // attention M-tile -> request
  uint4 *tile_desc;          // attention M-tile -> {request, first position, first suffix row, ntok | nblk << 8}
  uint32_t *pair_nsh;        // attention M-tile pair -> leading shared KV tiles
  float *attn_ml;            // cascade: per row log2 softmax mass of the shared-prefix partial
  uint64_t *evicted_list;
  uint32_t *guard_prompt;    // guard: DS_current prompt rows
  // inverted index of the pool (select_inv.cu; allocated when max_pool > SIM_BIG_POOL):
  // key (token, chunk) -> posting list of (demo, count)
  uint32_t inv_slots = 0, inv_mask = 0;
  uint64_t *inv_key;         // ((chunk << 32) | token) + 1; 0 = empty
  uint32_t *inv_off, *inv_len, *inv_fill;
  uint32_t *post_demo;       // (demo - chunk * SIM_CHUNK) << 18 | count
  // multi-GPU exchange (records.cu; allocated when max_global_batch > max_batch)
  uint32_t n_ranks_max = 1;  // ceil(max_global_batch / max_batch)
  uint32_t rec_R = 0;        // block records per export
  uint32_t ring_cap = 0;     // block-record FIFO capacity
  uint32_t map_slots = 0, map_smask = 0;
  uint64_t *ins_list;        // this batch's newly resident block hashes (il_commit_index)
  uint64_t *ring;            // block-record FIFO
  uint64_t *map_key;         // residency map: open addressing, key = chain hash (0 = empty)
  uint32_t *map_mask;        //   owner-rank bitmask (0 = dead key, reclaimed by the rebuild)
  uint64_t *map_tmp_key;     //   rebuild scratch
  uint32_t *map_tmp_mask;
  uint32_t *box_hit;         // per request: box-level hit count of the last prefix match
  // in-batch dedup (IL_F_DEDUP, match.cu): snapshot hits before dedup, and the batch's table
  // hash -> lowest admission index presenting it as a block it computes
  uint32_t *dec_cu;          // 0, 1, .., max_batch (il_decode_attn's row offsets)
  uint32_t *hit_local;
  uint64_t *bd_key;          // 0 = empty (chain hashes are never 0, Z18)
  uint32_t *bd_owner;        // ~(lowest admission index); 0 = none
  uint32_t *bd_list;         // slots taken this batch
  uint32_t bd_mask = 0;
  uint32_t *icl_fds;         // il_commit_apply: gathered ICL records, global admission order
  il_refine_info *icl_info;
  bool map_active = false;   // host: an il_commit_apply with n_ranks > 1 has run
  bool exported = false;     // host: il_commit_export ran for the current batch
  const uint32_t* sel_topk = nullptr;   // host: il_select_batch ran for (sel_B, sel_topk)
  uint32_t sel_B = 0;
  // pointers remembered between calls (caller-owned)
  const uint32_t* final_ds = nullptr;
  const il_refine_info* info = nullptr;
  const uint32_t* prompt_tok = nullptr;
  const uint32_t* prompt_len = nullptr;
  const uint64_t* block_hash = nullptr;
  const uint32_t* hit = nullptr;
  const int32_t* block_table = nullptr;
  int num_sms = 148;
  int ev_blocks = 0, rb_blocks = 0, mb_blocks = 0;   // cooperative grid sizes (k_evict, k_rebuild,
                                                     // k_map_rebuild), set per context
  int ev_per_sm = 1, rb_per_sm = 1, mb_per_sm = 1;   // their CTAs per SM
  int attn_ctas = 0;                                 // il_set_sm_split: attention grid (0 = every SM)
  uint64_t launches = 0;     // kernels launched by this context (host counter)
};

// ---------------------------------------------------------------- error plumbing (host)
void set_error(const std::string& msg);
il_status cuda_check(cudaError_t e, const char* what);
// per-context one-time setup on the current device (il_create): kernel attributes and
// occupancy-derived grid sizes are per device, so nothing is cached process-wide
il_status match_setup(Ctx* c);
il_status commit_setup(Ctx* c);
il_status attn_setup(Ctx* c);
il_status records_setup(Ctx* c);
il_status records_reset(Ctx* c, cudaStream_t st);
il_status inv_build(Ctx* c, uint32_t n_demos, cudaStream_t st);       // select_inv.cu (pool_load)
il_status inv_select(Ctx* c, uint32_t B, const uint32_t* q_off, const uint32_t* q_tok,
                     const uint32_t* q_src, uint32_t* topk, cudaStream_t st);
il_status inv_setup(Ctx* c);
// shared between commit.cu and records.cu
il_status commit_table(Ctx* c, uint32_t B, const uint32_t* final_ds, const il_refine_info* info,
                       cudaStream_t st, uint64_t b_cur);
il_status end_batch(Ctx* c, cudaStream_t st);
// record-buffer layout (il.h il_record_bytes)
struct RecHeader {
  uint32_t magic, B, k, n_blk;
  uint64_t batch;
  uint32_t backlog, pad[9];
};
static_assert(sizeof(RecHeader) == 64, "record header");
constexpr uint32_t REC_MAGIC = 0x43524C49u;   // 'ILRC'
__host__ __device__ inline size_t rec_fds_off() { return 64; }
__host__ __device__ inline size_t rec_info_off(uint32_t max_batch, uint32_t k) {
  return 64 + (((size_t)max_batch * k * 4 + 15) & ~size_t(15));
}
__host__ __device__ inline size_t rec_blk_off(uint32_t max_batch, uint32_t k) {
  return rec_info_off(max_batch, k) + (size_t)max_batch * 16;
}
__host__ __device__ inline size_t rec_bytes(uint32_t max_batch, uint32_t k, uint32_t R) {
  return (rec_blk_off(max_batch, k) + (size_t)R * 8 + 255) & ~size_t(255);
}
#define IL_CUDA(call)                                                  \
  do {                                                                 \
    cudaError_t _e = (call);                                           \
    if (_e != cudaSuccess) return ::il::cuda_check(_e, #call);         \
  } while (0)
#define IL_LAUNCH_CHECK(what)                                          \
  do {                                                                 \
    cudaError_t _e = cudaGetLastError();                               \
    if (_e != cudaSuccess) return ::il::cuda_check(_e, what);          \
  } while (0)

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ void latch(DevScalars* sc, uint32_t code) {
  atomicCAS(&sc->status, 0u, code);
}

// Chain hash (Z17): splitmix64 finalizer; 16 independent lane terms per block,
// summed mod 2^64, then a serial fold H_j = mix(H_{j-1} * PHI + content_j).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
constexpr uint64_t PHI64 = 0x9E3779B97F4A7C15ull;
__host__ __device__ __forceinline__ uint64_t root_hash(uint64_t seed) {
  return mix64(seed ^ 0x494E4645524C4F47ull);
}
__device__ __forceinline__ uint64_t lane_term(uint32_t tok, uint32_t i) {
  return mix64(((uint64_t)tok << 8) ^ (uint64_t)i ^ PHI64);
}
__device__ __forceinline__ uint64_t chain_step(uint64_t prev, uint64_t content) {
  uint64_t h = mix64(prev * PHI64 + content);
  h = (h == KEY_EMPTY) ? 1ull : h;
  h = (h == KEY_TOMB) ? (KEY_TOMB - 1ull) : h;
  return h;
}
// content hash of the 16 tokens at t (16-byte aligned).  kReadOnly: the row was written by an
// earlier kernel and stays read-only for this one, so the non-coherent path (__ldg) is allowed;
// otherwise (a row written earlier in the SAME kernel, e.g. the guard of k_refine) ld.global.cg.
template <bool kReadOnly = true>
__device__ __forceinline__ uint64_t block_content(const uint32_t* __restrict__ t, uint32_t tok[16]) {
  const uint4* v = reinterpret_cast<const uint4*>(t);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 x = kReadOnly ? __ldg(v + q) : __ldcg(v + q);   // .cg: coherent at L2, never .nc
    tok[4 * q + 0] = x.x; tok[4 * q + 1] = x.y; tok[4 * q + 2] = x.z; tok[4 * q + 3] = x.w;
  }
  uint64_t s = 0;
#pragma unroll
  for (uint32_t i = 0; i < 16; ++i) s += lane_term(tok[i], i);
  return mix64(s);
}

__device__ __forceinline__ uint64_t stamp_of(uint64_t b, uint32_t i) { return (b << 32) | (uint64_t)i; }

// open-addressing probe of the prefix index: returns page or NONE32
__device__ __forceinline__ uint32_t index_find(const uint64_t* __restrict__ slot_key,
                                               const uint32_t* __restrict__ slot_page,
                                               uint32_t mask, uint64_t key, uint32_t* slot_out) {
  uint32_t s = (uint32_t)(key ^ (key >> 32)) & mask;
  for (uint32_t n = 0; n <= mask; ++n) {
    uint64_t k = slot_key[s];
    if (k == key) { if (slot_out) *slot_out = s; return slot_page[s]; }
    if (k == KEY_EMPTY) return NONE32;
    s = (s + 1) & mask;
  }
  return NONE32;
}

__host__ __device__ __forceinline__ uint32_t cdiv(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

// residency map lookup (multi-GPU): some rank holds the block with chain hash `key`
__device__ __forceinline__ bool map_has(const Ctx& c, uint64_t key) {
  uint32_t s = (uint32_t)(key ^ (key >> 32)) & c.map_smask;
  for (uint32_t n = 0; n <= c.map_smask; ++n) {
    const uint64_t k = c.map_key[s];
    if (k == key) return c.map_mask[s] != 0;
    if (k == KEY_EMPTY) return false;
    s = (s + 1) & c.map_smask;
  }
  return false;
}


// block-wide exclusive scan of one value per thread (1024 threads)
__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t* s_w, uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(~0u, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t t = s_w[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(~0u, t, o);
      if (lane >= (uint32_t)o) t += y;
    }
    s_w[lane] = t;
  }
  __syncthreads();
  const uint32_t before = (w ? s_w[w - 1] : 0) + x - v;
  *total = s_w[31];
  __syncthreads();
  return before;
}

// block-wide inclusive prefix max of one int32 per thread (1024 threads)
__device__ __forceinline__ int32_t block_scan_max(int32_t v, int32_t* s_w) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(~0u, x, o);
    if (lane >= (uint32_t)o) x = max(x, y);
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    int32_t t = s_w[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(~0u, t, o);
      if (lane >= (uint32_t)o) t = max(t, y);
    }
    s_w[lane] = t;
  }
  __syncthreads();
  const int32_t r = w ? max(x, s_w[w - 1]) : x;
  __syncthreads();
  return r;
}

}  // namespace il

struct il_ctx : public il::Ctx {};
