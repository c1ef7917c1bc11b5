/* il.h — C ABI of libinferlog_b200.so: the InferLog hot path on B200 (sm_100a).
 *
 * The path (§3.2, on top of prefix caching P:192-198):
 *   il_refine_batch  kNN demo selection + PAIR matching / modifying /
 *                    reordering against the ICL Table + prompt render
 *   il_prefix_match  chained 16-token KV-block hashes + longest cached prefix (P:195-198,
 *                    fig:prefixcache) + LRU pin / evict / page allocation
 *   il_prefill_attn  only the uncached suffix runs: append its K/V to pages, then causal
 *                    attention over the paged cached prefix + the suffix
 *   il_commit        after the batch: insert the new blocks into the prefix index and apply
 *                    the ICL Table update rules
 *
 * Conventions
 *  - Pointers are DEVICE pointers unless the name ends in _h (host).  Every buffer is owned
 *    by the caller (PyTorch allocates them); the workspace is handed over once at create and
 *    the library never allocates device memory.
 *  - All calls are asynchronous on the caller's stream and never synchronize, except
 *    il_status_sync / il_stats_sync.  Device-computed sizes (sum of suffix lengths, pages
 *    needed) stay on the device.
 *  - Errors: host-detectable errors return immediately (IL_ERR_ARG / IL_ERR_STATE).  Errors
 *    the device detects (capacity, an over-long prompt) latch into a device status word and
 *    surface from il_status_sync(); after a latched error the context's cache state is
 *    unspecified and it must be reloaded with il_pool_load.  il_last_error() returns the
 *    calling thread's last message.
 *  - Threading: one context per GPU; calls on a context must be serialized in admission
 *    order (single writer).
 *  - Determinism: integer outputs (top-k, final DS, PMC, rule, chain hashes, hit counts,
 *    evicted set, table and index contents) are bit-exact functions of (config, inputs,
 *    history) and equal the CPU oracle's (tests/test_parity_*.py).  Physical page numbers
 *    are NOT part of that contract.
 *
 * Batch semantics (reading Z1): every request of a batch matches against the
 * table and index as they were after the previous commit ("snapshot"), and the commit
 * applies the batch's updates in admission order.  B = 1 reproduces the sequential
 * semantics of the paper's OrderedDict ICL Table exactly.
 */
#ifndef INFERLOG_IL_H
#define INFERLOG_IL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct il_ctx il_ctx;
typedef struct CUstream_st* il_stream;   /* == cudaStream_t; NULL = legacy default stream */
typedef uint16_t il_bf16;                /* bfloat16 bit pattern */

typedef enum {
  IL_OK = 0,
  IL_ERR_ARG = 1,       /* bad size / flag; k > eligible demos ("argument error");
                           a rendered prompt longer than max_prompt_tokens (latched) */
  IL_ERR_CAPACITY = 2,  /* batch needs more KV pages than free + evictable, or
                           more suffix rows than max_suffix_tokens (latched) */
  IL_ERR_STATE = 3,     /* call out of order: refine before pool_load, commit before match */
  IL_ERR_INTERNAL = 4,  /* device invariant broken ("internal error") */
  IL_ERR_CUDA = 5       /* a CUDA runtime call failed (message in il_last_error) */
} il_status;

typedef enum { IL_SIM_COSINE = 0, IL_SIM_JACCARD = 1 } il_sim;

enum {
  IL_F_PAIR = 1u << 0,         /* PAIR on; off = naive prefix caching (paper baseline "PC") */
  IL_F_GUARD = 1u << 1,        /* never-worse guard (Z25; not in the paper) */
  IL_F_EXCLUDE_SELF = 1u << 2, /* a query never selects its own dataset row */
  IL_F_VERIFY = 1u << 3,       /* a hit also requires equal block tokens + parent hash (Z19) */
  IL_F_DEDUP = 1u << 4         /* NEXT-1 in-batch dedup (Z22b): a full block an earlier
                                  request of the batch computes (same depth, same prefix, equal
                                  tokens) is not computed again; the later request's hit run
                                  continues through it and its block table points at the
                                  earlier request's page.  hit_blocks then counts those too. */
};

typedef struct {
  uint32_t k;                  /* demonstrations per prompt (N in P:357), 1..8 */
  uint32_t table_capacity;     /* T: ICL Table entries, <= 8192 */
  uint32_t kv_pages;           /* C: 16-token KV pages in the caller's page tensors */
  uint32_t max_batch;          /* B per call, <= 8192 */
  uint32_t max_prompt_tokens;  /* prompt row stride; longer prompts latch IL_ERR_ARG */
  uint32_t max_pool;           /* M: demos in the pool */
  uint32_t max_pool_tokens;    /* sum over demos of (log + template) tokens */
  uint32_t max_log_tokens;     /* longest log (demo or query), <= 256 */
  uint32_t max_suffix_tokens;  /* rows of q / k_new / v_new / out the caller allocated */
  uint32_t n_q_heads, n_kv_heads, head_dim;   /* Hq % Hkv == 0; head_dim 64 or 128 */
  uint32_t metric;             /* il_sim */
  uint32_t flags;              /* IL_F_* */
  uint64_t hash_seed;          /* chain-hash root (Z17) */
  uint32_t max_global_batch;   /* records per il_commit_records / il_commit_apply (multi-GPU:
                                  world x B); 0 = max_batch.  > max_batch enables the multi-GPU
                                  block records and the residency map (ranks = ceil(./max_batch) <= 32) */
  uint32_t max_block_records;  /* multi-GPU: block records one il_commit_export carries; 0 = 16 x max_batch */
  uint32_t max_decode_tokens;  /* D: KV pages reserved per request for D decode tokens after the prompt
                                  (il_prefix_match allocates ceil((L + D) / 16) - hit pages, il_commit
                                  frees them); prompts must fit max_prompt_tokens - D.  0 = prefill only */
  uint32_t reserved1;          /* must be 0 */
} il_config;

/* Per-request refinement outcome (SPEC S:190-193 RefinementResult). */
typedef struct {
  uint64_t target_stamp;       /* recency stamp of DS_target, (batch << 32 | admission index); 0 = none */
  int32_t target_slot;         /* device table slot of DS_target; -1 = none */
  uint8_t pmc;                 /* prefix-matching count of DS_target; 0 = none */
  uint8_t rule;                /* 1, 2 or 3 */
  uint8_t reverted;            /* the guard kept DS_current (Z25) */
  uint8_t matched;             /* a target with PMC >= 1 was found */
} il_refine_info;

typedef struct {               /* counters of the last committed batch (il_stats_sync) */
  uint64_t batch;              /* b of the last commit (1-based) */
  uint32_t resident_blocks;    /* |prefix index| */
  uint32_t free_pages;
  uint32_t table_entries;
  uint32_t evicted_blocks;     /* evicted by the last il_prefix_match */
  uint32_t need_pages;         /* pages the last il_prefix_match allocated */
  uint32_t suffix_tokens;      /* sum of suffix lengths of the last il_prefix_match */
  uint32_t index_rebuilds;     /* tombstone compactions so far */
  uint32_t status;             /* latched il_status */
  uint64_t launches;           /* kernels this context has launched so far */
  uint32_t hit_blocks;         /* sum of capped hits of the last il_prefix_match (this rank;
                                  with IL_F_DEDUP including the in-batch shared blocks) */
  uint32_t box_hit_blocks;     /* the same against the box (this rank's index or the residency map) */
  uint32_t full_blocks;        /* sum of floor(L_i / 16) of the last il_prefix_match */
  uint32_t record_backlog;     /* block records waiting for a later il_commit_export */
  uint32_t map_slots_used;     /* residency-map slots holding a key (live or dead) */
  uint32_t dedup_blocks;       /* IL_F_DEDUP: blocks of hit_blocks shared in-batch (not cached) */
} il_stats;

/* ---- lifecycle ---------------------------------------------------------------------- */
il_status il_workspace_bytes(const il_config* cfg_h, size_t* bytes_h);
il_status il_create(const il_config* cfg_h, void* workspace, size_t bytes, il_stream s, il_ctx** out_h);
il_status il_destroy(il_ctx* ctx);
il_status il_status_sync(il_ctx* ctx, il_stream s);      /* sync s, return + clear latched status */
il_status il_stats_sync(il_ctx* ctx, il_stream s, il_stats* out_h);
/* The same counters written to DEVICE memory by a kernel on s (no sync; capturable in a CUDA
 * graph): per-batch accounting inside a timed loop.  out_d: one il_stats, 8-byte aligned;
 * `launches` holds the host counter at the time of the call (at capture, for a graph). */
il_status il_stats_async(il_ctx* ctx, il_stats* out_d, il_stream s);
const char* il_last_error(void);                          /* thread-local */
/* Cross-batch pipelining (a serving schedule, not a change of what is computed): the attention
 * of batch b (il_synth_qkv* + il_prefill_attn on one stream) may run CONCURRENTLY with
 * il_commit of batch b and il_select_batch / il_refine_batch / il_prefix_match of batch b+1 on a
 * second stream, provided (1) the two batches use different per-batch buffers (prompts, block
 * tables, cu_q, prefix_len, Q, out, ...), (2) calls that read or write KV page CONTENTS for batch
 * b+1 (il_synth_qkv_paged, il_prefill_attn) are ordered after batch b's il_prefill_attn, and (3)
 * il_commit of batch b is ordered after its il_prefix_match.  Pages batch b reads may be freed or
 * evicted (metadata) by those calls, but only batch b+1's page writes reuse them.  For the two
 * streams to overlap on the device, il_set_sm_split(ctx, n) gives il_prefill_attn's persistent
 * grid n CTAs (one per SM) and sizes the cooperative integer kernels (LRU eviction, index
 * compaction, residency-map compaction) to fit on the remaining SMs; n = 0 restores the default
 * (attention on every SM).  IL_ERR_ARG if n >= the SM count.  Host-side only; takes effect for
 * later calls (and captures). */
il_status il_set_sm_split(il_ctx* ctx, uint32_t attn_ctas);

/* ---- il_pool_load: the candidate set ("samples 200 logs ... to construct the
 * candidate set").  CSR device arrays of n_demos demos: log tokens, template tokens,
 * interned template ids, dataset row (for IL_F_EXCLUDE_SELF), and the common
 * instruction.  Builds the per-demo token sets (a1) and rendered demos (a5), and
 * resets the ICL Table and the prefix index (demo ids change meaning).  The input buffers
 * may be freed once the stream reaches this call.  IL_ERR_ARG if n_demos is outside
 * [k, max_pool], the pool exceeds max_pool_tokens, or n_instr exceeds max_prompt_tokens or
 * 16,384 tokens (1,024 instruction blocks, the per-batch instruction pin covers no more). */
il_status il_pool_load(il_ctx* ctx, uint32_t n_demos,
                       const uint32_t* log_off, const uint32_t* log_tok,
                       const uint32_t* tpl_off, const uint32_t* tpl_tok,
                       const uint32_t* template_id, const uint32_t* src_index,
                       const uint32_t* instr_tok, uint32_t n_instr, il_stream s);

/* ---- il_refine_batch: for each of B query logs (CSR q_off[B+1] / q_tok), in admission
 * order i = 0..B-1:
 *   topk[i][0..k)      the k most similar demos (exact cosine over token counts or Jaccard
 *                      over token sets), emitted ascending by similarity, ties by demo index
 *                      (Z4-Z8)
 *   final_ds[i][0..k)  after PAIR against the table snapshot: rule 1 uses the
 *                      target verbatim, rule 2 keeps DS_current, rule 3 modifies + reorders
 *   info[i]            see il_refine_info
 *   prompt_tok[i][..]  instruction ++ render(d_1..d_k) ++ query, render(m) = log ++ [TPL] ++
 *                      template ++ [SEP] (Z9); row stride = cfg.max_prompt_tokens; the buffer
 *                      must be 16-byte aligned (IL_ERR_ARG otherwise)
 *   prompt_len[i]
 * q_src[i] is the query's dataset row (only read with IL_F_EXCLUDE_SELF; may be NULL). */
il_status il_refine_batch(il_ctx* ctx, uint32_t B,
                          const uint32_t* q_off, const uint32_t* q_tok, const uint32_t* q_src,
                          uint32_t* topk, uint32_t* final_ds, il_refine_info* info,
                          uint32_t* prompt_tok, uint32_t* prompt_len, il_stream s);

/* ---- il_prefix_match: for each prompt (row stride cfg.max_prompt_tokens):
 *   block_hash[i][j]   chain hash of full block j (Z17), j < floor(L_i/16); row stride = max_blocks
 *   hit_blocks[i]      leading blocks resident (and verified) in the index snapshot, capped at
 *                      floor((L_i-1)/16) so the last token is always computed (Z19, Z20)
 *   block_table[i][j]  page of block j: hit pages, then freshly allocated pages; row stride =
 *                      max_blocks = ceil(cfg.max_prompt_tokens / 16)
 *   prefix_len[i]      16 * hit_blocks[i];  cu_q[B+1] cumulative suffix lengths
 * Hit pages are pinned; if the batch needs more pages than are free, the least recently used
 * unpinned blocks are evicted in (stamp asc, depth desc) order (Z21).  prompt_tok,
 * prompt_len, block_hash, hit_blocks and block_table must stay valid until il_commit. */
il_status il_prefix_match(il_ctx* ctx, uint32_t B,
                          const uint32_t* prompt_tok, const uint32_t* prompt_len,
                          uint64_t* block_hash, uint32_t* hit_blocks,
                          int32_t* block_table, int32_t* prefix_len, int32_t* cu_q, il_stream s);

/* ---- il_prefill_attn: rows r in [cu_q[i], cu_q[i+1]) are the suffix tokens of request i at
 * absolute positions p = prefix_len[i] + (r - cu_q[i]).  prefix_len is 16 x hit after
 * il_prefix_match; any position works (paged DECODE: one row per request at
 * position L_i + t, its K/V written into the decode pages il_prefix_match reserved, attending over
 * the prompt and the t decode tokens before it; see max_decode_tokens).  First writes k_new/v_new rows into
 * the request's pages, then for every q-head h:
 *   out[r][h] = sum_{j <= p} softmax_j(q[r][h] . K_j * scale) V_j,  kv-head = h / (Hq/Hkv)
 * with K_j, V_j read from the pages (cached prefix and the just-written suffix alike).
 *   q, out        [max_suffix_tokens][Hq][d]  bf16;  lse [..][Hq] f32 natural log, or NULL
 *   k_new, v_new  [max_suffix_tokens][Hkv][d] bf16, or both NULL when the suffix K / V are already
 *                 in the pages (il_synth_qkv_paged: the projection epilogue wrote them)
 *   k_pages, v_pages  [C][Hkv][16][d] bf16, caller-owned, persistent across batches
 * bf16 in, fp32 accumulation (Z26); parity <= 1e-2 vs the fp64 oracle (Z27).
 * Runs on two tcgen05/TMA kernels (head_dim 64 or 128, Hq/Hkv in 1..8; il_create rejects any
 * other shape with IL_ERR_ARG, there is no other attention path): the keys every request of the
 * batch reads from the same pages (the instruction) as one dense pass over all suffix rows,
 * then each request's own keys, merged with the dense pass's partial through log-sum-exp (the
 * cascade).  Requires a preceding il_prefix_match of the same batch
 * (IL_ERR_STATE otherwise); out and the workspace hold the cascade's partial between the two
 * launches, so out must not be read before the call's work completes on stream s. */
il_status il_prefill_attn(il_ctx* ctx, uint32_t B, const int32_t* cu_q, const int32_t* prefix_len,
                          const int32_t* block_table,
                          const il_bf16* q, const il_bf16* k_new, const il_bf16* v_new,
                          il_bf16* k_pages, il_bf16* v_pages, il_bf16* out, float* lse,
                          float softmax_scale, il_stream s);

/* ---- il_decode_attn: paged decode attention (decode is the part of request
 * latency that is not prefill): ONE query row per request at absolute position pos[i]
 * (attending keys 0..pos[i], the prompt and the decode tokens before it), after il_prefix_match
 * reserved the pages for position pos[i] (il_config.max_decode_tokens).  Same page layout and
 * numerics as il_prefill_attn.
 *   pos          [B] int32   position of request i's row (= its prefix length)
 *   block_table  [B][max_blocks] as from il_prefix_match
 *   q            [B][Hq][d] bf16;  k_new, v_new [B][Hkv][d] bf16, appended at pos[i], or both NULL
 *                (the projection already wrote them into the pages)
 *   out          [B][Hq][d] bf16;  lse [B][Hq] fp32 natural-log LSE, or NULL
 * The keys below the batch-shared prefix run on the tensor kernel's dense phase (rows of all
 * requests stacked), each request's own keys on a CUDA-core kernel (one warp per request and kv
 * head: a one-row M-tile would be 97% padding).  IL_ERR_STATE before il_prefix_match; IL_ERR_ARG
 * for B > max_batch or one of k_new / v_new NULL. */
il_status il_decode_attn(il_ctx* ctx, uint32_t B, const int32_t* pos, const int32_t* block_table,
                         const il_bf16* q, const il_bf16* k_new, const il_bf16* v_new,
                         il_bf16* k_pages, il_bf16* v_pages, il_bf16* out, float* lse,
                         float softmax_scale, il_stream s);

/* ---- il_commit: end of batch ("update the elements in the ICL Table after processing
 * the request").  Inserts the batch's new full blocks into the prefix index (first request in
 * admission order owns the page; duplicates and partial-block pages are freed, Z22-Z23) and
 * applies the ICL Table records in admission order (rule 1 refreshes the target; rules 2/3
 * upsert the final DS; the target of rule 3 keeps its position), then keeps the T most recent
 * entries (Z2, Z3, Z14). */
il_status il_commit(il_ctx* ctx, il_stream s);

/* ---- multi-GPU: requests shard by admission order (rank r takes the r-th
 * contiguous slice of the global batch), every rank keeps its own KV pages and prefix index,
 * and the ICL Table is REPLICATED: each rank refines its slice against the same table
 * snapshot, the per-request records of all ranks (final_ds[i][0..k), il_refine_info[i]) are
 * all-gathered in global admission order, and every rank applies all of them, so the tables
 * stay identical and equal to a one-GPU run over the global batch (P:356-363 applied to the
 * whole batch).
 *   il_commit_index    the prefix-index half of il_commit (this rank's blocks only)
 *   il_commit_records  the ICL Table half over B_global gathered records (device arrays,
 *                      global admission order; info[].target_slot refers to the replicated
 *                      table).  Ends the batch.  B_global <= cfg.max_global_batch.
 * il_commit == il_commit_index + il_commit_records over this rank's own records. */
il_status il_commit_index(il_ctx* ctx, il_stream s);
il_status il_commit_records(il_ctx* ctx, uint32_t B_global, const uint32_t* final_ds_all,
                            const il_refine_info* info_all, il_stream s);

/* ---- the per-batch exchange as ONE fixed-size record buffer per rank (
 * north star: "all-gather prefix-index updates").  A record buffer holds
 *   header (64 B): magic 'ILRC', B of this rank, k, n block records, batch b, backlog
 *   ICL records:   final_ds [max_batch][k] u32 (padded to 16 B), il_refine_info [max_batch]
 *   block records: [max_block_records] u64 chain hashes: every block this rank's prefix index
 *                  gained (il_commit_index) or lost (LRU eviction in il_prefix_match) since the
 *                  last export, oldest first.  More than max_block_records wait in the context
 *                  (FIFO, `record_backlog` in il_stats) for the next export; a FIFO overflow
 *                  latches IL_ERR_CAPACITY.
 * The caller all-gathers the n_ranks buffers rank-major (one all_gather_into_tensor) and every
 * rank calls il_commit_apply on the result:
 *   - the ICL records of all ranks are applied to the replicated table in global admission
 *     order (exactly il_commit_records over their concatenation);
 *   - the block records build the replicated RESIDENCY MAP, hash -> owner-rank bitmask
 *     ("shared prefix index", BASELINE configs[2]).  A block record toggles its rank's bit
 *     (an index gains and loses a hash alternately, so applying a buffer's records in any order
 *     gives the same map: the map equals the union of the ranks' indices whenever no records
 *     are waiting).
 * From then on il_prefix_match also computes every request's BOX-LEVEL hit count: the leading
 * blocks resident in this rank's index or in the map (chain hash only, not verified), capped
 * as Z20 -- the hit rate that box-wide reuse of remote pages would give (il_stats, il_box_hit_dump).
 *   il_record_bytes   bytes of one rank's record buffer (256-byte multiple)
 *   il_commit_export  after il_commit_index: write this rank's records into rec (device)
 *   il_commit_apply   recs_all = n_ranks buffers back to back, rank r's holding
 *                     batch_per_rank_h[r] requests (host array); sum <= max_global_batch.
 *                     Ends the batch (il_commit == index + export + apply over one rank). */
il_status il_record_bytes(const il_config* cfg_h, size_t* bytes_h);
il_status il_commit_export(il_ctx* ctx, void* rec, il_stream s);
il_status il_commit_apply(il_ctx* ctx, const void* recs_all, uint32_t n_ranks,
                          const uint32_t* batch_per_rank_h, il_stream s);
/* box-level hit counts of the last il_prefix_match ([B] host), zeros before any il_commit_apply */
il_status il_box_hit_dump(il_ctx* ctx, il_stream s, uint32_t* box_hit_h, uint32_t B);

/* ---- a1-a2 alone (kNN selection into topk), so that a multi-GPU driver can overlap the
 * previous batch's record all-gather with it: selection reads only the pool, never the ICL
 * Table.  A following il_refine_batch of the same B with the same topk buffer does not repeat
 * it. */
il_status il_select_batch(il_ctx* ctx, uint32_t B, const uint32_t* q_off, const uint32_t* q_tok,
                          const uint32_t* q_src, uint32_t* topk, il_stream s);

/* ---- bench / test helper (not part of the method): deterministic bf16 Q, K, V for the
 * suffix rows from (seed, token, absolute position, head, dim) — the counter-based
 * generator of DESIGN.md Z28, so cached pages equal recomputation.  q_scale scales Q.
 * il_synth_qkv_paged writes K and V straight into the request's KV pages (block_table of the
 * preceding il_prefix_match), as a model's QKV-projection epilogue writes the paged cache; the
 * following il_prefill_attn then gets k_new = v_new = NULL and skips its append pass.  A NULL q
 * skips the Q heads, NULL k / v (both) the K and V heads: under cross-batch pipelining the next
 * batch's Q can be written while this batch's attention runs, its K / V only after. */
il_status il_synth_qkv(il_ctx* ctx, uint32_t B, const uint32_t* prompt_tok, const int32_t* cu_q,
                       const int32_t* prefix_len, uint64_t seed, float q_scale,
                       il_bf16* q, il_bf16* k_new, il_bf16* v_new, il_stream s);
il_status il_synth_qkv_paged(il_ctx* ctx, uint32_t B, const uint32_t* prompt_tok, const int32_t* cu_q,
                             const int32_t* prefix_len, const int32_t* block_table, uint64_t seed,
                             float q_scale, il_bf16* q, il_bf16* k_pages, il_bf16* v_pages, il_stream s);

/* ---- debug / parity helpers: copy the resident index (hash, stamp, depth, parent hash;
 * unordered) and the ICL Table (ds [T][k], stamp [T]; empty slots have stamp 0) to host. */
il_status il_index_dump(il_ctx* ctx, il_stream s, uint64_t* hash_h, uint64_t* stamp_h,
                        uint32_t* depth_h, uint64_t* parent_h, uint32_t* n_h);
il_status il_table_dump(il_ctx* ctx, il_stream s, uint32_t* ds_h, uint64_t* stamp_h);
/* evicted block hashes of the last il_prefix_match (unordered) */
il_status il_evicted_dump(il_ctx* ctx, il_stream s, uint64_t* hash_h, uint32_t* n_h);

#ifdef __cplusplus
}
#endif
#endif
