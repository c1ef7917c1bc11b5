/* oracle.h — C ABI of liboracle.so.
 *
 * TEST INFRASTRUCTURE, NOT THE PRODUCT.  A plain, slow, obviously-correct CPU
 * implementation of the InferLog hot path (§3.2 "Prefix-Aware ICL Refinement",
 * P:316-363; prefix caching P:192-198) written from the paper and SURVEY.md §8(c).
 * It shares no code with paper_2507_08523_b200/ (the CUDA path) and neither imports the
 * other.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load it.
 *
 * Pins: see tests/test_oracle_pins.py.  The chain-hash VALUES (Z17) are "parity
 * unpinned" by the paper: they are fixed only by the spec text in DESIGN.md, which this
 * file and the CUDA path implement independently.
 *
 * Conventions: all pointers are host pointers; arrays are caller-owned.  Return 0 on
 * success, 1 = argument error, 2 = capacity error, 3 = state error.
 */
#ifndef INFERLOG_ORACLE_H
#define INFERLOG_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { OR_SIM_COSINE = 0, OR_SIM_JACCARD = 1 };
enum { OR_F_PAIR = 1u << 0, OR_F_GUARD = 1u << 1, OR_F_EXCLUDE_SELF = 1u << 2, OR_F_VERIFY = 1u << 3, OR_F_DEDUP = 1u << 4 };

typedef struct or_state or_state;

or_state* or_create(uint32_t k, uint32_t table_capacity, uint32_t kv_pages, uint32_t metric,
                    uint32_t flags, uint64_t hash_seed);
void or_destroy(or_state*);

int or_pool_load(or_state*, uint32_t n, const uint32_t* log_off, const uint32_t* log_tok,
                 const uint32_t* tpl_off, const uint32_t* tpl_tok, const uint32_t* template_id,
                 const uint32_t* src_index, const uint32_t* instr, uint32_t n_instr);

/* One batch.  Requests match against the snapshot
 * (Table_b, Index_b) and commit in admission order (reading Z1).
 * info[B][4] = {pmc, rule (1,2,3), reverted, matched}; target_stamp[B] (0 = none).
 * prompt_tok is [B][prompt_stride]; block_hash is [B][max_blocks].
 * evicted: in *n_evicted the capacity, out the count (hashes in eviction order). */
int or_run_batch(or_state*, uint32_t B, const uint32_t* q_off, const uint32_t* q_tok,
                 const uint32_t* q_src, uint32_t* topk, uint32_t* final_ds, int32_t* info,
                 uint64_t* target_stamp, uint32_t* prompt_len, uint32_t* prompt_tok,
                 uint32_t prompt_stride, uint64_t* block_hash, uint32_t max_blocks,
                 uint32_t* hit, uint64_t* evicted, uint32_t* n_evicted);

/* The same batch over G data-parallel ranks: rank r owns the admission slice
 * [r*B/G, (r+1)*B/G) and its own prefix index st[r]; the ICL Tables of all st[] must be
 * identical on entry and receive all B records in global admission order (table stamps use the
 * global admission index, a rank's index stamps the index within its slice).  Outputs as
 * or_run_batch for the global batch (hits from the owning rank's index; evictions rank-major,
 * n_evicted_rank[G] per rank, may be NULL).  Returns 4 if the tables differ on entry.  G = 1 is
 * or_run_batch. */
int or_run_batch_dp(or_state** st, uint32_t G, uint32_t B, const uint32_t* q_off, const uint32_t* q_tok,
                    const uint32_t* q_src, uint32_t* topk, uint32_t* final_ds, int32_t* info,
                    uint64_t* target_stamp, uint32_t* prompt_len, uint32_t* prompt_tok,
                    uint32_t prompt_stride, uint64_t* block_hash, uint32_t max_blocks,
                    uint32_t* hit, uint64_t* evicted, uint32_t* n_evicted, uint32_t* n_evicted_rank);

uint64_t or_batch_index(const or_state*);           /* b of the last committed batch */
/* reserve KV pages for d decode tokens per request: step 7 allocates
 * ceil((L + d) / 16) - h pages per request; prompts must fit prompt_stride - d.  Default 0. */
void or_set_decode(or_state*, uint32_t d);
/* SURVEY §8(e) residency map (replicated on every rank of a run_batch_dp): chain hash -> bitmask
 * of the ranks whose index holds it, i.e. the union of the ranks' indices after the batch; and
 * the box-level hit counts of the last batch ([B]): each request's own leading run continued
 * through blocks present in the map at the snapshot (hash only), capped as Z20. */
void or_box_hits(const or_state*, uint32_t* out);
uint32_t or_box_map_size(const or_state*);
void or_box_map_dump(const or_state*, uint64_t* hash, uint32_t* mask);   /* sorted by hash */
uint32_t or_index_size(const or_state*);
/* sorted by hash: hash, stamp, depth, parent hash */
void or_index_dump(const or_state*, uint64_t* hash, uint64_t* stamp, uint32_t* depth, uint64_t* parent);
uint32_t or_table_size(const or_state*);
/* sorted by stamp ascending (head = least recent): ds [n][k], stamp [n] */
void or_table_dump(const or_state*, uint32_t* ds, uint64_t* stamp);

/* --- pieces exposed for the pins (tests/test_oracle_pins.py) --- */
/* exact score as a fraction num/den (cosine: dot^2 / |m|^2 for a fixed query; jaccard: |A∩B|/|A∪B|) */
void or_similarity(uint32_t metric, const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb,
                   uint64_t* num, uint64_t* den, double* value);
int or_select(or_state*, const uint32_t* q, uint32_t nq, uint32_t q_src, uint32_t* out);
uint32_t or_pmc(uint32_t k, const uint32_t* cur_tpl, const uint32_t* entry_tpl);
void or_table_put(or_state*, const uint32_t* ds, uint64_t stamp);
/* refine one DS against the current table (no commit): returns pmc; out final_ds, info[4], *target_stamp */
int or_refine_one(or_state*, const uint32_t* cur_ds, uint32_t* final_ds, int32_t* info, uint64_t* target_stamp);
void or_render(const or_state*, const uint32_t* ds, const uint32_t* q, uint32_t nq, uint32_t* out, uint32_t* len);
/* the splitmix64 finaliser the chain hash is built from (Z17); pinned to published splitmix64 outputs */
uint64_t or_mix64(uint64_t x);
void or_chain_hash(uint64_t hash_seed, const uint32_t* tok, uint32_t n, uint64_t* out /* [n/16] */);
/* kv_sim-style sequential lookup / insert, B = 1 semantics */
uint32_t or_lookup(or_state*, const uint32_t* tok, uint32_t n, uint32_t capped);
int or_insert(or_state*, const uint32_t* tok, uint32_t n);

/* fp64 causal attention for one request.
 * q [S][Hq][d] rows are absolute positions P..L-1 (S = L - P); k, v [L][Hkv][d];
 * out [S][Hq][d]; lse [S][Hq] (natural log) or NULL.  kv-head = h / (Hq/Hkv). */
void or_attention(uint32_t Hq, uint32_t Hkv, uint32_t d, uint32_t L, uint32_t P,
                  const double* q, const double* k, const double* v, double scale,
                  double* out, double* lse);

#ifdef __cplusplus
}
#endif
#endif
