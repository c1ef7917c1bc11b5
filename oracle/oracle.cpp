// oracle.cpp — TEST INFRASTRUCTURE, NOT THE PRODUCT (see oracle.h).
//
// A plain CPU implementation of the InferLog hot path, written from PAPER.md and the
// readings in SURVEY.md §8(c) / DESIGN.md.  Each function cites the passage it follows.
// No blocking, fusion or reordering beyond the definitions: std::map / std::vector,
// fp64 for attention, unsigned __int128 for exact score comparisons.  OpenMP is used only
// to run independent requests of a batch side by side (steps 1-6 are per-request pure
// functions of the snapshot); every state mutation (steps 7, 9, 10) is sequential in
// admission order.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <vector>

typedef uint64_t u64;
typedef uint32_t u32;
typedef unsigned __int128 u128;

static const u32 TOK_SEP = 1, TOK_TPL = 2;   // reserved ids (SURVEY c.1 / DESIGN.md)
static const u32 BS = 16;                     // KV block size in tokens

struct Demo {
  std::vector<u32> log, tpl;
  u32 template_id, src;
};

struct Block {            // a resident KV block
  u64 parent;             // chain hash of the previous block (ROOT for depth 0)
  u32 tok[BS];
  u32 depth;
  u64 stamp;              // LRU recency (b << 32 | admission index), reading Z21
};

struct or_state {
  u32 k, T, C, metric, flags;
  u32 decode = 0;                          // D: pages reserved for D decode tokens per request
  u64 seed;
  bool loaded = false;
  std::vector<Demo> pool;
  std::vector<u32> instr;
  std::map<std::vector<u32>, u64> table;   // ICL Table: DS tuple -> stamp (P:354 OrderedDict, Z2)
  std::map<u64, Block> index;              // prefix cache: chain hash -> resident block
  u64 batch = 0;                           // b of the last committed batch
  // data-parallel: replicated residency map, chain hash -> owner-rank bitmask, and
  // the box-level hit counts of the last batch
  std::map<u64, u32> box;
  std::vector<u32> last_box;
};

// ---------------------------------------------------------------------------------------
// a1  Similarity (LILAC = Jaccard over token sets, DivLog = cosine; SPEC S:127-135,
//     Z4-Z6).  Scores are exact fractions; never compared as floats.
// ---------------------------------------------------------------------------------------
struct Frac { u64 num, den; };

static Frac similarity(u32 metric, const std::vector<u32>& a, const std::vector<u32>& b) {
  std::map<u32, u64> ca, cb;                   // token -> count
  for (u32 t : a) ca[t] += 1;
  for (u32 t : b) cb[t] += 1;
  if (metric == OR_SIM_JACCARD) {
    if (ca.empty() && cb.empty()) return {1, 1};          // S:131 both empty -> 1
    u64 inter = 0;
    for (auto& kv : ca) if (cb.count(kv.first)) inter += 1;
    u64 uni = ca.size() + cb.size() - inter;
    return {inter, uni};                                  // one empty -> 0/|B| (Z5)
  }
  // cosine over token-count vectors: cos = dot / sqrt(|a|^2 |b|^2); held as cos^2 = num/den
  u64 dot = 0, na = 0, nb = 0;
  for (auto& kv : ca) {
    na += kv.second * kv.second;
    auto it = cb.find(kv.first);
    if (it != cb.end()) dot += kv.second * it->second;
  }
  for (auto& kv : cb) nb += kv.second * kv.second;
  if (na == 0 || nb == 0) return {0, 1};                  // zero norm -> 0 (Z5)
  return {dot * dot, na * nb};
}

// a > b as exact rationals (Z6)
static bool frac_gt(const Frac& a, const Frac& b) {
  return (u128)a.num * b.den > (u128)b.num * a.den;
}
static bool frac_eq(const Frac& a, const Frac& b) {
  return (u128)a.num * b.den == (u128)b.num * a.den;
}

// a2  Top-k in ascending-similarity order (Z7, Z8)
static int select_examples(const or_state* s, const std::vector<u32>& q, u32 q_src, u32* out) {
  struct C { Frac f; u32 idx; };
  std::vector<C> cand;
  for (u32 m = 0; m < s->pool.size(); ++m) {
    if ((s->flags & OR_F_EXCLUDE_SELF) && s->pool[m].src == q_src) continue;
    cand.push_back({similarity(s->metric, q, s->pool[m].log), m});
  }
  if (cand.size() < s->k) return 1;                       // "n > |candidates| -> argument error"
  // the k best by (score desc, index asc)
  std::stable_sort(cand.begin(), cand.end(), [](const C& x, const C& y) {
    if (!frac_eq(x.f, y.f)) return frac_gt(x.f, y.f);
    return x.idx < y.idx;
  });
  std::vector<C> top(cand.begin(), cand.begin() + s->k);
  // emitted ascending by similarity, ties by candidate index ascending
  std::stable_sort(top.begin(), top.end(), [](const C& x, const C& y) {
    if (!frac_eq(x.f, y.f)) return frac_gt(y.f, x.f);
    return x.idx < y.idx;
  });
  for (u32 j = 0; j < s->k; ++j) out[j] = top[j].idx;
  return 0;
}

// ---------------------------------------------------------------------------------------
// a3  PMC (fig:pair; Z11): the longest prefix of the entry whose
//     templates can be matched one-to-one against the current template multiset.
// ---------------------------------------------------------------------------------------
static u32 pmc(u32 k, const u32* cur_tpl, const u32* entry_tpl) {
  std::map<u32, int> avail;
  for (u32 j = 0; j < k; ++j) avail[cur_tpl[j]] += 1;
  u32 p = 0;
  for (u32 j = 0; j < k; ++j) {
    auto it = avail.find(entry_tpl[j]);
    if (it == avail.end() || it->second == 0) break;
    it->second -= 1;
    p += 1;
  }
  return p;
}

// ---------------------------------------------------------------------------------------
// a5  Render (fig:prompt; Z9):
//     prompt = I ++ (log ++ [TPL] ++ template ++ [SEP]) per demo ++ query log
// ---------------------------------------------------------------------------------------
static std::vector<u32> render(const or_state* s, const std::vector<u32>& ds, const std::vector<u32>& q) {
  std::vector<u32> p(s->instr);
  for (u32 d : ds) {
    const Demo& m = s->pool[d];
    p.insert(p.end(), m.log.begin(), m.log.end());
    p.push_back(TOK_TPL);
    p.insert(p.end(), m.tpl.begin(), m.tpl.end());
    p.push_back(TOK_SEP);
  }
  p.insert(p.end(), q.begin(), q.end());
  return p;
}

// ---------------------------------------------------------------------------------------
// a6  Chained block hash ("hash of (parent chain_hash, this block's token
//     ids)"; function fixed by reading Z17 — parity unpinned by the paper).
// ---------------------------------------------------------------------------------------
static u64 mix64(u64 x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}
static u64 root_hash(u64 seed) { return mix64(seed ^ 0x494E4645524C4F47ull); }
static u64 block_content(const u32* t) {
  u64 sum = 0;
  for (u32 i = 0; i < BS; ++i) sum += mix64(((u64)t[i] << 8) ^ (u64)i ^ 0x9E3779B97F4A7C15ull);
  return mix64(sum);
}
static u64 chain(u64 prev, u64 content) {
  u64 h = mix64(prev * 0x9E3779B97F4A7C15ull + content);
  if (h == 0) h = 1;                       // 0 is the EMPTY sentinel (Z18)
  if (h == ~0ull) h = ~0ull - 1;           // ~0 is the TOMBSTONE sentinel (Z18)
  return h;
}
static std::vector<u64> chain_hashes(u64 seed, const std::vector<u32>& tok) {
  std::vector<u64> H;
  u64 prev = root_hash(seed);
  for (size_t j = 0; j + BS <= tok.size(); j += BS) {
    prev = chain(prev, block_content(&tok[j]));
    H.push_back(prev);
  }
  return H;
}

// Longest run of leading blocks resident (and verified, Z19) in `index` (P:195-198,
// fig:prefixcache).  Matching is order dependent: the run stops at the
// first missing block even if later blocks are resident.
static u32 leading_hits(const or_state* s, const std::vector<u32>& tok, const std::vector<u64>& H) {
  u64 prev = root_hash(s->seed);
  u32 h = 0;
  for (u32 j = 0; j < H.size(); ++j) {
    auto it = s->index.find(H[j]);
    if (it == s->index.end()) break;
    if (s->flags & OR_F_VERIFY) {
      if (it->second.parent != prev) break;
      if (std::memcmp(it->second.tok, &tok[j * BS], BS * sizeof(u32)) != 0) break;
    }
    h += 1;
    prev = H[j];
  }
  return h;
}
// Z20: at least the last prompt token is always computed
static u32 cap_hits(u32 h, size_t L) {
  u32 cap = L == 0 ? 0 : (u32)((L - 1) / BS);
  return std::min(h, cap);
}

// ---------------------------------------------------------------------------------------
// One request's refinement against the table snapshot.
// ---------------------------------------------------------------------------------------
struct Refined {
  std::vector<u32> final_ds;
  int pmc = 0, rule = 2, reverted = 0, matched = 0;
  u64 target_stamp = 0;
};

static Refined refine(const or_state* s, const std::vector<u32>& cur, const std::vector<u32>& q) {
  Refined r;
  r.final_ds = cur;
  if (!(s->flags & OR_F_PAIR)) return r;              // naive PC: unchanged
  const u32 k = s->k;
  std::vector<u32> cur_tpl(k);
  for (u32 j = 0; j < k; ++j) cur_tpl[j] = s->pool[cur[j]].template_id;
  // match_target: max PMC, ties -> most recently used (Z12)
  const std::vector<u32>* best = nullptr;
  u32 best_p = 0;
  u64 best_stamp = 0;
  for (auto& e : s->table) {
    std::vector<u32> et(k);
    for (u32 j = 0; j < k; ++j) et[j] = s->pool[e.first[j]].template_id;
    u32 p = pmc(k, cur_tpl.data(), et.data());
    if (p > best_p || (p == best_p && p > 0 && e.second > best_stamp)) {
      best = &e.first; best_p = p; best_stamp = e.second;
    }
  }
  if (best == nullptr || best_p == 0) return r;        // rule 2: PMC = 0
  r.pmc = (int)best_p; r.matched = 1; r.target_stamp = best_stamp;
  if (best_p == k) {                                    // rule 1
    r.rule = 1;
    r.final_ds = *best;
  } else {                                              // rule 3: modify + reorder
    r.rule = 3;
    std::vector<bool> replaced(k, false);
    std::vector<u32> out;
    for (u32 j = 0; j < best_p; ++j) {
      u32 t = s->pool[(*best)[j]].template_id;
      u32 q_pos = k;
      for (u32 qq = 0; qq < k; ++qq)                    // first unreplaced occurrence (Z13)
        if (!replaced[qq] && cur_tpl[qq] == t) { q_pos = qq; break; }
      if (q_pos == k) { r.rule = -1; return r; }        // "internal error": cannot happen
      replaced[q_pos] = true;
      out.push_back((*best)[j]);                        // the target's demo, verbatim
    }
    for (u32 qq = 0; qq < k; ++qq)
      if (!replaced[qq]) out.push_back(cur[qq]);        // the rest keep their order
    r.final_ds = out;
  }
  if (s->flags & OR_F_GUARD) {                          // never-worse guard (Z25; not in the paper)
    std::vector<u32> pf = render(s, r.final_ds, q), pc = render(s, cur, q);
    u32 hf = cap_hits(leading_hits(s, pf, chain_hashes(s->seed, pf)), pf.size());
    u32 hc = cap_hits(leading_hits(s, pc, chain_hashes(s->seed, pc)), pc.size());
    if (hf < hc) { r.final_ds = cur; r.reverted = 1; }
  }
  return r;
}

static u64 stamp_of(u64 b, u32 i) { return (b << 32) | (u64)i; }

// =======================================================================================
extern "C" {

or_state* or_create(u32 k, u32 T, u32 C, u32 metric, u32 flags, u64 hash_seed) {
  or_state* s = new or_state();
  s->k = k; s->T = T; s->C = C; s->metric = metric; s->flags = flags; s->seed = hash_seed;
  return s;
}
void or_destroy(or_state* s) { delete s; }

int or_pool_load(or_state* s, u32 n, const u32* log_off, const u32* log_tok, const u32* tpl_off,
                 const u32* tpl_tok, const u32* template_id, const u32* src_index,
                 const u32* instr, u32 n_instr) {
  if (s->k == 0 || n < s->k) return 1;
  s->pool.assign(n, Demo());
  for (u32 m = 0; m < n; ++m) {
    s->pool[m].log.assign(log_tok + log_off[m], log_tok + log_off[m + 1]);
    s->pool[m].tpl.assign(tpl_tok + tpl_off[m], tpl_tok + tpl_off[m + 1]);
    s->pool[m].template_id = template_id[m];
    s->pool[m].src = src_index[m];
  }
  s->instr.assign(instr, instr + n_instr);
  s->table.clear();                                  // demo ids change: reset (il.h pool_load)
  s->index.clear();
  s->box.clear();
  s->last_box.clear();
  s->batch = 0;
  s->loaded = true;
  return 0;
}

// The batch procedure over G data-parallel ranks; G = 1 is the one-GPU
// procedure.  Rank r owns the contiguous admission slice [r*B/G, (r+1)*B/G) of the global batch
// and its own prefix index st[r]->index (steps 6, 7, 9 use only that index); the ICL Table is
// replicated: every st[r]->table starts identical and step 10 applies ALL B records in global
// admission order to each of them.  Stamps use the global admission index i.
static int run_batch_dp(or_state** st, u32 G, u32 B, const u32* q_off, const u32* q_tok, const u32* q_src,
                        u32* topk, u32* final_ds, int32_t* info, u64* target_stamp, u32* prompt_len,
                        u32* prompt_tok, u32 prompt_stride, u64* block_hash, u32 max_blocks, u32* hit,
                        u64* evicted, u32* n_evicted, u32* n_evicted_rank) {
  for (u32 r = 0; r < G; ++r) {
    if (!st[r]->loaded) return 3;
    if (st[r]->batch != st[0]->batch || st[r]->table != st[0]->table) return 4;   // not replicated
  }
  const u32 k = st[0]->k;
  const u64 b = st[0]->batch + 1;
  std::vector<u32> owner(B);
  for (u32 r = 0; r < G; ++r)
    for (u32 i = (u32)((u64)r * B / G); i < (u32)((u64)(r + 1) * B / G); ++i) owner[i] = r;
  std::vector<std::vector<u32>> q(B), cur(B), prompt(B);
  std::vector<std::vector<u64>> H(B);
  std::vector<Refined> ref(B);
  std::vector<u32> h(B), boxh(B);
  std::vector<int> err(B, 0);

  // Steps 1-6 per request against the snapshot (Z1) of its rank.
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t ii = 0; ii < (int64_t)B; ++ii) {
    const u32 i = (u32)ii;
    const or_state* s = st[owner[i]];
    q[i].assign(q_tok + q_off[i], q_tok + q_off[i + 1]);
    cur[i].assign(k, 0);
    if (select_examples(s, q[i], q_src[i], cur[i].data())) { err[i] = 1; continue; }
    ref[i] = refine(s, cur[i], q[i]);
    if (ref[i].rule < 0) { err[i] = 4; continue; }
    prompt[i] = render(s, ref[i].final_ds, q[i]);
    if (prompt[i].size() + s->decode > prompt_stride || prompt[i].size() / BS > max_blocks) { err[i] = 1; continue; }
    H[i] = chain_hashes(s->seed, prompt[i]);
    const u32 hl = leading_hits(s, prompt[i], H[i]);
    h[i] = cap_hits(hl, prompt[i].size());
    // box-level hits: the rank's own leading run, continued through blocks the residency map
    // (the union of every rank's index at the snapshot) holds; hash only, capped as Z20
    u32 hb = hl;
    while (hb < H[i].size()) {
      auto it = s->box.find(H[i][hb]);
      if (it == s->box.end() || it->second == 0) break;
      hb += 1;
    }
    boxh[i] = cap_hits(hb, prompt[i].size());
  }
  for (u32 i = 0; i < B; ++i) if (err[i]) return err[i];

  // NEXT-1 in-batch dedup (OR_F_DEDUP; Z22b): a block that an earlier request of the
  // same rank computes in this batch (a full block at its position >= its own hit count h) is
  // not computed again.  Owner of a hash = the lowest admission index presenting it that way (and
  // its depth); request i's leading run continues from its hit count h_i through blocks whose
  // owner is an earlier request at the same depth with equal block tokens, capped as Z20.  The
  // run's pages are the owner's; only the snapshot hits [0, h_i) are touched and pinned.
  std::vector<u32> hloc = h;
  if (st[0]->flags & OR_F_DEDUP) {
    for (u32 r = 0; r < G; ++r) {
      std::map<u64, std::pair<u32, u32>> own;           // hash -> (first request, depth)
      for (u32 i = 0; i < B; ++i) {
        if (owner[i] != r) continue;
        for (u32 j = hloc[i]; j < H[i].size(); ++j) own.emplace(H[i][j], std::make_pair(i, j));
      }
      for (u32 i = 0; i < B; ++i) {
        if (owner[i] != r) continue;
        const u32 cap = cap_hits((u32)H[i].size(), prompt[i].size());
        u32 he = hloc[i];
        while (he < cap) {
          auto it = own.find(H[i][he]);
          if (it == own.end() || it->second.first >= i || it->second.second != he) break;
          const u32 o = it->second.first;
          if (!std::equal(&prompt[o][he * BS], &prompt[o][he * BS] + BS, &prompt[i][he * BS])) break;
          he += 1;
        }
        h[i] = he;
        boxh[i] = std::max(boxh[i], he);
      }
    }
  }

  // Step 7 per rank: touch + pin the hit blocks, then evict for the pages its slice needs (Z21).
  std::vector<std::vector<u64>> victims(G);
  for (u32 r = 0; r < G; ++r) {
    or_state* s = st[r];
    std::set<u64> pinned;
    u64 need = 0;
    for (u32 i = 0; i < B; ++i) {
      if (owner[i] != r) continue;
      for (u32 j = 0; j < hloc[i]; ++j) pinned.insert(H[i][j]);
      need += (prompt[i].size() + s->decode + BS - 1) / BS - h[i];   // (+ the decode reserve)
    }
    u64 free_pages = s->C - s->index.size();
    if (need > free_pages) {
      struct V { u64 stamp; u32 depth; u64 hash; };
      std::vector<V> cand;
      for (auto& e : s->index)
        if (!pinned.count(e.first)) cand.push_back({e.second.stamp, e.second.depth, e.first});
      if (cand.size() < need - free_pages) return 2;  // IL_ERR_CAPACITY, state untouched
      std::sort(cand.begin(), cand.end(), [](const V& x, const V& y) {
        if (x.stamp != y.stamp) return x.stamp < y.stamp;   // least recently used first
        if (x.depth != y.depth) return x.depth > y.depth;   // deeper first (keeps ancestors)
        return x.hash < y.hash;
      });
      for (u64 e = 0; e < need - free_pages; ++e) victims[r].push_back(cand[e].hash);
    }
  }
  size_t n_vict = 0;
  for (u32 r = 0; r < G; ++r) n_vict += victims[r].size();
  if (n_vict > *n_evicted) return 1;
  // index stamps use the admission index within the rank's slice (its LRU order); table stamps
  // (step 10) use the global admission index
  std::vector<u32> lo(G + 1);
  for (u32 r = 0; r <= G; ++r) lo[r] = (u32)((u64)r * B / G);
  for (u32 i = 0; i < B; ++i)
    for (u32 j = 0; j < hloc[i]; ++j) st[owner[i]]->index[H[i][j]].stamp = stamp_of(b, i - lo[owner[i]]);
  for (u32 r = 0; r < G; ++r)
    for (u64 v : victims[r]) st[r]->index.erase(v);

  // Step 9: insert the new full blocks in admission order, each into its rank's index; first
  // wins (Z22).  The blocks a rank's index gains or loses are its block records (§8(e)).
  std::vector<std::vector<u64>> gained(G);
  for (u32 i = 0; i < B; ++i) {
    or_state* s = st[owner[i]];
    const u32 il = i - lo[owner[i]];
    for (u32 j = h[i]; j < H[i].size(); ++j) {
      auto it = s->index.find(H[i][j]);
      if (it != s->index.end()) {
        it->second.stamp = std::max(it->second.stamp, stamp_of(b, il));
      } else {
        Block blk;
        blk.parent = j == 0 ? root_hash(s->seed) : H[i][j - 1];
        std::memcpy(blk.tok, &prompt[i][j * BS], sizeof(blk.tok));
        blk.depth = j;
        blk.stamp = stamp_of(b, il);
        s->index[H[i][j]] = blk;
        gained[owner[i]].push_back(H[i][j]);
      }
    }
  }
  // The residency map (replicated on every rank): each rank's lost and gained blocks toggle its
  // owner bit, so the map is the union of the ranks' indices with their owner sets.
  for (u32 r = 0; r < G; ++r) {
    for (u32 q = 0; q < G; ++q) {
      auto& bx = st[q]->box;
      for (const auto* lst : {&victims[r], &gained[r]})
        for (u64 x : *lst) {
          u32& m = bx[x];
          m ^= 1u << r;
          if (m == 0) bx.erase(x);
        }
    }
  }
  for (u32 r = 0; r < G; ++r) st[r]->last_box = boxh;

  // Step 10: ICL Table commit (Z2, Z3, Z14), all B records on every rank.  Rule 1
  // refreshes the target (its key IS final_ds); rules 2/3 and reverted requests upsert
  // final_ds; a rule-3 target keeps its position.  Then keep the T most recent entries.
  for (u32 r = 0; r < G; ++r) {
    or_state* s = st[r];
    if (s->flags & OR_F_PAIR) {
      for (u32 i = 0; i < B; ++i) {
        auto it = s->table.find(ref[i].final_ds);
        if (it == s->table.end()) s->table[ref[i].final_ds] = stamp_of(b, i);
        else it->second = std::max(it->second, stamp_of(b, i));
      }
      while (s->table.size() > s->T) {
        auto oldest = s->table.begin();
        for (auto it = s->table.begin(); it != s->table.end(); ++it)
          if (it->second < oldest->second) oldest = it;
        s->table.erase(oldest);
      }
    }
    s->batch = b;
  }

  // outputs
  for (u32 i = 0; i < B; ++i) {
    for (u32 j = 0; j < k; ++j) { topk[i * k + j] = cur[i][j]; final_ds[i * k + j] = ref[i].final_ds[j]; }
    info[i * 4 + 0] = ref[i].pmc; info[i * 4 + 1] = ref[i].rule;
    info[i * 4 + 2] = ref[i].reverted; info[i * 4 + 3] = ref[i].matched;
    target_stamp[i] = ref[i].target_stamp;
    prompt_len[i] = (u32)prompt[i].size();
    std::memcpy(prompt_tok + (size_t)i * prompt_stride, prompt[i].data(), prompt[i].size() * sizeof(u32));
    for (u32 j = 0; j < H[i].size(); ++j) block_hash[(size_t)i * max_blocks + j] = H[i][j];
    hit[i] = h[i];
  }
  size_t e = 0;
  for (u32 r = 0; r < G; ++r) {
    for (u64 v : victims[r]) evicted[e++] = v;
    if (n_evicted_rank) n_evicted_rank[r] = (u32)victims[r].size();
  }
  *n_evicted = (u32)n_vict;
  return 0;
}

int or_run_batch(or_state* s, u32 B, const u32* q_off, const u32* q_tok, const u32* q_src,
                 u32* topk, u32* final_ds, int32_t* info, u64* target_stamp, u32* prompt_len,
                 u32* prompt_tok, u32 prompt_stride, u64* block_hash, u32 max_blocks, u32* hit,
                 u64* evicted, u32* n_evicted) {
  return run_batch_dp(&s, 1, B, q_off, q_tok, q_src, topk, final_ds, info, target_stamp, prompt_len, prompt_tok,
                      prompt_stride, block_hash, max_blocks, hit, evicted, n_evicted, nullptr);
}

int or_run_batch_dp(or_state** st, u32 G, u32 B, const u32* q_off, const u32* q_tok, const u32* q_src,
                    u32* topk, u32* final_ds, int32_t* info, u64* target_stamp, u32* prompt_len,
                    u32* prompt_tok, u32 prompt_stride, u64* block_hash, u32 max_blocks, u32* hit,
                    u64* evicted, u32* n_evicted, u32* n_evicted_rank) {
  if (G == 0) return 1;
  return run_batch_dp(st, G, B, q_off, q_tok, q_src, topk, final_ds, info, target_stamp, prompt_len, prompt_tok,
                      prompt_stride, block_hash, max_blocks, hit, evicted, n_evicted, n_evicted_rank);
}

u64 or_batch_index(const or_state* s) { return s->batch; }
void or_set_decode(or_state* s, u32 d) { s->decode = d; }
u32 or_index_size(const or_state* s) { return (u32)s->index.size(); }
void or_index_dump(const or_state* s, u64* hash, u64* stamp, u32* depth, u64* parent) {
  size_t n = 0;
  for (auto& e : s->index) {
    hash[n] = e.first; stamp[n] = e.second.stamp; depth[n] = e.second.depth; parent[n] = e.second.parent;
    ++n;
  }
}
u32 or_table_size(const or_state* s) { return (u32)s->table.size(); }
void or_box_hits(const or_state* s, u32* out) {
  for (size_t i = 0; i < s->last_box.size(); ++i) out[i] = s->last_box[i];
}
u32 or_box_map_size(const or_state* s) { return (u32)s->box.size(); }
void or_box_map_dump(const or_state* s, u64* hash, u32* mask) {
  size_t n = 0;
  for (auto& e : s->box) { hash[n] = e.first; mask[n] = e.second; ++n; }
}
void or_table_dump(const or_state* s, u32* ds, u64* stamp) {
  std::vector<std::pair<u64, const std::vector<u32>*>> v;
  for (auto& e : s->table) v.push_back({e.second, &e.first});
  std::sort(v.begin(), v.end());
  for (size_t n = 0; n < v.size(); ++n) {
    stamp[n] = v[n].first;
    for (u32 j = 0; j < s->k; ++j) ds[n * s->k + j] = (*v[n].second)[j];
  }
}

void or_similarity(u32 metric, const u32* a, u32 na, const u32* b, u32 nb, u64* num, u64* den, double* value) {
  std::vector<u32> va(a, a + na), vb(b, b + nb);
  Frac f = similarity(metric, va, vb);
  *num = f.num; *den = f.den;
  *value = metric == OR_SIM_JACCARD ? (double)f.num / (double)f.den
                                    : std::sqrt((double)f.num / (double)f.den);
}

int or_select(or_state* s, const u32* q, u32 nq, u32 q_src, u32* out) {
  std::vector<u32> vq(q, q + nq);
  return select_examples(s, vq, q_src, out);
}

u32 or_pmc(u32 k, const u32* cur_tpl, const u32* entry_tpl) { return pmc(k, cur_tpl, entry_tpl); }

void or_table_put(or_state* s, const u32* ds, u64 stamp) {
  s->table[std::vector<u32>(ds, ds + s->k)] = stamp;
}

int or_refine_one(or_state* s, const u32* cur_ds, u32* final_ds, int32_t* info, u64* target_stamp) {
  std::vector<u32> cur(cur_ds, cur_ds + s->k), q;
  Refined r = refine(s, cur, q);
  for (u32 j = 0; j < s->k; ++j) final_ds[j] = r.final_ds[j];
  info[0] = r.pmc; info[1] = r.rule; info[2] = r.reverted; info[3] = r.matched;
  *target_stamp = r.target_stamp;
  return r.pmc;
}

void or_render(const or_state* s, const u32* ds, const u32* q, u32 nq, u32* out, u32* len) {
  std::vector<u32> vds(ds, ds + s->k), vq(q, q + nq);
  std::vector<u32> p = render(s, vds, vq);
  std::memcpy(out, p.data(), p.size() * sizeof(u32));
  *len = (u32)p.size();
}

u64 or_mix64(u64 x) { return mix64(x); }

void or_chain_hash(u64 seed, const u32* tok, u32 n, u64* out) {
  std::vector<u32> v(tok, tok + n);
  std::vector<u64> H = chain_hashes(seed, v);
  for (size_t j = 0; j < H.size(); ++j) out[j] = H[j];
}

// kv_sim lookup: longest resident chain; hit blocks refresh recency.
u32 or_lookup(or_state* s, const u32* tok, u32 n, u32 capped) {
  std::vector<u32> v(tok, tok + n);
  std::vector<u64> H = chain_hashes(s->seed, v);
  u32 h = leading_hits(s, v, H);
  s->batch += 1;
  for (u32 j = 0; j < h; ++j) s->index[H[j]].stamp = stamp_of(s->batch, 0);
  return capped ? cap_hits(h, n) : h;
}

// kv_sim insert: all full blocks become resident (dedup by chain hash);
// evict LRU blocks as needed, never the sequence's own; if the sequence alone has more
// full blocks than the capacity, insert only the first C.
int or_insert(or_state* s, const u32* tok, u32 n) {
  std::vector<u32> v(tok, tok + n);
  std::vector<u64> H = chain_hashes(s->seed, v);
  if (H.size() > s->C) H.resize(s->C);
  std::set<u64> own(H.begin(), H.end());
  u64 need = 0;
  for (u64 x : H) if (!s->index.count(x)) need += 1;
  u64 free_pages = s->C - s->index.size();
  if (need > free_pages) {
    struct V { u64 stamp; u32 depth; u64 hash; };
    std::vector<V> cand;
    for (auto& e : s->index) if (!own.count(e.first)) cand.push_back({e.second.stamp, e.second.depth, e.first});
    std::sort(cand.begin(), cand.end(), [](const V& x, const V& y) {
      if (x.stamp != y.stamp) return x.stamp < y.stamp;
      if (x.depth != y.depth) return x.depth > y.depth;
      return x.hash < y.hash;
    });
    for (u64 e = 0; e < need - free_pages && e < cand.size(); ++e) s->index.erase(cand[e].hash);
  }
  s->batch += 1;
  for (u32 j = 0; j < H.size(); ++j) {
    Block blk;
    blk.parent = j == 0 ? root_hash(s->seed) : H[j - 1];
    std::memcpy(blk.tok, &v[j * BS], sizeof(blk.tok));
    blk.depth = j;
    blk.stamp = stamp_of(s->batch, 0);
    s->index[H[j]] = blk;
  }
  return 0;
}

// a8  Prefill attention over cached prefix + causal suffix, fp64 (SURVEY c.2
//     step 8; Z26: scale given, causal over absolute positions, GQA kv head = h / g).
void or_attention(u32 Hq, u32 Hkv, u32 d, u32 L, u32 P, const double* q, const double* k,
                  const double* v, double scale, double* out, double* lse) {
  const u32 S = L - P, g = Hq / Hkv;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t si = 0; si < (int64_t)S; ++si) {
    for (int64_t hh = 0; hh < (int64_t)Hq; ++hh) {
      const u32 s = (u32)si, h = (u32)hh, p = P + s, kh = h / g;
      const double* qv = q + ((size_t)s * Hq + h) * d;
      std::vector<double> logit(p + 1);
      double mx = -INFINITY;
      for (u32 j = 0; j <= p; ++j) {
        const double* kv = k + ((size_t)j * Hkv + kh) * d;
        double dot = 0;
        for (u32 c = 0; c < d; ++c) dot += qv[c] * kv[c];
        logit[j] = dot * scale;
        mx = std::max(mx, logit[j]);
      }
      double denom = 0;
      for (u32 j = 0; j <= p; ++j) { logit[j] = std::exp(logit[j] - mx); denom += logit[j]; }
      double* o = out + ((size_t)s * Hq + h) * d;
      for (u32 c = 0; c < d; ++c) o[c] = 0;
      for (u32 j = 0; j <= p; ++j) {
        const double w = logit[j] / denom;
        const double* vv = v + ((size_t)j * Hkv + kh) * d;
        for (u32 c = 0; c < d; ++c) o[c] += w * vv[c];
      }
      if (lse) lse[(size_t)s * Hq + h] = mx + std::log(denom);
    }
  }
}

}  // extern "C"
