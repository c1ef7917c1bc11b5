// refine.cu — il_refine_batch: K1 exact similarity + top-k, K2/K3 PAIR (PMC, modify,
// reorder, rules, guard) + prompt render.
#include "il_internal.cuh"
#include "match_dev.cuh"
#include "sim_dev.cuh"

namespace il {

// ---------------------------------------------------------------------------------------
// K1  Similarity + top-k (Z4-Z8).
// One CTA per query.  The query's token multiset goes into a shared-memory hash table;
// every thread scores a strided subset of the pool by streaming each demo's sorted unique
// tokens (+ counts) and probing the table, keeping a private top-k.  Scores are exact
// fractions compared by cross-multiplication:
//   cosine : cos^2 * |q|^2 = dot^2 / |m|^2  (|q|^2 is common to one query)
//   jaccard: |A n B| / |A u B|
// Selection is by (score desc, index asc); the k winners are emitted (score asc, index asc).
// ---------------------------------------------------------------------------------------
constexpr int SIM_THREADS = 128;               // 4 warps = 4 queries per CTA
constexpr int QHASH = 512;

__device__ __forceinline__ uint32_t qslot(uint32_t t) { return (t * 0x9E3779B1u) >> (32 - 9); }

// QW warps per query (the CTA's 4 warps serve 4 / QW queries): QW = 1 for pools up to
// SIM_BIG_POOL demos (no block-wide rounds, most queries per SM), QW = 4 above (4x the lanes per
// query when the scoring loop dominates).
#ifndef IL_SIM_QW_SMALL
#define IL_SIM_QW_SMALL 2
#endif
template <int QW>
__global__ void __launch_bounds__(SIM_THREADS) k_sim_topk(Ctx c, uint32_t B, const uint32_t* __restrict__ q_off,
                                                          const uint32_t* __restrict__ q_tok,
                                                          const uint32_t* __restrict__ q_src,
                                                          uint32_t* __restrict__ topk) {
  // the query multiset goes into the query's shared-memory hash table, the query's lanes score
  // a strided subset of the pool
  constexpr uint32_t NW = SIM_THREADS / 32, NQ = NW / QW, GT = QW * 32;
  __shared__ uint32_t s_key_all[NQ][QHASH], s_cnt_all[NQ][QHASH];
  __shared__ uint64_t s_lnum[MAXK][SIM_THREADS];
  __shared__ uint32_t s_lden[MAXK][SIM_THREADS], s_lidx[MAXK][SIM_THREADS];
  __shared__ Cand s_wl[NW][MAXK];
  __shared__ uint32_t s_wn[NW], s_red[NW][2];
  __shared__ Cand s_sel_all[NQ][MAXK];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t grp = wid / QW, sub = wid % QW, gt = sub * 32 + lane;
  const uint32_t i = blockIdx.x * NQ + grp;
  bool live = i < B;                                    // (every warp still takes the barriers)
  uint32_t* s_key = s_key_all[grp];
  uint32_t* s_cnt = s_cnt_all[grp];
  Cand* s_sel = s_sel_all[grp];
  const uint32_t k = c.cfg.k;
  for (uint32_t x = gt; x < QHASH; x += GT) { s_key[x] = NONE32; s_cnt[x] = 0; }
  __syncthreads();
  uint32_t qa = 0, qL = 0;
  if (live) {
    qa = q_off[i]; qL = q_off[i + 1] - qa;
    if (qL > c.cfg.max_log_tokens) {
      if (gt == 0) latch(c.sc, IL_ERR_ARG);
      live = false; qL = 0;
    }
  }
  for (uint32_t x = gt; x < qL; x += GT) {
    const uint32_t t = q_tok[qa + x];
    uint32_t s = qslot(t);
    while (true) {
      const uint32_t old = atomicCAS(&s_key[s], NONE32, t);
      if (old == NONE32 || old == t) break;
      s = (s + 1) & (QHASH - 1);
    }
    atomicAdd(&s_cnt[s], 1u);
  }
  __syncthreads();
  uint32_t nq = 0, nuq = 0;
  for (uint32_t x = gt; x < QHASH; x += GT)
    if (s_key[x] != NONE32) { nq += s_cnt[x] * s_cnt[x]; nuq += 1; }
  for (int o = 16; o; o >>= 1) { nq += __shfl_xor_sync(~0u, nq, o); nuq += __shfl_xor_sync(~0u, nuq, o); }
  if (QW > 1) {
    if (lane == 0) { s_red[wid][0] = nq; s_red[wid][1] = nuq; }
    __syncthreads();
    nq = nuq = 0;
    for (uint32_t q = 0; q < QW; ++q) { nq += s_red[grp * QW + q][0]; nuq += s_red[grp * QW + q][1]; }
  }
  const bool jac = c.cfg.metric == IL_SIM_JACCARD;
  const bool excl = (c.cfg.flags & IL_F_EXCLUDE_SELF) != 0;
  const uint32_t my_src = (live && excl && q_src) ? q_src[i] : NONE32;

  // private sorted list, always MAXK long: padded with a sentinel every real candidate beats
  Cand top[MAXK];
#pragma unroll
  for (int q = 0; q < MAXK; ++q) { top[q].num = 0; top[q].den = 1; top[q].idx = NONE32; }
  uint32_t ntop = 0;
  for (uint32_t m = gt; m < (live ? c.n_demos : 0u); m += GT) {
    if (excl && c.src[m] == my_src) continue;
    const uint32_t a = c.log_off[m], nu = c.uniq_n[m];
    uint32_t dot = 0, inter = 0;
    // 8 tokens (+ counts) are loaded before any is probed: the loop is L2-latency bound
    for (uint32_t u0 = 0; u0 < nu; u0 += 8) {
      uint32_t tk[8], ct[8];
#pragma unroll
      for (uint32_t e = 0; e < 8; ++e) {
        const bool in = u0 + e < nu;
        tk[e] = in ? c.uniq_tok[a + u0 + e] : NONE32;
        ct[e] = in ? c.uniq_cnt[a + u0 + e] : 0u;
      }
#pragma unroll
      for (uint32_t e = 0; e < 8; ++e) {
        const uint32_t t = tk[e];
        uint32_t s = qslot(t), cq = 0;
        while (t != NONE32) {
          const uint32_t key = s_key[s];
          if (key == t) { cq = s_cnt[s]; break; }
          if (key == NONE32) break;
          s = (s + 1) & (QHASH - 1);
        }
        dot += cq * ct[e];
        inter += cq != 0;
      }
    }
    Cand x;
    x.idx = m;
    if (jac) {
      if (nuq == 0 && nu == 0) { x.num = 1; x.den = 1; }
      else { x.num = inter; x.den = nuq + nu - inter; }
    } else {
      const uint32_t nm = c.norm2[m];
      if (nq == 0 || nm == 0) { x.num = 0; x.den = 1; }                   // zero norm (Z5)
      else { x.num = (uint64_t)dot * dot; x.den = nm; }
    }
    // insert into the private sorted list: position q takes x if x ranks before its old
    // entry, else keeps it; entries below shift down one (static register indices only)
    Cand prev = top[0];
    bool bprev = better(x, prev);
    if (bprev) top[0] = x;
#pragma unroll
    for (int q = 1; q < MAXK; ++q) {
      const Cand cur = top[q];
      const bool bq = better(x, cur);
      if (bq) top[q] = bprev ? prev : x;
      prev = cur;
      bprev = bq;
    }
    ntop = min(ntop + 1, (uint32_t)MAXK);
  }
  ntop = min(ntop, k);
  // merge: the lanes' sorted lists go to shared memory (static register indices), k rounds of
  // warp argmax per warp (the winning lane pops its head), then (QW > 1) the query's first warp
  // merges its QW warp lists the same way
#pragma unroll
  for (int q = 0; q < MAXK; ++q)
    if ((uint32_t)q < ntop) { s_lnum[q][tid] = top[q].num; s_lden[q][tid] = (uint32_t)top[q].den; s_lidx[q][tid] = top[q].idx; }
  __syncwarp();
  uint32_t nsel = warp_merge([&](uint32_t q) { Cand x; x.num = s_lnum[q][tid]; x.den = s_lden[q][tid]; x.idx = s_lidx[q][tid]; return x; },
                             ntop, k, lane, QW == 1 ? s_sel : s_wl[wid]);
  if (QW > 1) {
    if (lane == 0) s_wn[wid] = nsel;
    __syncthreads();
    if (sub != 0) return;
    const uint32_t wn = lane < QW ? s_wn[grp * QW + lane] : 0u;
    nsel = warp_merge([&](uint32_t q) { return s_wl[grp * QW + lane][q]; }, wn, k, lane, s_sel);
  }
  __syncwarp();
  if (!live) return;
  if (nsel < k) {
    if (lane == 0) latch(c.sc, IL_ERR_ARG);             // fewer than k candidates
    return;
  }
  if (lane < k) {
    // emit ascending by similarity, ties by index ascending: position = rank
    const Cand me = s_sel[lane];
    uint32_t pos = 0;
    for (uint32_t r = 0; r < k; ++r) {
      const Cand o = s_sel[r];
      const uint64_t l = o.num * me.den, rr = me.num * o.den;
      pos += (l < rr || (l == rr && o.idx < me.idx)) ? 1u : 0u;
    }
    topk[(size_t)i * k + pos] = me.idx;
  }
}

// ---------------------------------------------------------------------------------------
// K2/K3  PAIR against the ICL-Table snapshot + render.  One warp per request.
//  PMC (Z11): greedy multiset-feasible prefix; lanes scan table slots, warp argmax
//  of (pmc, stamp).  Rules: 1 -> target verbatim; 2 -> unchanged;
//  3 -> the target's first pmc demos replace the first unreplaced same-template current
//  demos (Z13) and go first, the rest keep their order.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void render_row(const Ctx& c, const uint32_t* ds, uint32_t k,
                                           const uint32_t* __restrict__ q, uint32_t qL,
                                           uint32_t* __restrict__ out, uint32_t lane) {
  uint32_t o = c.n_instr;
  for (uint32_t x = lane; x < c.n_instr; x += 32) out[x] = c.instr[x];
  for (uint32_t j = 0; j < k; ++j) {
    const uint32_t d = ds[j], a = c.rend_off[d], n = c.rend_len[d];
    for (uint32_t x = lane; x < n; x += 32) out[o + x] = c.rend_tok[a + x];
    o += n;
  }
  for (uint32_t x = lane; x < qL; x += 32) out[o + x] = q[x];
}

// One CTA (128 threads) per request: threads scan table slots (SoA template rows: coalesced),
// block argmax of (pmc, stamp), thread 0 applies the rules, all threads render, warp 0 runs
// the guard's two hash-match passes.
constexpr int REF_THREADS = 128;

__global__ void __launch_bounds__(REF_THREADS) k_refine(Ctx c, uint32_t B, const uint32_t* __restrict__ q_off,
                                                        const uint32_t* __restrict__ q_tok,
                                                        const uint32_t* __restrict__ topk,
                                                        uint32_t* __restrict__ final_ds, il_refine_info* __restrict__ info,
                                                        uint32_t* __restrict__ prompt_tok,
                                                        uint32_t* __restrict__ prompt_len) {
  __shared__ uint32_t s_cur[MAXK], s_fin[MAXK];
  __shared__ uint32_t s_bp[REF_THREADS / 32], s_bs[REF_THREADS / 32];
  __shared__ uint64_t s_bst[REF_THREADS / 32];
  __shared__ il_refine_info s_inf;
  __shared__ uint32_t s_L, s_rendered;
  const uint32_t i = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t k = c.cfg.k, T = c.cfg.table_capacity;
  if (tid < k) s_cur[tid] = topk[(size_t)i * k + tid];
  __syncthreads();
  uint32_t cur[MAXK], tc[MAXK];
#pragma unroll
  for (int j = 0; j < MAXK; ++j) {
    cur[j] = (uint32_t)j < k ? s_cur[j] : 0;
    tc[j] = (uint32_t)j < k ? c.tid[cur[j]] : NONE32;
  }
  uint32_t bp = 0, bs = NONE32;
  uint64_t bst = 0;
  if (c.cfg.flags & IL_F_PAIR) {
    // SCAN slots per thread per round, every stamp and template id loaded before any is used
    // (the scan is L2-latency bound: keep the loads in flight together)
    // PMC >= 1 needs the entry's first template in the request's multiset: each round loads
    // SCAN slots' stamps and first templates together (the scan is L2-latency bound), and only
    // entries passing that test load the rest of their templates
    constexpr uint32_t SCAN = 8;
    for (uint32_t s0 = tid; s0 < T; s0 += SCAN * REF_THREADS) {
      uint64_t st[SCAN];
      uint32_t t0[SCAN];
#pragma unroll
      for (uint32_t u = 0; u < SCAN; ++u) {
        const uint32_t s = s0 + u * REF_THREADS;
        st[u] = s < T ? c.tab_stamp[s] : 0ull;
        t0[u] = s < T ? c.tab_tpl[s] : NONE32;
      }
#pragma unroll
      for (uint32_t u = 0; u < SCAN; ++u) {
        bool any = false;
#pragma unroll
        for (int q = 0; q < MAXK; ++q) any |= tc[q] == t0[u];
        if (st[u] == 0 || !any) continue;              // PMC = 0: never selected
        const uint32_t s = s0 + u * REF_THREADS;
        uint32_t used = 0, p = 0;
        bool run = true;
#pragma unroll
        for (uint32_t j = 0; j < MAXK; ++j) {
          if (run && j < k) {                          // (predicated: the loop stays unrolled)
            const uint32_t tj = j == 0 ? t0[u] : c.tab_tpl[(size_t)j * T + s];
            bool found = false;
#pragma unroll
            for (int q = 0; q < MAXK; ++q) {
              if (!found && !((used >> q) & 1u) && tc[q] == tj) { used |= 1u << q; found = true; }
            }
            if (!found) run = false; else ++p;
          }
        }
        if (p > bp || (p == bp && p > 0 && st[u] > bst)) { bp = p; bst = st[u]; bs = s; }
      }
    }
    for (int o = 16; o; o >>= 1) {
      const uint32_t op = __shfl_xor_sync(~0u, bp, o), os = __shfl_xor_sync(~0u, bs, o);
      const uint64_t ost = __shfl_xor_sync(~0u, bst, o);
      if (op > bp || (op == bp && ost > bst)) { bp = op; bst = ost; bs = os; }
    }
    if (lane == 0) { s_bp[wid] = bp; s_bs[wid] = bs; s_bst[wid] = bst; }
  }
  __syncthreads();
  if (tid == 0) {
    il_refine_info inf;
    inf.target_stamp = 0; inf.target_slot = -1; inf.pmc = 0; inf.rule = 2; inf.reverted = 0; inf.matched = 0;
    uint32_t fin[MAXK];
    for (uint32_t j = 0; j < k; ++j) fin[j] = cur[j];
    if (c.cfg.flags & IL_F_PAIR) {
      bp = 0; bs = NONE32; bst = 0;
      for (uint32_t q = 0; q < REF_THREADS / 32; ++q)
        if (s_bp[q] > bp || (s_bp[q] == bp && s_bst[q] > bst)) { bp = s_bp[q]; bst = s_bst[q]; bs = s_bs[q]; }
      if (bp > 0) {
        inf.pmc = (uint8_t)bp; inf.matched = 1; inf.target_stamp = bst; inf.target_slot = (int32_t)bs;
        uint32_t tds[MAXK];
        for (uint32_t j = 0; j < k; ++j) tds[j] = c.tab_ds[(size_t)bs * k + j];
        if (bp == k) {
          inf.rule = 1;
          for (uint32_t j = 0; j < k; ++j) fin[j] = tds[j];
        } else {
          inf.rule = 3;
          uint32_t rep = 0, o = 0;
          for (uint32_t j = 0; j < bp; ++j) {
            const uint32_t t = c.tid[tds[j]];
            uint32_t q = 0;
            while (q < k && (((rep >> q) & 1u) || c.tid[cur[q]] != t)) ++q;
            if (q == k) latch(c.sc, IL_ERR_INTERNAL);             // cannot happen
            rep |= 1u << q;
            fin[o++] = tds[j];
          }
          for (uint32_t q = 0; q < k; ++q)
            if (!((rep >> q) & 1u)) fin[o++] = cur[q];
        }
      }
    }
    for (uint32_t j = 0; j < k; ++j) s_fin[j] = fin[j];
    s_inf = inf;
  }
  __syncthreads();
  uint32_t fin[MAXK];
  bool changed = false;
#pragma unroll
  for (int j = 0; j < MAXK; ++j) {
    fin[j] = (uint32_t)j < k ? s_fin[j] : 0;
    changed |= (uint32_t)j < k && fin[j] != cur[j];
  }
  const uint32_t qa = q_off[i], qL = q_off[i + 1] - qa;
  const uint32_t stride = c.cfg.max_prompt_tokens;
  auto plen = [&](const uint32_t* ds) {
    uint32_t L = c.n_instr + qL;
    for (uint32_t j = 0; j < k; ++j) L += c.rend_len[ds[j]];
    return L;
  };
  uint32_t* row = prompt_tok + (size_t)i * stride;
  auto render = [&](const uint32_t* ds, uint32_t* out) {        // all threads of the CTA
    uint32_t o = c.n_instr;
    {                                                  // instruction: 16-byte vectors (row stride and
      const uint32_t nv = c.n_instr / 4;               // buffers are 16-byte aligned), then the tail
      const uint4* src = reinterpret_cast<const uint4*>(c.instr);
      uint4* dst = reinterpret_cast<uint4*>(out);
      for (uint32_t x = tid; x < nv; x += REF_THREADS) dst[x] = src[x];
      for (uint32_t x = 4 * nv + tid; x < c.n_instr; x += REF_THREADS) out[x] = c.instr[x];
    }
    for (uint32_t j = 0; j < k; ++j) {
      const uint32_t d = ds[j], a = c.rend_off[d], n = c.rend_len[d];
      for (uint32_t x = tid; x < n; x += REF_THREADS) out[o + x] = c.rend_tok[a + x];
      o += n;
    }
    for (uint32_t x = tid; x < qL; x += REF_THREADS) out[o + x] = q_tok[qa + x];
  };
  uint32_t L = plen(fin);
  if (tid == 0) { s_L = L; s_rendered = 0; }
  if ((c.cfg.flags & IL_F_GUARD) && changed) {
    // never-worse guard (Z25): compare the capped hits of DS_final and DS_current against
    // the index snapshot; keep DS_current if DS_final is strictly worse.
    const uint32_t Lc = plen(cur);
    uint32_t* grow = c.guard_prompt + (size_t)i * stride;
    if (L <= stride && Lc <= stride) {
      render(fin, row);
      render(cur, grow);
      __syncthreads();
      if (wid == 0) {
        const uint32_t hf = warp_hash_match<false>(c, row, L, nullptr, nullptr, true);
        const uint32_t hc = warp_hash_match<false>(c, grow, Lc, nullptr, nullptr, true);
        if (lane == 0) {
          s_rendered = 1;
          if (hf < hc) { s_inf.reverted = 1; s_L = Lc; s_rendered = 0; }
        }
      }
      __syncthreads();
      if (s_inf.reverted) {
#pragma unroll
        for (int j = 0; j < MAXK; ++j) fin[j] = cur[j];
      }
    }
  }
  __syncthreads();
  L = s_L;
  if (L + c.cfg.max_decode_tokens > stride) {          // (the decode reserve shares the row's blocks)
    if (tid == 0) latch(c.sc, IL_ERR_ARG);
    L = 0;
  } else if (!s_rendered) {
    render(fin, row);
  }
  if (tid == 0) {
    prompt_len[i] = L;
    info[i] = s_inf;
  }
  if (tid == 0)
    for (uint32_t j = 0; j < k; ++j) final_ds[(size_t)i * k + j] = fin[j];
}

}  // namespace il

using namespace il;

// a1 + a2: exact similarity against the whole pool, top-k in ascending order
static il_status select_launch(Ctx* c, uint32_t B, const uint32_t* q_off, const uint32_t* q_tok,
                               const uint32_t* q_src, uint32_t* topk, cudaStream_t st) {
  if (c->n_demos > SIM_BIG_POOL && c->inv_slots)
    return inv_select(c, B, q_off, q_tok, q_src, topk, st);
  if (c->n_demos > SIM_BIG_POOL)
    k_sim_topk<4><<<cdiv(B, SIM_THREADS / 128), SIM_THREADS, 0, st>>>(*c, B, q_off, q_tok, q_src, topk);
  else
    k_sim_topk<IL_SIM_QW_SMALL><<<cdiv(B, SIM_THREADS / (32 * IL_SIM_QW_SMALL)), SIM_THREADS, 0, st>>>(
        *c, B, q_off, q_tok, q_src, topk);
  IL_LAUNCH_CHECK("k_sim_topk");
  c->launches += 1;
  return IL_OK;
}

extern "C" il_status il_select_batch(il_ctx* c, uint32_t B, const uint32_t* q_off, const uint32_t* q_tok,
                                     const uint32_t* q_src, uint32_t* topk, il_stream s) {
  if (!c->pool_loaded) { set_error("il_select_batch before il_pool_load"); return IL_ERR_STATE; }
  if (B > c->cfg.max_batch) { set_error("B > max_batch"); return IL_ERR_ARG; }
  if (B == 0) return IL_OK;
  il_status r = select_launch(c, B, q_off, q_tok, q_src, topk, (cudaStream_t)s);
  if (r != IL_OK) return r;
  c->sel_topk = topk;
  c->sel_B = B;
  return IL_OK;
}

extern "C" il_status il_refine_batch(il_ctx* c, uint32_t B, const uint32_t* q_off, const uint32_t* q_tok,
                                     const uint32_t* q_src, uint32_t* topk, uint32_t* final_ds,
                                     il_refine_info* info, uint32_t* prompt_tok, uint32_t* prompt_len,
                                     il_stream s) {
  if (!c->pool_loaded) { set_error("il_refine_batch before il_pool_load"); return IL_ERR_STATE; }
  if (B > c->cfg.max_batch) { set_error("B > max_batch"); return IL_ERR_ARG; }
  if (B == 0) return IL_OK;
  if (((uintptr_t)prompt_tok & 15) != 0) { set_error("prompt_tok must be 16-byte aligned"); return IL_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)s;
  const bool selected = c->sel_topk == topk && c->sel_B == B;   // il_select_batch already ran
  c->sel_topk = nullptr;
  if (!selected) {
    il_status r = select_launch(c, B, q_off, q_tok, q_src, topk, st);
    if (r != IL_OK) return r;
  }
  if (c->cfg.flags & IL_F_GUARD) k_instr_probe<<<1, 256, 0, st>>>(*c, 1u);
  k_refine<<<B, REF_THREADS, 0, st>>>(*c, B, q_off, q_tok, topk, final_ds, info, prompt_tok, prompt_len);
  IL_LAUNCH_CHECK("il_refine_batch");
  c->launches += (c->cfg.flags & IL_F_GUARD) ? 2 : 1;
  c->final_ds = final_ds;
  c->info = info;
  c->refined = true;
  c->last_B = B;
  return IL_OK;
}
