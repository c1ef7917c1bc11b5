// select_inv.cu — a1-a2 for large demo pools (configs 4-5: 10k-50k demos):
// exact cosine / Jaccard similarity + top-k through an inverted index of the pool.
//
// The per-query pool scan (k_sim_topk) reads every demo's token set for every query: at a
// 10,000-demo pool that is ~1.6 MB of L2 traffic and ~1.5e5 hash probes per query.  Here the
// pool is indexed once at il_pool_load: for each (token, chunk of SIM_CHUNK demos) the posting
// list of (demo, count).  A query then touches only the demos that share a token with it:
//   dot(q, m) = sum_{t in q} c_q(t) c_m(t)   (cosine)      inter(q, m) = |{t in q and m}|  (Jaccard)
// accumulated in shared memory per chunk by walking the postings of the query's distinct
// tokens; every demo of the chunk is then scored exactly from its accumulator (demos sharing no
// token score 0, as in the definition) and ranked with the same exact fraction order as
// k_sim_topk (Z4-Z8).  The result is identical to the full scan.
#include "il_internal.cuh"
#include "sim_dev.cuh"

namespace il {

__device__ __forceinline__ uint64_t inv_keyof(uint32_t tok, uint32_t chunk) {
  return (((uint64_t)chunk << 32) | tok) + 1ull;
}
__device__ __forceinline__ uint32_t inv_hash(uint64_t key, uint32_t mask) {
  return (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 32) & mask;
}
__device__ __forceinline__ uint32_t inv_find(const Ctx& c, uint64_t key) {
  uint32_t s = inv_hash(key, c.inv_mask);
  for (uint32_t n = 0; n <= c.inv_mask; ++n) {
    const uint64_t k = c.inv_key[s];
    if (k == key) return s;
    if (k == 0) return NONE32;
    s = (s + 1) & c.inv_mask;
  }
  return NONE32;
}

__global__ void k_inv_reset(Ctx c) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < c.inv_slots; s += stride) {
    c.inv_key[s] = 0; c.inv_len[s] = 0; c.inv_fill[s] = 0;
  }
}

// one warp per demo: insert its (token, chunk) keys, count postings
__global__ void __launch_bounds__(256) k_inv_count(Ctx c, uint32_t n) {
  const uint32_t m = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (m >= n) return;
  const uint32_t a = c.log_off[m], nu = c.uniq_n[m], ch = m / SIM_CHUNK;
  for (uint32_t u = lane; u < nu; u += 32) {
    const uint64_t key = inv_keyof(c.uniq_tok[a + u], ch);
    uint32_t s = inv_hash(key, c.inv_mask);
    while (true) {
      const uint64_t old = atomicCAS((unsigned long long*)&c.inv_key[s], 0ull, (unsigned long long)key);
      if (old == 0 || old == key) break;
      s = (s + 1) & c.inv_mask;
    }
    atomicAdd(&c.inv_len[s], 1u);
  }
}

// one CTA: exclusive scan of the posting lengths over all slots -> inv_off
__global__ void __launch_bounds__(1024) k_inv_scan(Ctx c) {
  __shared__ uint32_t s_w[32];
  const uint32_t per = cdiv(c.inv_slots, 1024), lo = threadIdx.x * per, hi = min(lo + per, c.inv_slots);
  uint32_t sum = 0;
  for (uint32_t s = lo; s < hi; ++s) sum += c.inv_len[s];
  uint32_t total;
  uint32_t acc = block_scan(sum, s_w, &total);
  for (uint32_t s = lo; s < hi; ++s) { c.inv_off[s] = acc; acc += c.inv_len[s]; }
}

// one warp per demo: append (demo, count) to its postings (order inside a list is irrelevant:
// every demo occurs once per list and the accumulation is an integer sum)
__global__ void __launch_bounds__(256) k_inv_fill(Ctx c, uint32_t n) {
  const uint32_t m = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (m >= n) return;
  const uint32_t a = c.log_off[m], nu = c.uniq_n[m], ch = m / SIM_CHUNK;
  for (uint32_t u = lane; u < nu; u += 32) {
    const uint32_t s = inv_find(c, inv_keyof(c.uniq_tok[a + u], ch));
    const uint32_t pos = c.inv_off[s] + atomicAdd(&c.inv_fill[s], 1u);
    c.post_demo[pos] = ((m - ch * SIM_CHUNK) << 18) | c.uniq_cnt[a + u];   // demo in chunk | count (<= 256)
  }
}

constexpr int INV_THREADS = 256;
constexpr int INV_QHASH = 512;
constexpr uint32_t INV_SMEM = SIM_CHUNK * 2;      // the per-chunk accumulator: 16-bit per demo, two per word
// (dot <= 255 x 255 < 2^16 with logs of <= 255 tokens (validate), so a half never carries into
// the other)

__device__ __forceinline__ uint32_t inv_qslot(uint32_t t) { return (t * 0x9E3779B1u) >> (32 - 9); }

// One CTA per query.
__global__ void __launch_bounds__(INV_THREADS) k_sim_inv(Ctx c, uint32_t B, const uint32_t* __restrict__ q_off,
                                                         const uint32_t* __restrict__ q_tok,
                                                         const uint32_t* __restrict__ q_src,
                                                         uint32_t* __restrict__ topk) {
  constexpr uint32_t NW = INV_THREADS / 32;
  extern __shared__ uint32_t s_acc[];                 // [SIM_CHUNK / 2] packed u16 accumulators
  __shared__ uint32_t s_key[INV_QHASH], s_cnt[INV_QHASH];
  __shared__ uint32_t s_ut[256], s_uc[256], s_po[256], s_pre[257];
  __shared__ uint32_t s_nu, s_red[NW][2];
  __shared__ Cand s_wl[NW][MAXK], s_sel[MAXK];
  __shared__ uint32_t s_wn[NW];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t i = blockIdx.x;
  const uint32_t k = c.cfg.k, n = c.n_demos;
  const uint32_t qa = q_off[i];
  uint32_t qL = q_off[i + 1] - qa;
  if (qL > c.cfg.max_log_tokens) {                      // (uniform)
    if (tid == 0) latch(c.sc, IL_ERR_ARG);
    return;
  }
  // query multiset: distinct tokens with counts
  for (uint32_t x = tid; x < INV_QHASH; x += INV_THREADS) { s_key[x] = NONE32; s_cnt[x] = 0; }
  if (tid == 0) s_nu = 0;
  __syncthreads();
  for (uint32_t x = tid; x < qL; x += INV_THREADS) {
    const uint32_t t = q_tok[qa + x];
    uint32_t s = inv_qslot(t);
    while (true) {
      const uint32_t old = atomicCAS(&s_key[s], NONE32, t);
      if (old == NONE32 || old == t) break;
      s = (s + 1) & (INV_QHASH - 1);
    }
    atomicAdd(&s_cnt[s], 1u);
  }
  __syncthreads();
  uint32_t nq = 0;
  for (uint32_t x = tid; x < INV_QHASH; x += INV_THREADS) {
    if (s_key[x] == NONE32) continue;
    const uint32_t u = atomicAdd(&s_nu, 1u);
    s_ut[u] = s_key[x]; s_uc[u] = s_cnt[x];
    nq += s_cnt[x] * s_cnt[x];
  }
  for (int o = 16; o; o >>= 1) nq += __shfl_xor_sync(~0u, nq, o);
  if (lane == 0) s_red[wid][0] = nq;
  __syncthreads();
  nq = 0;
  for (uint32_t w = 0; w < NW; ++w) nq += s_red[w][0];
  const uint32_t nuq = s_nu;
  const bool jac = c.cfg.metric == IL_SIM_JACCARD;
  const bool excl = (c.cfg.flags & IL_F_EXCLUDE_SELF) != 0;
  const uint32_t my_src = (excl && q_src) ? q_src[i] : NONE32;

  // one sorted top-k list per WARP: lane j < k holds entry j (best first).  Lanes score 32
  // demos at a time; a demo whose fp32 quotient is clearly below the list's k-th entry (margin
  // 2^-20, far above the quotients' rounding error) ranks below it exactly and is dropped; the
  // few others are inserted one at a time with the exact comparison (warp-parallel insert).
  Cand e;
  e.num = 0; e.den = 1; e.idx = NONE32;
  uint32_t nw = 0;                                      // entries in the warp's list (uniform)
  float fk = 0.f;
  Cand last = e;                                        // the list's k-th entry, in every lane
  const uint32_t n_chunks = cdiv(n, SIM_CHUNK);
  for (uint32_t ch = 0; ch < n_chunks; ++ch) {
    const uint32_t m0 = ch * SIM_CHUNK, mc = min(SIM_CHUNK, n - m0);
    for (uint32_t x = tid; x < (mc + 1) / 2; x += INV_THREADS) s_acc[x] = 0;
    __syncthreads();
    // the postings of the query's distinct tokens in this chunk: token lookups, then their
    // concatenation is cut into NW equal segments (warp w walks segment w: a long posting list
    // is shared by several warps), lanes take 4 consecutive 32-wide rows of postings at a time
    uint32_t len = 0;
    if (tid < nuq) {
      const uint32_t sl = inv_find(c, inv_keyof(s_ut[tid], ch));
      s_po[tid] = sl == NONE32 ? 0u : c.inv_off[sl];
      len = sl == NONE32 ? 0u : c.inv_len[sl];
    }
    {
      uint32_t x = len;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(~0u, x, o);
        if (lane >= (uint32_t)o) x += y;
      }
      if (lane == 31) s_red[wid][1] = x;
      __syncthreads();
      uint32_t base = 0;
      for (uint32_t w = 0; w < wid; ++w) base += s_red[w][1];
      s_pre[tid + 1] = base + x;
      if (tid == 0) s_pre[0] = 0;
    }
    __syncthreads();
    {
      const uint32_t tot = s_pre[nuq], seg = cdiv(tot, NW);
      const uint32_t x_lo = min(tot, wid * seg), x_hi = min(tot, x_lo + seg);
      uint32_t u = 0;                                   // token holding x_lo: s_pre[u] <= x_lo < s_pre[u + 1]
      {
        uint32_t lo = 0, hi = nuq;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (s_pre[mid] <= x_lo) lo = mid; else hi = mid;
        }
        u = lo;
      }
      for (uint32_t x0 = x_lo; x0 < x_hi;) {
        while (s_pre[u + 1] <= x0) ++u;                  // (warp-uniform)
        const uint32_t end = min(x_hi, s_pre[u + 1]);
        const uint32_t off = s_po[u] - s_pre[u], cq = jac ? 1u : s_uc[u];
        uint32_t pk[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t x = x0 + 32 * e + lane;
          pk[e] = x < end ? __ldg(c.post_demo + (off + x)) : NONE32;   // (u32 sum: off may wrap)
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (pk[e] != NONE32) {
            const uint32_t d = pk[e] >> 18;
            atomicAdd(&s_acc[d >> 1], (jac ? 1u : cq * (pk[e] & 0x3FFFFu)) << (16 * (d & 1)));
          }
        x0 = min(end, x0 + 128);
      }
    }
    __syncthreads();
    // score every demo of the chunk exactly; warp-level top-k
    for (uint32_t x0 = wid * 32; x0 < mc; x0 += INV_THREADS) {
      const uint32_t x = x0 + lane, m = m0 + x;
      Cand y;
      y.num = 0; y.den = 1; y.idx = m;
      bool cand = x < mc && !(excl && c.src[m] == my_src);
      if (cand) {
        const uint32_t acc = (s_acc[x >> 1] >> (16 * (x & 1))) & 0xFFFFu;
        float fy;
        if (jac) {
          const uint32_t nu = c.uniq_n[m];
          if (nuq == 0 && nu == 0) { y.num = 1; y.den = 1; }
          else { y.num = acc; y.den = nuq + nu - acc; }
          fy = __fdividef((float)y.num, (float)y.den);
        } else {
          const uint32_t nm = c.norm2[m];
          if (nq != 0 && nm != 0) { y.num = (uint64_t)acc * acc; y.den = nm; }   // else 0 (Z5)
          const float fa = (float)acc;
          fy = y.num ? __fdividef(fa * fa, (float)y.den) : 0.f;
        }
        // (fy and fk: relative error < 2^-21 each, far inside the 2^-20 margin)
        cand = nw < k || (fy >= fk && better(y, last));   // exact test only near the threshold
      }
      uint32_t msk = __ballot_sync(~0u, cand);
      while (msk) {
        const uint32_t src = __ffs(msk) - 1;
        msk &= msk - 1;
        Cand cy;
        cy.num = __shfl_sync(~0u, y.num, src); cy.den = __shfl_sync(~0u, y.den, src);
        cy.idx = __shfl_sync(~0u, y.idx, src);
        if (nw >= k && !better(cy, last)) continue;    // (uniform: an earlier insert raised the bar)
        const bool bt = lane < k && (lane >= nw || better(cy, e));
        const bool bl = __shfl_up_sync(~0u, bt, 1) && lane > 0;
        Cand el;
        el.num = __shfl_up_sync(~0u, e.num, 1); el.den = __shfl_up_sync(~0u, e.den, 1);
        el.idx = __shfl_up_sync(~0u, e.idx, 1);
        if (bt) e = bl ? el : cy;
        nw = min(nw + 1, k);
        if (nw == k) {
          last.num = __shfl_sync(~0u, e.num, k - 1); last.den = __shfl_sync(~0u, e.den, k - 1);
          last.idx = __shfl_sync(~0u, e.idx, k - 1);
          fk = ((float)last.num / (float)last.den) * (1.f - 9.5367431640625e-7f);   // IEEE quotient (rare)
        }
      }
    }
    __syncthreads();                                    // s_acc reused by the next chunk (and the merge)
  }
  if (lane < k) s_wl[wid][lane] = e;
  const uint32_t nsel_w = nw;
  if (lane == 0) s_wn[wid] = nsel_w;
  __syncthreads();
  if (wid != 0) return;
  const uint32_t wn = lane < NW ? s_wn[lane] : 0u;
  const uint32_t nsel = warp_merge([&](uint32_t q) { return s_wl[lane][q]; }, wn, k, lane, s_sel);
  __syncwarp();
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

}  // namespace il

using namespace il;

il_status il::inv_setup(Ctx* c) {
  if (!c->inv_slots) return IL_OK;
  IL_CUDA(cudaFuncSetAttribute(k_sim_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, INV_SMEM));
  return IL_OK;
}

il_status il::inv_build(Ctx* c, uint32_t n, cudaStream_t st) {
  if (!c->inv_slots) return IL_OK;
  k_inv_reset<<<c->num_sms * 4, 256, 0, st>>>(*c);
  k_inv_count<<<cdiv(n * 32, 256), 256, 0, st>>>(*c, n);
  k_inv_scan<<<1, 1024, 0, st>>>(*c);
  k_inv_fill<<<cdiv(n * 32, 256), 256, 0, st>>>(*c, n);
  IL_LAUNCH_CHECK("inverted index build");
  c->launches += 4;
  return IL_OK;
}

il_status il::inv_select(Ctx* c, uint32_t B, const uint32_t* q_off, const uint32_t* q_tok, const uint32_t* q_src,
                         uint32_t* topk, cudaStream_t st) {
  k_sim_inv<<<B, INV_THREADS, INV_SMEM, st>>>(*c, B, q_off, q_tok, q_src, topk);
  IL_LAUNCH_CHECK("k_sim_inv");
  c->launches += 1;
  return IL_OK;
}
