// ctx.cu — lifecycle, workspace carve-up, status latch, pool load (K0), dumps.
#include <algorithm>
#include <cstring>
#include <new>
#include <vector>

#include "il_internal.cuh"

namespace il {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
il_status cuda_check(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return IL_ERR_CUDA;
}

struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base((char*)b) {}
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? (T*)(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

static uint32_t slots_for(uint32_t C) {
  uint32_t n = 1;
  while (n < 2 * C) n <<= 1;
  return std::max(n, 64u);
}

static size_t carve(Ctx* c, void* ws) {
  const il_config& g = c->cfg;
  Carver w(ws);
  const size_t M = g.max_pool, PT = g.max_pool_tokens, T = g.table_capacity, C = g.kv_pages;
  const size_t B = g.max_batch, MB = c->max_blocks, NS = c->n_slots;
  c->sc = w.take<DevScalars>(1);
  c->log_off = w.take<uint32_t>(M + 1); c->log_tok = w.take<uint32_t>(PT);
  c->tpl_off = w.take<uint32_t>(M + 1); c->tpl_tok = w.take<uint32_t>(PT);
  c->tid = w.take<uint32_t>(M); c->src = w.take<uint32_t>(M);
  c->uniq_tok = w.take<uint32_t>(PT); c->uniq_cnt = w.take<uint32_t>(PT);
  c->uniq_n = w.take<uint32_t>(M); c->norm2 = w.take<uint32_t>(M);
  c->rend_off = w.take<uint32_t>(M + 1); c->rend_tok = w.take<uint32_t>(2 * PT + 2 * M);
  c->rend_len = w.take<uint32_t>(M);
  c->instr = w.take<uint32_t>(g.max_prompt_tokens);
  c->instr_hash = w.take<uint64_t>(g.max_prompt_tokens / 16 + 1);
  c->instr_pages = w.take<int32_t>(g.max_prompt_tokens / 16 + 1);
  c->tab_ds = w.take<uint32_t>(T * g.k); c->tab_tpl = w.take<uint32_t>(T * g.k);
  c->tab_stamp = w.take<uint64_t>(T);
  c->slot_key = w.take<uint64_t>(NS); c->slot_page = w.take<uint32_t>(NS);
  c->claim = w.take<uint32_t>(NS); c->cstamp = w.take<uint64_t>(NS);
  c->pg_hash = w.take<uint64_t>(C); c->pg_parent = w.take<uint64_t>(C); c->pg_stamp = w.take<uint64_t>(C);
  c->pg_tok = w.take<uint32_t>(C * BS); c->pg_depth = w.take<uint32_t>(C);
  c->pg_slot = w.take<uint32_t>(C); c->pg_state = w.take<uint32_t>(C); c->pg_pin = w.take<uint32_t>(C);
  c->free_list = w.take<uint32_t>(C);
  c->need_off = w.take<uint32_t>(B + 1);
  c->occ = w.take<uint32_t>(B * MB);
  c->hist = w.take<uint32_t>(4096);
  const size_t R = std::max<size_t>(B, g.max_global_batch);   // table-commit records
  c->max_records = (uint32_t)R;
  c->tab_find = w.take<int32_t>(R); c->tab_last = w.take<uint32_t>(R); c->tab_hash = w.take<uint64_t>(R);
  c->tab_slot = w.take<uint32_t>(R);
  {
    uint32_t n = 64;
    while (n < 2 * R) n <<= 1;
    c->dd_mask = n - 1;
    c->dd_key = w.take<uint64_t>(n); c->dd_max = w.take<uint32_t>(n);
  }
  c->tile_off = w.take<uint32_t>(B + 1);
  c->tile_req = w.take<uint32_t>((size_t)g.max_suffix_tokens / 16 + B + 1);
  c->tile_desc = w.take<uint4>((size_t)g.max_suffix_tokens / 16 + B + 1);
  c->pair_nsh = w.take<uint32_t>((size_t)g.max_suffix_tokens / 32 + B + 1);
  c->attn_ml = w.take<float>((size_t)g.max_suffix_tokens * g.n_q_heads);
  c->evicted_list = w.take<uint64_t>(C);
  c->hit_local = w.take<uint32_t>(B);
  c->dec_cu = w.take<uint32_t>(B + 1);
  if (g.flags & IL_F_DEDUP) {                          // every full block of the batch, half full
    uint32_t n = 1024;
    while (n < 2ull * B * MB) n <<= 1;
    c->bd_mask = n - 1;
    c->bd_key = w.take<uint64_t>(n); c->bd_owner = w.take<uint32_t>(n); c->bd_list = w.take<uint32_t>(B * MB);
  } else {
    c->bd_mask = 0; c->bd_key = nullptr; c->bd_owner = c->bd_list = nullptr;
  }
  c->guard_prompt = (g.flags & IL_F_GUARD) ? w.take<uint32_t>(B * g.max_prompt_tokens) : nullptr;
  // inverted index for large pools (a1-a2, select_inv.cu): slots for every (token, chunk) key
  if (g.max_pool > SIM_BIG_POOL) {
    uint32_t n = 1024;
    while (n < 2 * PT) n <<= 1;
    c->inv_slots = n; c->inv_mask = n - 1;
    c->inv_key = w.take<uint64_t>(n);
    c->inv_off = w.take<uint32_t>(n); c->inv_len = w.take<uint32_t>(n); c->inv_fill = w.take<uint32_t>(n);
    c->post_demo = w.take<uint32_t>(PT);
  } else {
    c->inv_slots = c->inv_mask = 0;
    c->inv_key = nullptr; c->inv_off = c->inv_len = c->inv_fill = c->post_demo = nullptr;
  }
  // multi-GPU exchange: block-record FIFO, residency map (2 x ranks x C slots), box hits, gathered
  // ICL records
  c->n_ranks_max = g.max_global_batch > B ? (uint32_t)((g.max_global_batch + B - 1) / B) : 1;
  if (c->n_ranks_max > 1) {
    c->rec_R = g.max_block_records ? g.max_block_records : 16 * (uint32_t)B;
    c->ring_cap = (uint32_t)(4 * C + B * MB + c->rec_R);
    uint32_t n = 1024;
    while (n < 2ull * c->n_ranks_max * C) n <<= 1;
    c->map_slots = n; c->map_smask = n - 1;
    c->ins_list = w.take<uint64_t>(std::min<size_t>(C, B * MB));
    c->ring = w.take<uint64_t>(c->ring_cap);
    c->map_key = w.take<uint64_t>(n); c->map_mask = w.take<uint32_t>(n);
    c->map_tmp_key = w.take<uint64_t>(n); c->map_tmp_mask = w.take<uint32_t>(n);
    c->box_hit = w.take<uint32_t>(B);
    c->icl_fds = w.take<uint32_t>(R * g.k);
    c->icl_info = w.take<il_refine_info>(R);
  } else {
    c->rec_R = c->ring_cap = c->map_slots = c->map_smask = 0;
    c->ins_list = c->ring = c->map_key = c->map_tmp_key = nullptr;
    c->map_mask = c->map_tmp_mask = c->box_hit = c->icl_fds = nullptr;
    c->icl_info = nullptr;
  }
  return w.off + 256;
}

static il_status validate(const il_config* g) {
  if (!g) { set_error("null config"); return IL_ERR_ARG; }
  if (g->k < 1 || g->k > MAXK) { set_error("k must be in 1..8"); return IL_ERR_ARG; }
  if (g->table_capacity < 1 || g->table_capacity > 8192) { set_error("table_capacity in 1..8192"); return IL_ERR_ARG; }
  if (g->kv_pages < 1) { set_error("kv_pages >= 1"); return IL_ERR_ARG; }
  if (g->max_batch < 1 || g->max_batch > 8192) { set_error("max_batch in 1..8192"); return IL_ERR_ARG; }
  if (g->max_global_batch > 8192) { set_error("max_global_batch <= 8192"); return IL_ERR_ARG; }
  if (g->max_global_batch > g->max_batch && (g->max_global_batch + g->max_batch - 1) / g->max_batch > 32) {
    set_error("at most 32 ranks (max_global_batch / max_batch)"); return IL_ERR_ARG;
  }
  if (g->max_block_records > (1u << 24)) { set_error("max_block_records <= 2^24"); return IL_ERR_ARG; }
  if (g->flags & ~0x1Fu) { set_error("unknown il_config.flags bits"); return IL_ERR_ARG; }
  if (g->reserved1 != 0) { set_error("il_config.reserved1 must be 0"); return IL_ERR_ARG; }
  if (g->max_decode_tokens >= g->max_prompt_tokens) { set_error("max_decode_tokens >= max_prompt_tokens"); return IL_ERR_ARG; }
  if (g->max_prompt_tokens < 16 || (g->max_prompt_tokens % 16)) { set_error("max_prompt_tokens: multiple of 16"); return IL_ERR_ARG; }
  if (g->max_pool < g->k) { set_error("max_pool < k"); return IL_ERR_ARG; }
  if (g->max_log_tokens < 1 || g->max_log_tokens > 256) { set_error("max_log_tokens in 1..256"); return IL_ERR_ARG; }
  if (g->max_pool > SIM_BIG_POOL && g->max_log_tokens > 255) {
    set_error("pools above 1,024 demos (inverted-index selection) need max_log_tokens <= 255"); return IL_ERR_ARG;
  }
  if (g->n_kv_heads < 1 || g->n_q_heads % g->n_kv_heads) { set_error("Hq % Hkv != 0"); return IL_ERR_ARG; }
  if (g->head_dim != 64 && g->head_dim != 128) { set_error("head_dim must be 64 or 128"); return IL_ERR_ARG; }
  if (g->n_q_heads / g->n_kv_heads > 8) { set_error("Hq / Hkv must be <= 8"); return IL_ERR_ARG; }
  if (g->metric > 1) { set_error("metric"); return IL_ERR_ARG; }
  return IL_OK;
}

// --------------------------------------------------------------------------- kernels
__global__ void k_reset_index(Ctx c) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < c.n_slots; s += stride) {
    c.slot_key[s] = KEY_EMPTY; c.slot_page[s] = NONE32; c.claim[s] = NONE32; c.cstamp[s] = 0;
  }
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < c.cfg.kv_pages; p += stride) {
    c.pg_state[p] = 0; c.pg_pin[p] = 0; c.pg_stamp[p] = 0; c.pg_slot[p] = NONE32;
    c.free_list[p] = c.cfg.kv_pages - 1 - p;   // pop order 0, 1, 2, ...
  }
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < c.cfg.table_capacity; t += stride)
    c.tab_stamp[t] = 0;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < 4096; t += stride) c.hist[t] = 0;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t <= c.dd_mask; t += stride) { c.dd_key[t] = 0; c.dd_max[t] = 0; }
  if (c.bd_key)
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t <= c.bd_mask; t += stride) { c.bd_key[t] = 0; c.bd_owner[t] = 0; }
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t <= c.cfg.max_batch; t += stride) c.dec_cu[t] = t;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    DevScalars z;
    memset(&z, 0, sizeof(z));
    z.n_free = c.cfg.kv_pages;
    *c.sc = z;
  }
}

// Per-demo token set for a1: sorted unique log tokens with counts, |set|, sum of counts^2.
// One warp per demo (8 per CTA), logs staged in shared memory; rank-based sort (<= 256 tokens).
__global__ void __launch_bounds__(256) k_pool_sets(Ctx c, uint32_t n, const uint32_t* __restrict__ log_off,
                                                   const uint32_t* __restrict__ log_tok) {
  __shared__ uint32_t s_tok[8][256];
  __shared__ uint8_t s_first[8][256];
  const uint32_t wl = threadIdx.x >> 5, warp = blockIdx.x * 8 + wl, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const uint32_t a = log_off[warp], L = log_off[warp + 1] - a;
  if (L > c.cfg.max_log_tokens || L > 256) { if (lane == 0) latch(c.sc, IL_ERR_ARG); return; }
  for (uint32_t x = lane; x < L; x += 32) s_tok[wl][x] = log_tok[a + x];
  __syncwarp();
  for (uint32_t x = lane; x < L; x += 32) {
    const uint32_t t = s_tok[wl][x];
    bool first = true;
    for (uint32_t y = 0; y < x; ++y) first &= s_tok[wl][y] != t;
    s_first[wl][x] = first;
  }
  __syncwarp();
  uint32_t nu = 0, n2 = 0;
  for (uint32_t x = lane; x < L; x += 32) {
    if (!s_first[wl][x]) continue;
    const uint32_t t = s_tok[wl][x];
    uint32_t rank = 0, cnt = 0;           // rank among distinct tokens; multiplicity
    for (uint32_t y = 0; y < L; ++y) {
      const uint32_t u = s_tok[wl][y];
      rank += (u < t) && s_first[wl][y];
      cnt += u == t;
    }
    c.uniq_tok[a + rank] = t;
    c.uniq_cnt[a + rank] = cnt;
    nu += 1; n2 += cnt * cnt;
  }
  for (int o = 16; o; o >>= 1) { nu += __shfl_xor_sync(~0u, nu, o); n2 += __shfl_xor_sync(~0u, n2, o); }
  if (lane == 0) { c.uniq_n[warp] = nu; c.norm2[warp] = n2; }
}

__global__ void k_pool_copy(Ctx c, uint32_t n, const uint32_t* __restrict__ log_off,
                            const uint32_t* __restrict__ log_tok, const uint32_t* __restrict__ tpl_off,
                            const uint32_t* __restrict__ tpl_tok, const uint32_t* __restrict__ tid,
                            const uint32_t* __restrict__ src, const uint32_t* __restrict__ instr,
                            uint32_t n_instr) {
  const uint32_t stride = gridDim.x * blockDim.x, t0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t m = t0; m <= n; m += stride) { c.log_off[m] = log_off[m]; c.tpl_off[m] = tpl_off[m]; }
  for (uint32_t m = t0; m < n; m += stride) {
    c.tid[m] = tid[m]; c.src[m] = src[m];
    c.rend_len[m] = (log_off[m + 1] - log_off[m]) + (tpl_off[m + 1] - tpl_off[m]) + 2;
  }
  for (uint32_t x = t0; x < log_off[n]; x += stride) c.log_tok[x] = log_tok[x];
  for (uint32_t x = t0; x < tpl_off[n]; x += stride) c.tpl_tok[x] = tpl_tok[x];
  for (uint32_t x = t0; x < n_instr; x += stride) c.instr[x] = instr[x];
}

// chain hashes of the instruction's full blocks (one warp; the same fold as every prompt's
// first blocks, since every prompt starts with the instruction)
__global__ void k_instr_hash(Ctx c, uint32_t nI) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t prev = root_hash(c.cfg.hash_seed);
  for (uint32_t base = 0; base < nI; base += 32) {
    const uint32_t j = base + lane;
    uint32_t tok[16];
    uint64_t content = 0;
    if (j < nI) content = block_content(c.instr + (size_t)BS * j, tok);
    const uint32_t nb = min(32u, nI - base);
    for (uint32_t t = 0; t < nb; ++t) {
      prev = chain_step(prev, __shfl_sync(~0u, content, t));
      if (lane == t) c.instr_hash[j] = prev;
    }
  }
}

// exclusive scan of rend_len -> rend_off (one CTA)
__global__ void k_pool_scan(Ctx c, uint32_t n) {
  __shared__ uint32_t part[1024];
  const uint32_t tid = threadIdx.x, per = cdiv(n, blockDim.x);
  uint32_t s = 0;
  for (uint32_t m = tid * per; m < min(n, (tid + 1) * per); ++m) s += c.rend_len[m];
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    uint32_t acc = 0;
    for (uint32_t t = 0; t < blockDim.x; ++t) { uint32_t v = part[t]; part[t] = acc; acc += v; }
    c.rend_off[n] = acc;
  }
  __syncthreads();
  uint32_t acc = part[tid];
  for (uint32_t m = tid * per; m < min(n, (tid + 1) * per); ++m) { c.rend_off[m] = acc; acc += c.rend_len[m]; }
}

// render(m) = log ++ [TPL] ++ template ++ [SEP]  (Z9), one warp per demo
__global__ void k_pool_render(Ctx c, uint32_t n) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n) return;
  const uint32_t o = c.rend_off[warp];
  const uint32_t la = c.log_off[warp], ll = c.log_off[warp + 1] - la;
  const uint32_t ta = c.tpl_off[warp], tl = c.tpl_off[warp + 1] - ta;
  for (uint32_t x = lane; x < ll + tl + 2; x += 32) {
    uint32_t v;
    if (x < ll) v = c.log_tok[la + x];
    else if (x == ll) v = TOK_TPL;
    else if (x < ll + 1 + tl) v = c.tpl_tok[ta + x - ll - 1];
    else v = TOK_SEP;
    c.rend_tok[o + x] = v;
  }
}

__global__ void k_gather_index(Ctx c, uint64_t* hash, uint64_t* stamp, uint32_t* depth, uint64_t* parent,
                               uint32_t* counter) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < c.cfg.kv_pages; p += gridDim.x * blockDim.x) {
    if (c.pg_state[p] == 1) {
      uint32_t o = atomicAdd(counter, 1u);
      hash[o] = c.pg_hash[p]; stamp[o] = c.pg_stamp[p]; depth[o] = c.pg_depth[p]; parent[o] = c.pg_parent[p];
    }
  }
}

}  // namespace il

using namespace il;

extern "C" {

const char* il_last_error(void) { return g_last_error.c_str(); }

il_status il_workspace_bytes(const il_config* cfg, size_t* bytes) {
  il_status st = validate(cfg);
  if (st) return st;
  Ctx c;
  c.cfg = *cfg;
  c.max_blocks = cdiv(cfg->max_prompt_tokens, BS);
  c.n_slots = slots_for(cfg->kv_pages);
  *bytes = carve(&c, nullptr);
  return IL_OK;
}

il_status il_create(const il_config* cfg, void* ws, size_t bytes, il_stream s, il_ctx** out) {
  il_status st = validate(cfg);
  if (st) return st;
  il_ctx* c = new (std::nothrow) il_ctx();
  if (!c) { set_error("host OOM"); return IL_ERR_INTERNAL; }
  c->cfg = *cfg;
  c->max_blocks = cdiv(cfg->max_prompt_tokens, BS);
  c->n_slots = slots_for(cfg->kv_pages);
  c->slot_mask = c->n_slots - 1;
  size_t need = carve(c, nullptr);
  if (bytes < need || ((uintptr_t)ws & 255)) {
    set_error("workspace too small or not 256-byte aligned");
    delete c;
    return IL_ERR_ARG;
  }
  carve(c, ws);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
  for (il_status (*f)(Ctx*) : {match_setup, commit_setup, attn_setup, records_setup, inv_setup}) {
    st = f(c);
    if (st) { delete c; return st; }
  }
  k_reset_index<<<c->num_sms * 4, 256, 0, (cudaStream_t)s>>>(*c);
  IL_LAUNCH_CHECK("k_reset_index");
  st = records_reset(c, (cudaStream_t)s);
  if (st) { delete c; return st; }
  *out = c;
  return IL_OK;
}

il_status il_destroy(il_ctx* c) {
  delete c;
  return IL_OK;
}

il_status il_status_sync(il_ctx* c, il_stream s) {
  uint32_t st = 0;
  IL_CUDA(cudaMemcpyAsync(&st, &c->sc->status, 4, cudaMemcpyDeviceToHost, (cudaStream_t)s));
  IL_CUDA(cudaStreamSynchronize((cudaStream_t)s));
  if (st) {
    IL_CUDA(cudaMemsetAsync(&c->sc->status, 0, 4, (cudaStream_t)s));
    IL_CUDA(cudaStreamSynchronize((cudaStream_t)s));
    set_error(st == IL_ERR_CAPACITY ? "device: capacity exceeded (KV pages or suffix rows)"
              : st == IL_ERR_ARG    ? "device: argument error (prompt / log too long, k > candidates)"
                                    : "device: internal invariant broken");
  }
  return (il_status)st;
}

static __global__ void k_stats(Ctx c, il_stats* out, uint64_t launches) {
  const DevScalars& h = *c.sc;
  out->batch = h.batch_done;
  out->resident_blocks = h.resident;
  out->free_pages = h.n_free;
  out->table_entries = h.table_entries;
  out->evicted_blocks = h.evicted;
  out->need_pages = h.need_total;
  out->suffix_tokens = h.suffix_total;
  out->index_rebuilds = h.rebuilds;
  out->status = h.status;
  out->launches = launches;
  out->hit_blocks = h.hit_sum;
  out->box_hit_blocks = h.box_hit_sum;
  out->full_blocks = h.full_sum;
  out->record_backlog = (uint32_t)(h.ring_tail - h.ring_head);
  out->map_slots_used = h.map_used;
  out->dedup_blocks = h.dedup_sum;
}

il_status il_set_sm_split(il_ctx* c, uint32_t attn_ctas) {
  if (attn_ctas >= (uint32_t)c->num_sms) { set_error("il_set_sm_split: attn_ctas >= SM count"); return IL_ERR_ARG; }
  const int aux = attn_ctas ? c->num_sms - (int)attn_ctas : c->num_sms;
  c->attn_ctas = (int)attn_ctas;
  c->ev_blocks = c->ev_per_sm * aux;
  c->rb_blocks = c->rb_per_sm * aux;
  c->mb_blocks = c->mb_per_sm * aux;
  return IL_OK;
}

il_status il_stats_async(il_ctx* c, il_stats* out, il_stream s) {
  if (!out || ((uintptr_t)out & 7)) { set_error("il_stats_async: null or misaligned output"); return IL_ERR_ARG; }
  k_stats<<<1, 1, 0, (cudaStream_t)s>>>(*c, out, c->launches);
  IL_LAUNCH_CHECK("k_stats");
  c->launches += 1;
  return IL_OK;
}

il_status il_stats_sync(il_ctx* c, il_stream s, il_stats* out) {
  DevScalars h;
  IL_CUDA(cudaMemcpyAsync(&h, c->sc, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)s));
  IL_CUDA(cudaStreamSynchronize((cudaStream_t)s));
  out->batch = h.batch_done;
  out->resident_blocks = h.resident;
  out->free_pages = h.n_free;
  out->table_entries = h.table_entries;
  out->evicted_blocks = h.evicted;
  out->need_pages = h.need_total;
  out->suffix_tokens = h.suffix_total;
  out->index_rebuilds = h.rebuilds;
  out->status = h.status;
  out->launches = c->launches;
  out->hit_blocks = h.hit_sum;
  out->box_hit_blocks = h.box_hit_sum;
  out->full_blocks = h.full_sum;
  out->record_backlog = (uint32_t)(h.ring_tail - h.ring_head);
  out->map_slots_used = h.map_used;
  out->dedup_blocks = h.dedup_sum;
  return IL_OK;
}

il_status il_pool_load(il_ctx* c, uint32_t n, const uint32_t* log_off, const uint32_t* log_tok,
                       const uint32_t* tpl_off, const uint32_t* tpl_tok, const uint32_t* template_id,
                       const uint32_t* src_index, const uint32_t* instr_tok, uint32_t n_instr,
                       il_stream s) {
  const il_config& g = c->cfg;
  if (n < g.k || n > g.max_pool) { set_error("n_demos must be in [k, max_pool]"); return IL_ERR_ARG; }
  if (n_instr > g.max_prompt_tokens) { set_error("instruction longer than max_prompt_tokens"); return IL_ERR_ARG; }
  // the per-batch instruction touch/pin (k_alloc_scan) covers at most 1,024 instruction blocks
  if (n_instr / BS > 1024) { set_error("instruction longer than 16,384 tokens"); return IL_ERR_ARG; }
  // the pool token total is needed on the host to bound the copy: read it (one-off, not on the path)
  uint32_t tot[2];
  IL_CUDA(cudaMemcpyAsync(&tot[0], log_off + n, 4, cudaMemcpyDeviceToHost, (cudaStream_t)s));
  IL_CUDA(cudaMemcpyAsync(&tot[1], tpl_off + n, 4, cudaMemcpyDeviceToHost, (cudaStream_t)s));
  IL_CUDA(cudaStreamSynchronize((cudaStream_t)s));
  if (tot[0] > g.max_pool_tokens || tot[1] > g.max_pool_tokens) {
    set_error("pool has more tokens than max_pool_tokens");
    return IL_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)s;
  k_reset_index<<<c->num_sms * 4, 256, 0, st>>>(*c);
  if (il_status r = records_reset(c, st)) return r;
  c->map_active = false;
  k_pool_copy<<<c->num_sms * 2, 256, 0, st>>>(*c, n, log_off, log_tok, tpl_off, tpl_tok, template_id,
                                                src_index, instr_tok, n_instr);
  k_pool_sets<<<cdiv(n, 8), 256, 0, st>>>(*c, n, log_off, log_tok);
  k_pool_scan<<<1, 1024, 0, st>>>(*c, n);
  k_pool_render<<<cdiv(n * 32, 256), 256, 0, st>>>(*c, n);
  if (il_status r = inv_build(c, n, st)) return r;
  if (n_instr / BS) k_instr_hash<<<1, 32, 0, st>>>(*c, n_instr / BS);
  IL_LAUNCH_CHECK("pool_load kernels");
  c->n_demos = n;
  c->n_instr = n_instr;
  c->n_instr_blocks = n_instr / BS;
  c->pool_loaded = true;
  c->refined = c->matched = c->index_done = c->exported = false;
  c->sel_topk = nullptr;
  c->batch = 0;
  return IL_OK;
}

il_status il_index_dump(il_ctx* c, il_stream s, uint64_t* hash_h, uint64_t* stamp_h, uint32_t* depth_h,
                        uint64_t* parent_h, uint32_t* n_h) {
  const size_t C = c->cfg.kv_pages;
  cudaStream_t st = (cudaStream_t)s;
  uint64_t *h, *sp, *pa;
  uint32_t *dp, *cnt;
  IL_CUDA(cudaMallocAsync(&h, C * 8, st)); IL_CUDA(cudaMallocAsync(&sp, C * 8, st));
  IL_CUDA(cudaMallocAsync(&pa, C * 8, st)); IL_CUDA(cudaMallocAsync(&dp, C * 4, st));
  IL_CUDA(cudaMallocAsync(&cnt, 4, st));
  IL_CUDA(cudaMemsetAsync(cnt, 0, 4, st));
  k_gather_index<<<c->num_sms, 256, 0, st>>>(*c, h, sp, dp, pa, cnt);
  uint32_t n = 0;
  IL_CUDA(cudaMemcpyAsync(&n, cnt, 4, cudaMemcpyDeviceToHost, st));
  IL_CUDA(cudaStreamSynchronize(st));
  IL_CUDA(cudaMemcpyAsync(hash_h, h, n * 8, cudaMemcpyDeviceToHost, st));
  IL_CUDA(cudaMemcpyAsync(stamp_h, sp, n * 8, cudaMemcpyDeviceToHost, st));
  IL_CUDA(cudaMemcpyAsync(depth_h, dp, n * 4, cudaMemcpyDeviceToHost, st));
  IL_CUDA(cudaMemcpyAsync(parent_h, pa, n * 8, cudaMemcpyDeviceToHost, st));
  IL_CUDA(cudaFreeAsync(h, st)); IL_CUDA(cudaFreeAsync(sp, st)); IL_CUDA(cudaFreeAsync(pa, st));
  IL_CUDA(cudaFreeAsync(dp, st)); IL_CUDA(cudaFreeAsync(cnt, st));
  IL_CUDA(cudaStreamSynchronize(st));
  *n_h = n;
  return IL_OK;
}

il_status il_table_dump(il_ctx* c, il_stream s, uint32_t* ds_h, uint64_t* stamp_h) {
  cudaStream_t st = (cudaStream_t)s;
  IL_CUDA(cudaMemcpyAsync(ds_h, c->tab_ds, (size_t)c->cfg.table_capacity * c->cfg.k * 4, cudaMemcpyDeviceToHost, st));
  IL_CUDA(cudaMemcpyAsync(stamp_h, c->tab_stamp, (size_t)c->cfg.table_capacity * 8, cudaMemcpyDeviceToHost, st));
  IL_CUDA(cudaStreamSynchronize(st));
  return IL_OK;
}

il_status il_evicted_dump(il_ctx* c, il_stream s, uint64_t* hash_h, uint32_t* n_h) {
  cudaStream_t st = (cudaStream_t)s;
  uint32_t n = 0;
  IL_CUDA(cudaMemcpyAsync(&n, &c->sc->evicted, 4, cudaMemcpyDeviceToHost, st));
  IL_CUDA(cudaStreamSynchronize(st));
  IL_CUDA(cudaMemcpyAsync(hash_h, c->evicted_list, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
  IL_CUDA(cudaStreamSynchronize(st));
  *n_h = n;
  return IL_OK;
}

}  // extern "C"
