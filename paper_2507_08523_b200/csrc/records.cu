// records.cu — the multi-GPU exchange of SURVEY §8(e) as one fixed-size record buffer per rank
// (il.h il_record_bytes / il_commit_export / il_commit_apply): the rank's ICL records (P:356-363,
// applied to the replicated table in global admission order) and its prefix-index updates
// (block records: every chain hash its index gained or lost), which build the replicated
// residency map hash -> owner-rank bitmask, the "shared prefix index" of BASELINE configs[2].
// Also il_select_batch (a1-a2 alone, so the record all-gather can overlap it).
#include <cooperative_groups.h>

#include <algorithm>

#include "il_internal.cuh"

namespace cg = cooperative_groups;

namespace il {

// One CTA.  (1) this batch's block records -- evicted hashes (il_prefix_match) then newly
// resident hashes (il_commit_index) -- are appended to the context's FIFO; (2) up to rec_R of
// the oldest records are popped into the buffer; (3) the ICL records of the batch are copied.
__global__ void __launch_bounds__(1024) k_export(Ctx c, uint8_t* __restrict__ rec, uint32_t B) {
  DevScalars* sc = c.sc;
  const uint32_t tid = threadIdx.x, k = c.cfg.k;
  const uint32_t n_ev = sc->evicted, n_in = sc->inserted;
  const uint64_t head = sc->ring_head, tail = sc->ring_tail;
  const uint64_t cap = c.ring_cap;
  if (tail + n_ev + n_in - head > cap) {                   // FIFO overflow: uniform branch
    if (tid == 0) latch(sc, IL_ERR_CAPACITY);
    return;
  }
  for (uint32_t x = tid; x < n_ev; x += blockDim.x) c.ring[(tail + x) % cap] = c.evicted_list[x];
  for (uint32_t x = tid; x < n_in; x += blockDim.x) c.ring[(tail + n_ev + x) % cap] = c.ins_list[x];
  const uint64_t tail2 = tail + n_ev + n_in;
  const uint64_t pend = tail2 - head;
  const uint32_t n_out = (uint32_t)(pend < c.rec_R ? pend : c.rec_R);
  uint64_t* blk = reinterpret_cast<uint64_t*>(rec + rec_blk_off(c.cfg.max_batch, k));
  __syncthreads();                                         // ring writes before the pops below
  for (uint32_t x = tid; x < n_out; x += blockDim.x) blk[x] = c.ring[(head + x) % cap];
  uint32_t* fds = reinterpret_cast<uint32_t*>(rec + rec_fds_off());
  il_refine_info* inf = reinterpret_cast<il_refine_info*>(rec + rec_info_off(c.cfg.max_batch, k));
  if (c.final_ds)
    for (uint32_t x = tid; x < B * k; x += blockDim.x) fds[x] = c.final_ds[x];
  if (c.info)
    for (uint32_t x = tid; x < B; x += blockDim.x) inf[x] = c.info[x];
  if (tid == 0) {
    RecHeader h{};
    h.magic = REC_MAGIC; h.B = B; h.k = k; h.n_blk = n_out;
    h.batch = sc->batch_done + 1;
    h.backlog = (uint32_t)(tail2 - head - n_out);
    *reinterpret_cast<RecHeader*>(rec) = h;
    sc->ring_head = head + n_out;
    sc->ring_tail = tail2;
  }
}

struct RankOffsets { uint32_t off[33]; };

// The ICL records of every rank, rank-major = global admission order, into one contiguous array
// (what the table commit consumes).  A buffer whose header disagrees with the host's batch sizes
// latches IL_ERR_ARG and contributes nothing.
__global__ void k_gather_icl(Ctx c, const uint8_t* __restrict__ recs, size_t rec_bytes, uint32_t n_ranks,
                             RankOffsets ro) {
  const uint32_t k = c.cfg.k;
  const uint32_t r = blockIdx.y;
  const uint8_t* rec = recs + (size_t)r * rec_bytes;
  const RecHeader* h = reinterpret_cast<const RecHeader*>(rec);
  const uint32_t B = ro.off[r + 1] - ro.off[r];
  if (h->magic != REC_MAGIC || h->B != B || h->k != k) {
    if (blockIdx.x == 0 && threadIdx.x == 0) latch(c.sc, IL_ERR_ARG);
    return;
  }
  const uint32_t* fds = reinterpret_cast<const uint32_t*>(rec + rec_fds_off());
  const il_refine_info* inf = reinterpret_cast<const il_refine_info*>(rec + rec_info_off(c.cfg.max_batch, k));
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < B * k; x += gridDim.x * blockDim.x)
    c.icl_fds[(size_t)ro.off[r] * k + x] = fds[x];
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < B; x += gridDim.x * blockDim.x)
    c.icl_info[ro.off[r] + x] = inf[x];
}

// Block records -> residency map.  Rank r's record toggles bit r of the hash's mask: a rank's
// index gains and loses a given hash strictly alternately, so after any set of complete record
// windows the bit equals "resident on rank r" whatever order the toggles were applied in.
// Open addressing with lock-free CAS of EMPTY slots; a key whose mask returns to 0 stays as a
// dead key (a later insert revives it) until the rebuild compacts the table.
__global__ void k_map_apply(Ctx c, const uint8_t* __restrict__ recs, size_t rec_bytes, uint32_t n_ranks) {
  const uint32_t r = blockIdx.y;
  const uint8_t* rec = recs + (size_t)r * rec_bytes;
  const RecHeader* h = reinterpret_cast<const RecHeader*>(rec);
  if (h->magic != REC_MAGIC) return;                       // (k_gather_icl latched)
  const uint32_t n = min(h->n_blk, c.rec_R);
  const uint64_t* blk = reinterpret_cast<const uint64_t*>(rec + rec_blk_off(c.cfg.max_batch, c.cfg.k));
  uint32_t fresh = 0;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    const uint64_t key = blk[x];
    uint32_t s = (uint32_t)(key ^ (key >> 32)) & c.map_smask;
    while (true) {
      const uint64_t cur = c.map_key[s];
      if (cur == key) break;
      if (cur == KEY_EMPTY) {
        const uint64_t old = atomicCAS((unsigned long long*)&c.map_key[s], (unsigned long long)KEY_EMPTY,
                                       (unsigned long long)key);
        if (old == KEY_EMPTY) { ++fresh; break; }
        if (old == key) break;
      }
      s = (s + 1) & c.map_smask;
    }
    atomicXor(&c.map_mask[s], 1u << r);
  }
  for (int o = 16; o; o >>= 1) fresh += __shfl_xor_sync(~0u, fresh, o);
  if ((threadIdx.x & 31) == 0 && fresh) atomicAdd(&c.sc->map_used, fresh);
}

// Compaction when more than half the slots hold a key: live entries (mask != 0) are copied out,
// the table cleared and the live entries re-inserted (one cooperative grid).
__global__ void __launch_bounds__(512) k_map_rebuild(Ctx c) {
  cg::grid_group grid = cg::this_grid();
  DevScalars* sc = c.sc;
  if ((uint64_t)sc->map_used * 2 <= c.map_slots) return;  // uniform
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  grid.sync();                                             // every CTA has read map_used
  if (gtid == 0) sc->map_used = 0;
  grid.sync();
  for (uint32_t s = gtid; s < c.map_slots; s += gs) {
    const uint64_t key = c.map_key[s];
    const uint32_t m = c.map_mask[s];
    if (key != KEY_EMPTY && m != 0) {
      const uint32_t e = atomicAdd(&sc->map_used, 1u);     // map_used counts live entries here
      c.map_tmp_key[e] = key;
      c.map_tmp_mask[e] = m;
    }
  }
  grid.sync();
  for (uint32_t s = gtid; s < c.map_slots; s += gs) { c.map_key[s] = KEY_EMPTY; c.map_mask[s] = 0; }
  grid.sync();
  const uint32_t live = sc->map_used;
  for (uint32_t e = gtid; e < live; e += gs) {
    const uint64_t key = c.map_tmp_key[e];
    uint32_t s = (uint32_t)(key ^ (key >> 32)) & c.map_smask;
    while (atomicCAS((unsigned long long*)&c.map_key[s], (unsigned long long)KEY_EMPTY, (unsigned long long)key) !=
           KEY_EMPTY)
      s = (s + 1) & c.map_smask;
    c.map_mask[s] = c.map_tmp_mask[e];
  }
  if (gtid == 0) sc->map_rebuilds += 1;
}

__global__ void k_map_reset(Ctx c) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < c.map_slots; s += stride) {
    c.map_key[s] = KEY_EMPTY; c.map_mask[s] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c.sc->map_used = 0; c.sc->ring_head = 0; c.sc->ring_tail = 0;
  }
}

}  // namespace il

using namespace il;

il_status il::records_setup(Ctx* c) {
  if (!c->map_slots) return IL_OK;
  int per_sm = 0;
  IL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_map_rebuild, 512, 0));
  c->mb_per_sm = std::max(1, std::min(per_sm, 2));
  c->mb_blocks = c->mb_per_sm * c->num_sms;
  return IL_OK;
}

// (also called by il_pool_load: the map describes this pool's blocks)
il_status il::records_reset(Ctx* c, cudaStream_t st) {
  if (!c->map_slots) return IL_OK;
  k_map_reset<<<c->num_sms * 4, 256, 0, st>>>(*c);
  IL_LAUNCH_CHECK("k_map_reset");
  c->launches += 1;
  return IL_OK;
}

extern "C" il_status il_record_bytes(const il_config* g, size_t* bytes) {
  if (!g || !bytes) { set_error("null argument"); return IL_ERR_ARG; }
  const uint32_t R = g->max_block_records ? g->max_block_records : 16 * g->max_batch;
  *bytes = rec_bytes(g->max_batch, g->k, R);
  return IL_OK;
}

extern "C" il_status il_commit_export(il_ctx* c, void* rec, il_stream s) {
  if (!c->map_slots) { set_error("il_commit_export needs max_global_batch > max_batch"); return IL_ERR_STATE; }
  if (!c->index_done || c->exported) { set_error("il_commit_export: call once, after il_commit_index"); return IL_ERR_STATE; }
  if (!rec || ((uintptr_t)rec & 15)) { set_error("record buffer null or not 16-byte aligned"); return IL_ERR_ARG; }
  k_export<<<1, 1024, 0, (cudaStream_t)s>>>(*c, (uint8_t*)rec, c->last_B);
  IL_LAUNCH_CHECK("k_export");
  c->launches += 1;
  c->exported = true;
  return IL_OK;
}

extern "C" il_status il_commit_apply(il_ctx* c, const void* recs, uint32_t n_ranks, const uint32_t* bpr,
                                     il_stream s) {
  if (!c->exported) { set_error("il_commit_apply before il_commit_export"); return IL_ERR_STATE; }
  if (n_ranks < 1 || n_ranks > c->n_ranks_max || !bpr || !recs) {
    set_error("il_commit_apply: n_ranks must be in [1, ceil(max_global_batch / max_batch)]");
    return IL_ERR_ARG;
  }
  RankOffsets ro{};
  for (uint32_t r = 0; r < n_ranks; ++r) {
    if (bpr[r] > c->cfg.max_batch) { set_error("batch_per_rank > max_batch"); return IL_ERR_ARG; }
    ro.off[r + 1] = ro.off[r] + bpr[r];
  }
  const uint32_t Bg = ro.off[n_ranks];
  if (Bg > c->max_records) { set_error("sum of batch_per_rank > max_global_batch"); return IL_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)s;
  const size_t rb = rec_bytes(c->cfg.max_batch, c->cfg.k, c->rec_R);
  const uint8_t* r8 = (const uint8_t*)recs;
  k_gather_icl<<<dim3(8, n_ranks), 256, 0, st>>>(*c, r8, rb, n_ranks, ro);
  k_map_apply<<<dim3(std::max(1u, cdiv(c->rec_R, 256u * 8u)), n_ranks), 256, 0, st>>>(*c, r8, rb, n_ranks);
  {
    Ctx cc = *c;
    void* args[] = {&cc};
    IL_CUDA(cudaLaunchCooperativeKernel((void*)k_map_rebuild, dim3(c->mb_blocks), dim3(512), args, 0, st));
  }
  IL_LAUNCH_CHECK("il_commit_apply (records)");
  c->launches += 3;
  if (n_ranks > 1) c->map_active = true;
  if (c->cfg.flags & IL_F_PAIR) {
    il_status r = commit_table(c, Bg, c->icl_fds, c->icl_info, st, c->batch + 1);
    if (r != IL_OK) return r;
  }
  return end_batch(c, st);
}

extern "C" il_status il_box_hit_dump(il_ctx* c, il_stream s, uint32_t* out_h, uint32_t B) {
  if (B > c->cfg.max_batch) { set_error("B > max_batch"); return IL_ERR_ARG; }
  if (!c->box_hit || !c->map_active) {
    for (uint32_t i = 0; i < B; ++i) out_h[i] = 0;
    return IL_OK;
  }
  IL_CUDA(cudaMemcpyAsync(out_h, c->box_hit, (size_t)B * 4, cudaMemcpyDeviceToHost, (cudaStream_t)s));
  IL_CUDA(cudaStreamSynchronize((cudaStream_t)s));
  return IL_OK;
}
