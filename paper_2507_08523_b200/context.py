"""Thin Python binding over the C ABI (include/il.h): same names, argument marshalling only.

PyTorch provides device memory and the stream; every step of the path runs in the CUDA
kernels of libinferlog_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L


@dataclass
class Config:
    k: int
    table_capacity: int
    kv_pages: int
    max_batch: int
    max_prompt_tokens: int
    max_pool: int
    max_pool_tokens: int
    max_log_tokens: int = 255
    max_suffix_tokens: int = 0          # 0 -> max_batch * max_prompt_tokens
    n_q_heads: int = 32
    n_kv_heads: int = 8
    head_dim: int = 128
    metric: int = L.IL_SIM_COSINE
    flags: int = L.IL_F_PAIR | L.IL_F_VERIFY
    hash_seed: int = 0
    max_global_batch: int = 0           # multi-GPU: world * max_batch records per table commit
    max_block_records: int = 0          # multi-GPU: block records per export (0 = 16 * max_batch)
    max_decode_tokens: int = 0          # KV pages reserved per request for decode tokens (NEXT-4)

    @property
    def max_blocks(self) -> int:
        return (self.max_prompt_tokens + 15) // 16

    def c(self) -> L.il_config:
        m = self.max_suffix_tokens or self.max_batch * self.max_prompt_tokens
        return L.il_config(self.k, self.table_capacity, self.kv_pages, self.max_batch,
                           self.max_prompt_tokens, self.max_pool, self.max_pool_tokens,
                           self.max_log_tokens, m, self.n_q_heads, self.n_kv_heads, self.head_dim,
                           self.metric, self.flags, self.hash_seed, self.max_global_batch,
                           self.max_block_records, self.max_decode_tokens, 0)

    def record_bytes(self) -> int:
        cc = self.c()
        n = C.c_size_t(0)
        L.check(L.load().il_record_bytes(C.byref(cc), C.byref(n)), "il_record_bytes")
        return int(n.value)


def _p(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream(stream=None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class Context:
    """One il_ctx on one GPU (single writer)."""

    def __init__(self, cfg: Config, device=None, stream=None):
        self.cfg = cfg
        self.lib = L.load()
        self.device = torch.device(device if device is not None else "cuda")
        cc = cfg.c()
        nbytes = C.c_size_t(0)
        L.check(self.lib.il_workspace_bytes(C.byref(cc), C.byref(nbytes)), "il_workspace_bytes")
        self.workspace = torch.empty(nbytes.value + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        aligned = (base + 255) & ~255
        h = C.c_void_p()
        L.check(self.lib.il_create(C.byref(cc), C.c_void_p(aligned), nbytes.value, _stream(stream), C.byref(h)),
                "il_create")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.il_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ calls
    def pool_load(self, log_off, log_tok, tpl_off, tpl_tok, template_id, src_index, instr, stream=None):
        L.check(self.lib.il_pool_load(self.h, int(template_id.numel()), _p(log_off), _p(log_tok), _p(tpl_off),
                                      _p(tpl_tok), _p(template_id), _p(src_index), _p(instr),
                                      int(instr.numel()), _stream(stream)), "il_pool_load")

    def refine_batch(self, B, q_off, q_tok, q_src, topk, final_ds, info, prompt_tok, prompt_len, stream=None):
        L.check(self.lib.il_refine_batch(self.h, B, _p(q_off), _p(q_tok), _p(q_src), _p(topk), _p(final_ds),
                                         _p(info), _p(prompt_tok), _p(prompt_len), _stream(stream)),
                "il_refine_batch")

    def prefix_match(self, B, prompt_tok, prompt_len, block_hash, hit_blocks, block_table, prefix_len, cu_q,
                     stream=None):
        L.check(self.lib.il_prefix_match(self.h, B, _p(prompt_tok), _p(prompt_len), _p(block_hash),
                                         _p(hit_blocks), _p(block_table), _p(prefix_len), _p(cu_q),
                                         _stream(stream)), "il_prefix_match")

    def prefill_attn(self, B, cu_q, prefix_len, block_table, q, k_new, v_new, k_pages, v_pages, out, lse,
                     scale, stream=None):
        L.check(self.lib.il_prefill_attn(self.h, B, _p(cu_q), _p(prefix_len), _p(block_table), _p(q),
                                         _p(k_new), _p(v_new), _p(k_pages), _p(v_pages), _p(out), _p(lse),
                                         float(scale), _stream(stream)), "il_prefill_attn")

    def decode_attn(self, B, pos, block_table, q, k_new, v_new, k_pages, v_pages, out, lse, scale, stream=None):
        L.check(self.lib.il_decode_attn(self.h, B, _p(pos), _p(block_table), _p(q), _p(k_new), _p(v_new),
                                        _p(k_pages), _p(v_pages), _p(out), _p(lse), float(scale), _stream(stream)),
                "il_decode_attn")

    def commit(self, stream=None):
        L.check(self.lib.il_commit(self.h, _stream(stream)), "il_commit")

    def commit_index(self, stream=None):
        L.check(self.lib.il_commit_index(self.h, _stream(stream)), "il_commit_index")

    def commit_records(self, B_global, final_ds_all, info_all, stream=None):
        L.check(self.lib.il_commit_records(self.h, B_global, _p(final_ds_all), _p(info_all), _stream(stream)),
                "il_commit_records")

    def commit_export(self, rec, stream=None):
        L.check(self.lib.il_commit_export(self.h, _p(rec), _stream(stream)), "il_commit_export")

    def commit_apply(self, recs_all, batch_per_rank, stream=None):
        bpr = (C.c_uint32 * len(batch_per_rank))(*[int(x) for x in batch_per_rank])
        L.check(self.lib.il_commit_apply(self.h, _p(recs_all), len(batch_per_rank), bpr, _stream(stream)),
                "il_commit_apply")

    def select_batch(self, B, q_off, q_tok, q_src, topk, stream=None):
        L.check(self.lib.il_select_batch(self.h, B, _p(q_off), _p(q_tok), _p(q_src), _p(topk), _stream(stream)),
                "il_select_batch")

    def box_hit_dump(self, B, stream=None) -> np.ndarray:
        out = np.zeros(max(B, 1), np.uint32)
        L.check(self.lib.il_box_hit_dump(self.h, _stream(stream), out.ctypes.data_as(C.c_void_p), B),
                "il_box_hit_dump")
        return out[:B]

    def synth_qkv(self, B, prompt_tok, cu_q, prefix_len, seed, q_scale, q, k_new, v_new, stream=None):
        L.check(self.lib.il_synth_qkv(self.h, B, _p(prompt_tok), _p(cu_q), _p(prefix_len), int(seed),
                                      float(q_scale), _p(q), _p(k_new), _p(v_new), _stream(stream)),
                "il_synth_qkv")

    def synth_qkv_paged(self, B, prompt_tok, cu_q, prefix_len, block_table, seed, q_scale, q, k_pages, v_pages,
                        stream=None):
        L.check(self.lib.il_synth_qkv_paged(self.h, B, _p(prompt_tok), _p(cu_q), _p(prefix_len), _p(block_table),
                                            int(seed), float(q_scale), _p(q), _p(k_pages), _p(v_pages),
                                            _stream(stream)), "il_synth_qkv_paged")

    def status_sync(self, stream=None):
        L.check(self.lib.il_status_sync(self.h, _stream(stream)), "device status")

    def stats(self, stream=None) -> dict:
        st = L.il_stats()
        L.check(self.lib.il_stats_sync(self.h, _stream(stream), C.byref(st)), "il_stats_sync")
        return {f: getattr(st, f) for f, _ in L.il_stats._fields_}

    def set_sm_split(self, attn_ctas: int) -> None:
        """il_set_sm_split: the attention's persistent grid on attn_ctas SMs, the cooperative
        integer kernels sized for the rest (cross-batch pipelining); 0 = default."""
        L.check(self.lib.il_set_sm_split(self.h, attn_ctas), "il_set_sm_split")

    def stats_async(self, out: torch.Tensor, stream=None):
        """il_stats written by a kernel into `out` (a device tensor of >= 48 bytes; no sync)."""
        L.check(self.lib.il_stats_async(self.h, _p(out), _stream(stream)), "il_stats_async")

    @staticmethod
    def stats_from_bytes(raw: np.ndarray) -> dict:
        st = L.il_stats.from_buffer_copy(np.ascontiguousarray(raw, np.uint8).tobytes()[:C.sizeof(L.il_stats)])
        return {f: getattr(st, f) for f, _ in L.il_stats._fields_}

    def index_dump(self, stream=None):
        n = self.cfg.kv_pages
        h = np.zeros(n, np.uint64); s = np.zeros(n, np.uint64); d = np.zeros(n, np.uint32)
        p = np.zeros(n, np.uint64); cnt = np.zeros(1, np.uint32)
        L.check(self.lib.il_index_dump(self.h, _stream(stream), h.ctypes.data_as(C.c_void_p),
                                       s.ctypes.data_as(C.c_void_p), d.ctypes.data_as(C.c_void_p),
                                       p.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p)),
                "il_index_dump")
        m = int(cnt[0])
        order = np.argsort(h[:m], kind="stable")
        return h[:m][order], s[:m][order], d[:m][order], p[:m][order]

    def table_dump(self, stream=None):
        T, k = self.cfg.table_capacity, self.cfg.k
        ds = np.zeros((T, k), np.uint32); st = np.zeros(T, np.uint64)
        L.check(self.lib.il_table_dump(self.h, _stream(stream), ds.ctypes.data_as(C.c_void_p),
                                       st.ctypes.data_as(C.c_void_p)), "il_table_dump")
        live = st != 0
        order = np.argsort(st[live], kind="stable")
        return ds[live][order], st[live][order]

    def evicted_dump(self, stream=None):
        h = np.zeros(self.cfg.kv_pages, np.uint64); n = np.zeros(1, np.uint32)
        L.check(self.lib.il_evicted_dump(self.h, _stream(stream), h.ctypes.data_as(C.c_void_p),
                                         n.ctypes.data_as(C.c_void_p)), "il_evicted_dump")
        return np.sort(h[:int(n[0])])


INFO_DTYPE = np.dtype([("target_stamp", "<u8"), ("target_slot", "<i4"), ("pmc", "u1"), ("rule", "u1"),
                       ("reverted", "u1"), ("matched", "u1")])
