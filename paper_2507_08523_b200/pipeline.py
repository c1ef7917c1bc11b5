"""Batch driver: one pass of the hot path over one batch of concurrent requests.

    il_refine_batch -> il_prefix_match -> (il_synth_qkv: stands in for the QKV projection)
    -> il_prefill_attn -> il_commit

All buffers are preallocated for the configured maxima (PyTorch memory); all calls are
asynchronous on one stream; nothing is copied back to the host in steady state.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .context import Config, Context, INFO_DTYPE


def _dev_u32(a, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.uint32)).view(np.int32)).to(device)


class Pipeline:
    def __init__(self, cfg: Config, device="cuda", qkv_seed: int = 3000, q_scale: float = 1.0,
                 max_query_tokens: int | None = None, stream: torch.cuda.Stream | None = None,
                 fused_kv: bool = False, slots: int = 1):
        self.cfg = cfg
        self.device = torch.device(device)
        self.stream = stream
        self.ctx = Context(cfg, self.device, stream)
        self.qkv_seed, self.q_scale = qkv_seed, q_scale
        # fused_kv: the projection stand-in writes K / V straight into the pages (il_synth_qkv_paged)
        # and il_prefill_attn skips its append pass
        self.fused_kv = fused_kv
        B, S, MB, k = cfg.max_batch, cfg.max_prompt_tokens, cfg.max_blocks, cfg.k
        dev, i32 = self.device, torch.int32
        rows = cfg.max_suffix_tokens or B * S
        Hq, Hkv, d = cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
        bf = torch.bfloat16
        mq = max_query_tokens or B * cfg.max_log_tokens
        self._rows = rows
        # per-batch buffers; `slots` > 1 gives every slot its own set, so that the attention of one
        # batch can run while the integer stages of the next use the other slot (il.h: cross-batch
        # pipelining; `use(slot)` selects the set the calls below read and write)
        self._slots = []
        for _ in range(slots):
            self._slots.append(dict(
                topk=torch.zeros(B, k, dtype=i32, device=dev),
                final_ds=torch.zeros(B, k, dtype=i32, device=dev),
                info=torch.zeros(B, 16, dtype=torch.uint8, device=dev),
                prompt_tok=torch.zeros(B, S, dtype=i32, device=dev),
                prompt_len=torch.zeros(B, dtype=i32, device=dev),
                block_hash=torch.zeros(B, MB, dtype=torch.int64, device=dev),
                hit=torch.zeros(B, dtype=i32, device=dev),
                block_table=torch.zeros(B, MB, dtype=i32, device=dev),
                prefix_len=torch.zeros(B, dtype=i32, device=dev),
                cu_q=torch.zeros(B + 1, dtype=i32, device=dev),
                q=torch.empty(rows, Hq, d, dtype=bf, device=dev),
                # (the append path's K / V buffers only when the projection does not write the pages)
                k_new=None if fused_kv else torch.empty(rows, Hkv, d, dtype=bf, device=dev),
                v_new=None if fused_kv else torch.empty(rows, Hkv, d, dtype=bf, device=dev),
                out=torch.empty(rows, Hq, d, dtype=bf, device=dev),
                lse=torch.empty(rows, Hq, dtype=torch.float32, device=dev),
                q_off=torch.zeros(B + 1, dtype=i32, device=dev),
                q_tok=torch.zeros(mq, dtype=i32, device=dev),
                q_src=torch.zeros(B, dtype=i32, device=dev)))
        self.use(0)
        self.k_pages = torch.zeros(cfg.kv_pages, Hkv, 16, d, dtype=bf, device=dev)
        self.v_pages = torch.zeros(cfg.kv_pages, Hkv, 16, d, dtype=bf, device=dev)
        self.scale = d ** -0.5
        self.B = 0

    def use(self, slot: int) -> None:
        """Select the per-batch buffer set the following calls use."""
        for name, t in self._slots[slot].items():
            setattr(self, name, t)
        self.slot = slot

    def _append_buffers(self) -> None:
        if self.k_new is None:                          # (fused_kv switched off after construction)
            cfg, sl = self.cfg, self._slots[self.slot]
            for name in ("k_new", "v_new"):
                sl[name] = torch.empty(self._rows, cfg.n_kv_heads, cfg.head_dim, dtype=torch.bfloat16,
                                       device=self.device)
            self.use(self.slot)

    # -------------------------------------------------------------- inputs
    def load_pool(self, pool, instr) -> None:
        dev = self.device
        t = [_dev_u32(x, dev) for x in (pool.log_off, pool.log_tok, pool.tpl_off, pool.tpl_tok,
                                        pool.template_id, pool.src_index, instr)]
        self.ctx.pool_load(*t, stream=self.stream)
        self._pool_keepalive = t
        self.ctx.status_sync(self.stream)

    def stage_batch(self, batch) -> None:
        """Copy one batch of query logs into the resident input buffers (host -> device)."""
        B = batch.B
        n = int(batch.q_off[-1])
        self.q_off[:B + 1].copy_(torch.from_numpy(batch.q_off.view(np.int32)), non_blocking=True)
        self.q_tok[:n].copy_(torch.from_numpy(batch.q_tok.view(np.int32)), non_blocking=True)
        self.q_src[:B].copy_(torch.from_numpy(batch.q_src.view(np.int32)), non_blocking=True)
        self.B = B

    # -------------------------------------------------------------- the path
    def select(self, B=None) -> None:
        """a1-a2 alone (il_select_batch); a following refine() of the same batch skips it."""
        B = self.B if B is None else B
        self.ctx.select_batch(B, self.q_off, self.q_tok, self.q_src, self.topk, stream=self.stream)

    def refine(self, B=None) -> None:
        B = self.B if B is None else B
        self.ctx.refine_batch(B, self.q_off, self.q_tok, self.q_src, self.topk, self.final_ds, self.info,
                              self.prompt_tok, self.prompt_len, stream=self.stream)

    def match(self, B=None) -> None:
        B = self.B if B is None else B
        self.ctx.prefix_match(B, self.prompt_tok, self.prompt_len, self.block_hash, self.hit,
                              self.block_table, self.prefix_len, self.cu_q, stream=self.stream)

    def synth(self, B=None, part: str = "qkv") -> None:
        """The QKV-projection stand-in; part = "q" / "kv" writes only Q / only K and V (fused_kv:
        the pipelined schedule writes the next batch's Q before this batch's attention ends)."""
        B = self.B if B is None else B
        if self.fused_kv:
            q = None if part == "kv" else self.q
            kp, vp = (None, None) if part == "q" else (self.k_pages, self.v_pages)
            self.ctx.synth_qkv_paged(B, self.prompt_tok, self.cu_q, self.prefix_len, self.block_table, self.qkv_seed,
                                     self.q_scale, q, kp, vp, stream=self.stream)
            return
        assert part == "qkv", "split synth needs fused_kv"
        self._append_buffers()
        self.ctx.synth_qkv(B, self.prompt_tok, self.cu_q, self.prefix_len, self.qkv_seed, self.q_scale,
                           self.q, self.k_new, self.v_new, stream=self.stream)

    def attn(self, B=None, lse: bool = True) -> None:
        B = self.B if B is None else B
        if not self.fused_kv:
            self._append_buffers()
        kn, vn = (None, None) if self.fused_kv else (self.k_new, self.v_new)
        self.ctx.prefill_attn(B, self.cu_q, self.prefix_len, self.block_table, self.q, kn, vn,
                              self.k_pages, self.v_pages, self.out, self.lse if lse else None, self.scale,
                              stream=self.stream)

    def commit(self, B=None) -> None:
        self.ctx.commit(stream=self.stream)

    # -------------------------------------------------------------- CUDA graphs
    STAGES = ("refine", "match", "synth", "attn", "commit")

    def capture(self, B: int, stages=STAGES) -> dict:
        """Capture each stage for batch size B as a CUDA graph (one replay per stage removes the
        per-kernel launch gaps).  The graphs read the pipeline's own input buffers (stage the
        batch with stage_batch / load_inputs first) and every device state they touch (batch
        counter, index, table) lives on the device, so replays advance the stream like eager
        calls.  Call after at least one eager step (one-time function attributes)."""
        own = self.stream
        s = own if own is not None else torch.cuda.Stream(self.device)   # capture needs a side stream
        s.wait_stream(torch.cuda.current_stream(self.device))
        self.stream = s                                 # the library launches on the capture stream
        self.graphs = {}
        try:
            for name in stages:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    getattr(self, name)(B)
                self.graphs[name] = g
        finally:
            self.stream = own
        return self.graphs

    def load_inputs(self, q_off: torch.Tensor, q_tok: torch.Tensor, q_src: torch.Tensor, B: int) -> None:
        """Device-to-device copy of one batch's query CSR into the resident input buffers."""
        self.q_off[:B + 1].copy_(q_off[:B + 1], non_blocking=True)
        self.q_tok[:q_tok.numel()].copy_(q_tok, non_blocking=True)
        self.q_src[:B].copy_(q_src[:B], non_blocking=True)
        self.B = B

    # -------------------------------------------------------------- decode
    def decode_step(self, t: int, tokens: torch.Tensor, B=None, lse: bool = True) -> None:
        """Decode token t of every request (after il_prefill_attn, before il_commit; needs
        Config.max_decode_tokens > t): tokens[i] is written at position L_i + t of the prompt
        row, its Q / K / V come from il_synth_qkv (the QKV-projection stand-in) and il_decode_attn
        runs ONE row per request at position L_i + t: its K / V go into the reserved decode page,
        attention covers the prompt and the t decode tokens before it.  Output: dec_out[:B]."""
        B = self.B if B is None else B
        dev = self.device
        if not hasattr(self, "dec_q"):
            cfg, rows = self.cfg, self.cfg.max_batch + 256       # (whole 128-row Q tiles stay in bounds)
            bf = torch.bfloat16
            self.dec_q = torch.zeros(rows, cfg.n_q_heads, cfg.head_dim, dtype=bf, device=dev)
            self.dec_k = torch.zeros(rows, cfg.n_kv_heads, cfg.head_dim, dtype=bf, device=dev)
            self.dec_v = torch.zeros(rows, cfg.n_kv_heads, cfg.head_dim, dtype=bf, device=dev)
            self.dec_out = torch.zeros(rows, cfg.n_q_heads, cfg.head_dim, dtype=bf, device=dev)
            self.dec_lse = torch.zeros(rows, cfg.n_q_heads, dtype=torch.float32, device=dev)
            self.dec_cu = torch.arange(cfg.max_batch + 1, dtype=torch.int32, device=dev)
            self.dec_pos = torch.zeros(cfg.max_batch, dtype=torch.int32, device=dev)
        s = self.stream if self.stream is not None else torch.cuda.current_stream(dev)
        with torch.cuda.stream(s):
            pos = self.prompt_len[:B] + t
            self.dec_pos[:B].copy_(pos)
            self.prompt_tok.view(-1)[torch.arange(B, device=dev) * self.prompt_tok.shape[1] + pos] = tokens[:B].to(torch.int32)
        self.ctx.synth_qkv(B, self.prompt_tok, self.dec_cu, self.dec_pos, self.qkv_seed, self.q_scale,
                           self.dec_q, self.dec_k, self.dec_v, stream=self.stream)
        self.ctx.decode_attn(B, self.dec_pos, self.block_table, self.dec_q, self.dec_k, self.dec_v,
                             self.k_pages, self.v_pages, self.dec_out, self.dec_lse if lse else None, self.scale,
                             stream=self.stream)

    def launches(self) -> int:
        """Kernels this context has launched so far (host-side counter in the library)."""
        return int(self.ctx.stats(self.stream)["launches"])

    def step(self, B=None, attention: bool = True) -> None:
        self.refine(B)
        self.match(B)
        if attention:
            self.synth(B)
            self.attn(B)
        self.commit()

    # -------------------------------------------------------------- readback (tests / metrics)
    def info_np(self, B=None) -> np.ndarray:
        B = self.B if B is None else B
        return self.info[:B].cpu().numpy().reshape(-1).view(INFO_DTYPE)

    def u32(self, t: torch.Tensor) -> np.ndarray:
        return t.cpu().numpy().view(np.uint32)
