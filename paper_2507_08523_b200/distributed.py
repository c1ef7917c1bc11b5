"""Data-parallel multi-GPU driver: one process per GPU, torch.distributed.

The hot path shards by request: rank r takes the r-th contiguous slice of every global batch,
keeps its own KV pages and prefix index, and runs the whole path on its slice.  The only
exchanges are
  (1) the demo pool, broadcast once from rank 0 (`broadcast_pool`);
  (2) per batch, one all-gather of a fixed-size record buffer per rank (il_commit_export): the
      per-request ICL records (final DS + il_refine_info), which every rank applies in global
      admission order, so the ICL Table stays replicated and every rank refines the next batch
      against the same snapshot (P:356-363 applied to the whole global batch), and the rank's
      block records (prefix-index updates), which build the replicated residency map hash ->
      owner ranks and the box-level hit counts (oracle: run_batch_dp).
Nothing else moves: no KV pages, no requests.  This module is plumbing (slicing, collectives,
argument marshalling); every step of the path runs in the library's kernels.
"""
from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import torch
import torch.distributed as dist

POOL_FIELDS = ("log_off", "log_tok", "tpl_off", "tpl_tok", "template_id", "src_index")


def slice_of(B_global: int, rank: int, world: int) -> tuple[int, int]:
    """Admission slice [lo, hi) of the global batch owned by `rank`."""
    return rank * B_global // world, (rank + 1) * B_global // world


def broadcast_pool(pool, instr, device, src: int = 0, group=None):
    """Rank `src`'s pool (CSR arrays) and instruction, delivered to every rank as numpy arrays.
    Other ranks pass pool=None, instr=None."""
    rank = dist.get_rank(group)
    if rank == src:
        arrays = [np.asarray(getattr(pool, f), np.uint32) for f in POOL_FIELDS] + [np.asarray(instr, np.uint32)]
        sizes = torch.tensor([len(a) for a in arrays], dtype=torch.int64)
    else:
        arrays, sizes = None, torch.zeros(len(POOL_FIELDS) + 1, dtype=torch.int64)
    sizes = sizes.to(device)
    dist.broadcast(sizes, src, group=group)
    n = [int(x) for x in sizes.cpu()]
    flat = torch.empty(sum(n), dtype=torch.int32, device=device)
    if rank == src:
        flat.copy_(torch.from_numpy(np.concatenate(arrays).view(np.int32)))
    dist.broadcast(flat, src, group=group)
    parts = [p.cpu().numpy().view(np.uint32) for p in torch.split(flat, n)]
    return SimpleNamespace(**dict(zip(POOL_FIELDS, parts[:-1]))), parts[-1]


def all_gather_rows(out: torch.Tensor, local: torch.Tensor, group=None) -> torch.Tensor:
    """out[r * n:(r + 1) * n] = rank r's `local` (n rows), i.e. global admission order when every
    rank holds its contiguous slice.  NCCL: one all_gather_into_tensor; other backends: all_gather."""
    world = dist.get_world_size(group)
    n = local.shape[0]
    dst = out[:world * n]
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(dst, local.contiguous(), group=group)
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous(), group=group)
        dst.copy_(torch.cat(parts))
    return dst


class DataParallel:
    """Wraps one rank's Pipeline.  Every rank must call every method (collectives); slices are
    equal-sized (the global batch is world x B).

    Per batch b the exchange is ONE all-gather of a fixed-size record buffer per rank
    (il_commit_export: the rank's ICL records + the blocks its prefix index gained or lost),
    issued on a side stream so that it overlaps batch b+1's kNN selection (il_select_batch reads
    only the pool); il_commit_apply then applies every rank's records: the replicated ICL Table
    (global admission order) and the replicated residency map (box-level hits).

        select(b+1) | all-gather(b) on the comm stream
        apply(b) -> refine(b+1) -> match -> synth -> attn -> commit_index -> export(b+1) -> ...
    """

    def __init__(self, pl, group=None):
        self.pl, self.group = pl, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        if pl.cfg.max_global_batch < self.world * pl.cfg.max_batch:
            raise ValueError("Config.max_global_batch must be >= world * max_batch")
        dev = pl.device
        self.rec_bytes = pl.cfg.record_bytes()
        self.rec = torch.zeros(self.rec_bytes, dtype=torch.uint8, device=dev)
        self.rec_all = torch.zeros(self.world * self.rec_bytes, dtype=torch.uint8, device=dev)
        self.comm = torch.cuda.Stream(dev)
        self.gathered = None          # event: the last all-gather finished (records not yet applied)
        self.pending_B = 0

    def load_pool(self, pool, instr) -> None:
        p, ins = broadcast_pool(pool if self.rank == 0 else None, instr if self.rank == 0 else None,
                                self.pl.device, 0, self.group)
        self.pl.load_pool(p, ins)

    def _main(self):
        return self.pl.stream if self.pl.stream is not None else torch.cuda.current_stream(self.pl.device)

    # ------------------------------------------------------------ stages (each capturable)
    def select(self, B=None) -> None:
        pl = self.pl
        B = pl.B if B is None else B
        pl.ctx.select_batch(B, pl.q_off, pl.q_tok, pl.q_src, pl.topk, stream=pl.stream)

    def wait_gathered(self) -> None:
        """Make the main stream wait for the pending all-gather (an event wait)."""
        if self.gathered is not None:
            self._main().wait_event(self.gathered)
            self.gathered = None

    def apply_records(self) -> None:
        """il_commit_apply of the gathered buffers (every rank's records; ends that batch).  No
        stream wait: capturable in a CUDA graph; call wait_gathered() first."""
        self.pl.ctx.commit_apply(self.rec_all, [self.pending_B] * self.world, stream=self.pl.stream)

    def apply(self) -> None:
        """Wait for the pending all-gather and apply every rank's records (ends that batch)."""
        if self.gathered is None:
            return
        self.wait_gathered()
        self.apply_records()

    def export(self, B=None) -> None:
        """il_commit_index + il_commit_export of this rank's batch into its record buffer."""
        pl = self.pl
        pl.ctx.commit_index(stream=pl.stream)
        pl.ctx.commit_export(self.rec, stream=pl.stream)
        self.pending_B = pl.B if B is None else B

    def gather(self) -> None:
        """All-gather the record buffers (rank-major) on the comm stream, after the export."""
        main = self._main()
        ev = torch.cuda.Event()
        ev.record(main)
        self.comm.wait_event(ev)
        with torch.cuda.stream(self.comm):
            all_gather_rows(self.rec_all.view(self.world, -1), self.rec.view(1, -1), self.group)
            done = torch.cuda.Event()
            done.record(self.comm)
        self.gathered = done

    def commit(self, B=None) -> None:
        """The whole exchange for this batch, not overlapped: export, all-gather, apply."""
        self.export(B)
        self.gather()
        self.apply()

    def step(self, B=None, attention: bool = True) -> None:
        """One batch, pipelined with the previous batch's exchange; call flush() after the last."""
        pl = self.pl
        self.select(B)
        self.apply()
        pl.refine(B)
        pl.match(B)
        if attention:
            pl.synth(B)
            pl.attn(B)
        self.export(B)
        self.gather()

    def flush(self) -> None:
        self.apply()


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
