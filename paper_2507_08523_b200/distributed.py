"""Data-parallel multi-GPU driver: one process per GPU, torch.distributed.

The hot path shards by request: rank r takes the r-th contiguous slice of every global batch,
keeps its own KV pages and prefix index, and runs the whole path on its slice.  The only
exchanges are
  (1) the demo pool, broadcast once from rank 0 (`broadcast_pool`);
  (2) per batch, one all-gather of the per-request ICL records (final DS + il_refine_info),
      which every rank applies in global admission order (il_commit_records), so the ICL Table
      stays replicated and every rank refines the next batch against the same snapshot
      (P:356-363 applied to the whole global batch; oracle: run_batch_dp).
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
    equal-sized (the global batch is world x B)."""

    def __init__(self, pl, group=None):
        self.pl, self.group = pl, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        if pl.cfg.max_global_batch < self.world * pl.cfg.max_batch:
            raise ValueError("Config.max_global_batch must be >= world * max_batch")
        B, k, dev = pl.cfg.max_batch, pl.cfg.k, pl.device
        self.final_ds_all = torch.zeros(self.world * B, k, dtype=torch.int32, device=dev)
        self.info_all = torch.zeros(self.world * B, 16, dtype=torch.uint8, device=dev)

    def load_pool(self, pool, instr) -> None:
        p, ins = broadcast_pool(pool if self.rank == 0 else None, instr if self.rank == 0 else None,
                                self.pl.device, 0, self.group)
        self.pl.load_pool(p, ins)

    def commit(self, B=None) -> None:
        """il_commit_index, all-gather of the ICL records, il_commit_records (global order)."""
        pl = self.pl
        B = pl.B if B is None else B
        pl.ctx.commit_index(stream=pl.stream)
        with torch.cuda.stream(pl.stream) if pl.stream is not None else _nullctx():
            all_gather_rows(self.final_ds_all, pl.final_ds[:B], self.group)
            all_gather_rows(self.info_all, pl.info[:B], self.group)
        pl.ctx.commit_records(self.world * B, self.final_ds_all, self.info_all, stream=pl.stream)

    def step(self, B=None, attention: bool = True) -> None:
        pl = self.pl
        pl.refine(B)
        pl.match(B)
        if attention:
            pl.synth(B)
            pl.attn(B)
        self.commit(B)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
