"""The multi-GPU plumbing of paper_2507_08523_b200.distributed over gloo on CPU, world size 2
(SURVEY §8(e)): slices partition the global batch in admission order, the pool broadcast delivers
rank 0's pool to every rank, and the record all-gather returns every rank's records in rank-major
= global admission order on every rank (what il_commit_records consumes)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_08523_b200.distributed import all_gather_rows, broadcast_pool, slice_of


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from workload import gen
        ds = gen.make_dataset("S", 500, 14, 1.3, 1004)
        pool = gen.sample_pool(ds, 50, 2004) if rank == 0 else None
        instr = gen.instruction(32, 77) if rank == 0 else None
        p, ins = broadcast_pool(pool, instr, torch.device("cpu"))
        ref = gen.sample_pool(ds, 50, 2004)
        ok_pool = all(np.array_equal(getattr(p, f), np.asarray(getattr(ref, f), np.uint32))
                      for f in ("log_off", "log_tok", "tpl_off", "tpl_tok", "template_id", "src_index"))
        ok_pool &= np.array_equal(ins, np.asarray(gen.instruction(32, 77), np.uint32))
        # records: rank r's slice of a global batch of 10 requests, k = 3, plus 16-byte infos
        B = 10
        lo, hi = slice_of(B, rank, world)
        fds = torch.tensor([[1000 * i + j for j in range(3)] for i in range(lo, hi)], dtype=torch.int32)
        inf = torch.tensor([[i] * 16 for i in range(lo, hi)], dtype=torch.uint8)
        out_f = torch.zeros(B, 3, dtype=torch.int32)
        out_i = torch.zeros(B, 16, dtype=torch.uint8)
        all_gather_rows(out_f, fds)
        all_gather_rows(out_i, inf)
        want_f = np.array([[1000 * i + j for j in range(3)] for i in range(B)])
        ok_rec = np.array_equal(out_f.numpy(), want_f) and np.array_equal(out_i.numpy()[:, 0], np.arange(B))
        # the fused per-rank record buffer (il_commit_export layout: bytes): one row per rank
        nbytes = 4096
        buf = torch.full((1, nbytes), rank + 1, dtype=torch.uint8)
        buf[0, :8] = torch.tensor(list(np.int64(rank * 7919).tobytes()), dtype=torch.uint8)
        all_buf = torch.zeros(world, nbytes, dtype=torch.uint8)
        all_gather_rows(all_buf, buf)
        for r in range(world):
            ok_rec &= bool((all_buf[r, 8:] == r + 1).all())
            ok_rec &= int(np.frombuffer(all_buf[r, :8].numpy().tobytes(), np.int64)[0]) == r * 7919
        q.put((rank, ok_pool, ok_rec))
    finally:
        dist.destroy_process_group()


def test_slices_partition_the_batch_in_admission_order():
    for world in (1, 2, 3, 4, 8):
        for B in (1, 7, 64, 1024):
            got = [slice_of(B, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1


def test_pool_broadcast_and_record_gather_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_pool, ok_rec in res:
        assert ok_pool, f"rank {rank}: pool broadcast"
        assert ok_rec, f"rank {rank}: record all-gather order"
