"""The multi-GPU driver end to end (paper_2507_08523_b200.distributed.DataParallel)
with two real processes on the one test GPU, collectives over gloo (NCCL refuses two ranks on one
device): pool broadcast from rank 0, per batch il_select_batch -> il_commit_apply of the previous
batch's all-gathered record buffers -> refine -> match -> attention -> il_commit_index ->
il_commit_export -> all-gather on the side stream (pipelined: the exchange overlaps the next
batch's selection).  Every batch's top-k, final DS, PMC/rule, hits and box-level hits, and the
final replicated ICL Table, are compared bit for bit with the oracle's run_batch_dp."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SP = dict(B=64, C=500, n_logs=3000, ramp=(8, 32))
N_BATCHES = 12


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_2507_08523_b200 import Config, Pipeline
        from paper_2507_08523_b200.distributed import DataParallel, slice_of
        from tests.parity_util import StreamSpec, batch_plan, make_stream
        from workload import gen
        torch.cuda.set_device(0)
        sp = StreamSpec(**SP, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD)
        ds, pool, instr = make_stream(sp)
        cfg = Config(k=sp.k, table_capacity=sp.T, kv_pages=sp.C, max_batch=sp.B // world,
                     max_prompt_tokens=sp.max_prompt_tokens, max_pool=sp.M,
                     max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16, max_log_tokens=255,
                     n_q_heads=sp.Hq, n_kv_heads=sp.Hkv, head_dim=sp.d, flags=sp.flags, max_global_batch=sp.B,
                     max_block_records=2 * (sp.B // world) * (sp.max_prompt_tokens // 16))
        stream = torch.cuda.Stream()
        pl = Pipeline(cfg, "cuda", stream=stream)
        dp = DataParallel(pl)
        with torch.cuda.stream(stream):
            dp.load_pool(pool if rank == 0 else None, instr if rank == 0 else None)
        sp.n_batches = N_BATCHES
        out = []
        with torch.cuda.stream(stream):
            for b, (start, Bg) in enumerate(batch_plan(sp, ds.n)):
                lo, hi = slice_of(Bg, rank, world)
                pl.stage_batch(gen.make_batch(ds, start + lo, hi - lo))
                dp.step()
                stream.synchronize()
                n = hi - lo
                out.append(dict(topk=pl.u32(pl.topk[:n]), fin=pl.u32(pl.final_ds[:n]), info=pl.info_np(n),
                                hit=pl.u32(pl.hit[:n]), box=pl.ctx.box_hit_dump(n, stream)))
            dp.flush()
        stream.synchronize()
        pl.ctx.status_sync(stream)
        q.put((rank, out, pl.ctx.table_dump(), None))
    except Exception as e:      # report instead of hanging the parent
        import traceback
        q.put((rank, None, None, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_dataparallel_two_processes_one_gpu_gloo():
    import oracle as O
    from paper_2507_08523_b200.distributed import slice_of
    from tests.parity_util import StreamSpec, batch_plan, make_stream
    from workload import gen
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, out, tab, err = q.get(timeout=600)
        assert err is None, err
        res[rank] = (out, tab)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sp = StreamSpec(**SP, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD)
    ds, pool, instr = make_stream(sp)
    ranks = []
    for _ in range(world):
        o = O.Oracle(sp.k, sp.T, sp.C, flags=sp.flags)
        o.pool_load(pool, instr)
        ranks.append(o)
    sp.n_batches = N_BATCHES
    gain = 0
    for b, (start, Bg) in enumerate(batch_plan(sp, ds.n)):
        r = O.Oracle.run_batch_dp(ranks, gen.make_batch(ds, start, Bg), prompt_stride=sp.max_prompt_tokens,
                                  max_blocks=sp.max_prompt_tokens // 16)
        for g in range(world):
            lo, hi = slice_of(Bg, g, world)
            got = res[g][0][b]
            np.testing.assert_array_equal(got["topk"], r.topk[lo:hi], err_msg=f"b{b} r{g} topk")
            np.testing.assert_array_equal(got["fin"], r.final_ds[lo:hi], err_msg=f"b{b} r{g} final_ds")
            np.testing.assert_array_equal(got["info"]["pmc"], r.info[lo:hi, 0], err_msg=f"b{b} r{g} pmc")
            np.testing.assert_array_equal(got["info"]["rule"], r.info[lo:hi, 1], err_msg=f"b{b} r{g} rule")
            np.testing.assert_array_equal(got["hit"], r.hit[lo:hi], err_msg=f"b{b} r{g} hit")
            if b > 0:
                np.testing.assert_array_equal(got["box"], r.box_hit[lo:hi], err_msg=f"b{b} r{g} box hits")
                gain += int(r.box_hit[lo:hi].sum() - r.hit[lo:hi].sum())
    ods, ots = ranks[0].table_dump()
    for g in range(world):
        gds, gts = res[g][1]
        np.testing.assert_array_equal(gts, ots)
        np.testing.assert_array_equal(gds, ods)
    assert gain > 0
