"""Profiling aid: cross-batch pipelining at c3 (il.h il_set_sm_split): batch b's attention on
one stream, batch b's commit and batch b+1's select / refine / match on another, two buffer slots.
Prints ms per step for the serial schedule and for the pipelined one at several SM splits.

    python scripts/pipeline_probe.py [R ...]      # R = SMs left to the integer stream
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2507_08523_b200 import IL_F_GUARD, IL_F_PAIR, IL_F_VERIFY, Config, Pipeline  # noqa: E402
from workload import gen  # noqa: E402


def main():
    splits = [int(x) for x in sys.argv[1:]] or [8, 12, 16, 24]
    K, W = 40, 4
    cfg, ds, pool, instr = bench.workload(3, 0, 1, n_queries=(200 + W + 2 * K * (len(splits) + 2)) * 1024 + 65)
    dev = torch.device("cuda", 0)
    c = Config(k=cfg.k, table_capacity=cfg.T, kv_pages=cfg.C, max_batch=cfg.B, max_prompt_tokens=cfg.max_prompt_tokens,
               max_pool=cfg.M, max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16, max_log_tokens=255,
               max_suffix_tokens=cfg.B * cfg.max_prompt_tokens, n_q_heads=cfg.Hq, n_kv_heads=cfg.Hkv, head_dim=cfg.d,
               flags=IL_F_PAIR | IL_F_VERIFY | IL_F_GUARD)
    sA, sB = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    pl = Pipeline(c, dev, qkv_seed=cfg.qkv_seed, stream=sB, fused_kv=True, slots=2)
    with torch.cuda.stream(sB):
        pl.load_pool(pool, instr)
    plan = bench.plan_batches(cfg, 200 + W + 2 * K * (len(splits) + 2), 0, 1)
    pos = 0
    stats = torch.zeros(128, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(sB):                        # ramp + fill until a batch evicts
        while True:
            s, b = plan[pos]; pos += 1
            pl.stage_batch(gen.make_batch(ds, s, b))
            pl.step()
            pl.ctx.stats_async(stats, stream=sB)
            if pos > 2 and pl.ctx.stats_from_bytes(stats.cpu().numpy())["evicted_blocks"] > 0:
                break
    torch.cuda.synchronize()
    print(f"filled after {pos} batches", flush=True)

    def dev_in(j):
        bt = gen.make_batch(ds, *plan[j])
        return (torch.from_numpy(bt.q_off.view(np.int32)).to(dev), torch.from_numpy(bt.q_tok.view(np.int32)).to(dev),
                torch.from_numpy(bt.q_src.view(np.int32)).to(dev), bt.B)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    pl.B = cfg.B
    graphs = {}

    def capture():
        # graphs per slot: integer stages on sB, attention stages on sA (launch configurations,
        # incl. the SM split, are baked in at capture)
        torch.cuda.synchronize()
        graphs.clear()
        for slot in (0, 1):
            pl.use(slot)
            for name, st in (("select", sB), ("refine", sB), ("match", sB), ("synth", sA), ("attn", sA), ("commit", sB)):
                pl.stream = st
                st.wait_stream(torch.cuda.current_stream(dev))
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    getattr(pl, name)()
                graphs[slot, name] = g
        pl.stream = sB
        torch.cuda.synchronize()
    capture()

    def serial(n, fl=True):
        nonlocal pos
        ins = [dev_in(pos + j) for j in range(n)]
        pos += n
        pl.use(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(sB)
        with torch.cuda.stream(sB):
            for x in ins:
                if fl:
                    flush.zero_()
                pl.load_inputs(*x)
                for name in ("select", "refine", "match"):
                    graphs[0, name].replay()
                sA.wait_stream(sB)
                with torch.cuda.stream(sA):
                    graphs[0, "synth"].replay(); graphs[0, "attn"].replay()
                sB.wait_stream(sA)
                graphs[0, "commit"].replay()
        e1.record(sB)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    def pipelined(n, fl="A"):
        nonlocal pos
        ins = [dev_in(pos + j) for j in range(n)]
        pos += n
        ev_m = [torch.cuda.Event() for _ in range(n)]
        ev_a = [torch.cuda.Event() for _ in range(n)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(sB)
        sA.wait_stream(sB)
        for j, x in enumerate(ins):
            s = j % 2
            with torch.cuda.stream(sB):
                if j >= 2:
                    sB.wait_event(ev_a[j - 2])            # slot s: batch j-2's attention is done
                pl.use(s)
                if fl == "B":
                    flush.zero_()
                pl.load_inputs(*x)
                for name in ("select", "refine", "match"):
                    graphs[s, name].replay()
                ev_m[j].record(sB)
                graphs[s, "commit"].replay()
            with torch.cuda.stream(sA):
                sA.wait_event(ev_m[j])
                if fl == "A":
                    flush.zero_()
                graphs[s, "synth"].replay(); graphs[s, "attn"].replay()
                ev_a[j].record(sA)
        sB.wait_stream(sA)
        e1.record(sB)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    for _ in range(2):
        serial(W)
    if os.environ.get("PROBE_TRACE"):
        # kernel timeline of a few pipelined steps (CUPTI): which kernels of the integer stream
        # run beside the attention and which wait for it
        from torch.profiler import ProfilerActivity, profile
        pipelined(W, "none")
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            pipelined(6, "none")
        torch.cuda.synchronize()
        evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
        t0 = evs[0].time_range.start
        for e in evs[-int(os.environ.get("PROBE_TRACE_N", "80")):]:
            print(f"{e.time_range.start - t0:10.1f} +{e.time_range.elapsed_us():8.1f} us  {e.name[:70]}", flush=True)
        return
    print(f"serial: {serial(K):.4f} ms/step", flush=True)
    for fl in ("A", "B", "none"):
        pipelined(W, fl)
        t = pipelined(K, fl)
        print(f"pipelined, flush on {fl}: {t:.4f} ms/step", flush=True)
    print(f"serial without flush: {serial(K, False):.4f} ms/step", flush=True)
    for R in splits:
        pl.ctx.set_sm_split(148 - R if R else 0)
        capture()
        pipelined(W)
        t = pipelined(K)
        pl.ctx.status_sync(sB)
        print(f"pipelined, {R} SMs for the integer stream: {t:.4f} ms/step", flush=True)
    pl.ctx.set_sm_split(0)
    capture()
    print(f"serial again: {serial(K):.4f} ms/step", flush=True)
    pl.ctx.status_sync(sB)


if __name__ == "__main__":
    main()
