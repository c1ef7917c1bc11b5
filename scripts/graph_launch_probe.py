"""Profiling aid: host-side cost of replaying each stage's CUDA graph (does the host keep ahead
of the GPU?) and device time of each stage graph replayed back to back."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_08523_b200 import IL_F_GUARD, IL_F_PAIR, IL_F_VERIFY, Config, Pipeline  # noqa: E402
from workload import gen  # noqa: E402


def main():
    cfg, ds, pool, instr = bench.workload(3, 0, 1, 20000)
    c = Config(k=cfg.k, table_capacity=cfg.T, kv_pages=cfg.C, max_batch=cfg.B, max_prompt_tokens=cfg.max_prompt_tokens,
               max_pool=cfg.M, max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16,
               max_suffix_tokens=cfg.B * cfg.max_prompt_tokens, n_q_heads=cfg.Hq, n_kv_heads=cfg.Hkv, head_dim=cfg.d,
               flags=IL_F_PAIR | IL_F_VERIFY | IL_F_GUARD)
    s = torch.cuda.Stream()
    pl = Pipeline(c, "cuda", stream=s)
    with torch.cuda.stream(s):
        pl.load_pool(pool, instr)
        plan = bench.plan_batches(cfg, 12, 0, 1)
        for st, b in plan[:-3]:
            pl.stage_batch(gen.make_batch(ds, st, b)); pl.step()
        graphs = pl.capture(cfg.B)
        torch.cuda.synchronize()
        for n in pl.STAGES:
            for _ in range(3):
                torch.cuda.synchronize()
                t = time.perf_counter(); graphs[n].replay(); h = time.perf_counter() - t
                torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); graphs[n].replay(); e1.record(s); torch.cuda.synchronize()
            print(f"{n:8s} host replay {h * 1e6:8.1f} us   device {e0.elapsed_time(e1) * 1e3:8.1f} us", flush=True)
        # back to back, GPU busy (a 256 MiB memset first), events between stages as bench.py does
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        for rep in range(3):
            torch.cuda.synchronize()
            flush.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            hs = []
            for i, n in enumerate(pl.STAGES):
                ev[i].record(s)
                t = time.perf_counter(); graphs[n].replay(); hs.append(time.perf_counter() - t)
            ev[5].record(s)
            torch.cuda.synchronize()
            print("busy: " + "  ".join(f"{n} host {h * 1e6:.1f} dev {ev[i].elapsed_time(ev[i + 1]) * 1e3:.1f}"
                                       for i, (n, h) in enumerate(zip(pl.STAGES, hs))), flush=True)


if __name__ == "__main__":
    main()
