"""Profiling aid: kernel timeline (torch.profiler / CUPTI) of a few steady-state steps of the
default bench workload, to see gaps between the library's kernels inside each stage."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2507_08523_b200 import IL_F_GUARD, IL_F_PAIR, IL_F_VERIFY, Config, Pipeline  # noqa: E402
from workload import gen  # noqa: E402


def main():
    NB = int(os.environ.get('PROBE_BATCHES', '12'))
    cfg, ds, pool, instr = bench.workload(3, 0, 1, (NB + 2) * 1024)
    c = Config(k=cfg.k, table_capacity=cfg.T, kv_pages=cfg.C, max_batch=cfg.B, max_prompt_tokens=cfg.max_prompt_tokens,
               max_pool=cfg.M, max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16,
               max_suffix_tokens=cfg.B * cfg.max_prompt_tokens, n_q_heads=cfg.Hq, n_kv_heads=cfg.Hkv, head_dim=cfg.d,
               flags=IL_F_PAIR | IL_F_VERIFY | IL_F_GUARD)
    s = torch.cuda.Stream()
    pl = Pipeline(c, "cuda", stream=s)
    with torch.cuda.stream(s):
        pl.load_pool(pool, instr)
        plan = bench.plan_batches(cfg, NB, 0, 1)
        for st, b in plan[:-3]:
            pl.stage_batch(gen.make_batch(ds, st, b)); pl.step()
        torch.cuda.synchronize()
        graphs = None
        if "--graph" in sys.argv:                      # per-stage CUDA graphs, as bench.py replays them
            pl.stage_batch(gen.make_batch(ds, *plan[-4])); pl.step()
            graphs = pl.capture(cfg.B)
            torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for st, b in plan[-3:]:
                pl.stage_batch(gen.make_batch(ds, st, b))
                if graphs is None:
                    pl.step()
                else:
                    for n in pl.STAGES:
                        graphs[n].replay()
            torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    prev = None
    for e in ev[-60:]:
        gap = (e.time_range.start - prev) if prev else 0
        print(f"{(e.time_range.start - t0):9.1f} us  dur {e.time_range.elapsed_us():8.1f}  gap {gap:7.1f}  {e.name[:60]}")
        prev = e.time_range.end


if __name__ == "__main__":
    main()
