"""Profiling aid: run config-3 steps with libinferlog_b200_trace.so (per-tile clock64 stamps of
every role of the attention kernel in CTA 0) and print the steady-state timeline."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_08523_b200 import _lib  # noqa: E402

_lib.LIB_PATH = _lib.LIB_PATH.replace(".so", "_trace.so")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_08523_b200 import IL_F_GUARD, IL_F_PAIR, IL_F_VERIFY, Config, Pipeline  # noqa: E402
from workload import gen  # noqa: E402


def main():
    cfg, ds, pool, instr = bench.workload(3, 0, 1)
    c = Config(k=cfg.k, table_capacity=cfg.T, kv_pages=cfg.C, max_batch=cfg.B, max_prompt_tokens=cfg.max_prompt_tokens,
               max_pool=cfg.M, max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16,
               max_suffix_tokens=cfg.B * cfg.max_prompt_tokens, n_q_heads=cfg.Hq, n_kv_heads=cfg.Hkv, head_dim=cfg.d,
               flags=IL_F_PAIR | IL_F_VERIFY | IL_F_GUARD)
    pl = Pipeline(c, "cuda")
    pl.load_pool(pool, instr)
    for s, b in bench.plan_batches(cfg, 5, 0, 1):
        pl.stage_batch(gen.make_batch(ds, s, b))
        pl.step()
    torch.cuda.synchronize()
    tr = np.zeros((8, 4096), np.uint64)
    lib = _lib.load()
    lib.il_debug_trace.argtypes = [C.c_void_p]
    _lib.check(lib.il_debug_trace(tr.ctypes.data_as(C.c_void_p)), "trace")
    names = ["K-load", "V-load", "QK-issue", "PV-issue", "sm-start", "sm-maxsync", "P0-done", "P1-done"]
    n = int((tr[2] > 0).sum())
    t0 = int(tr[2][0])
    rel = tr.astype(np.int64) - t0
    print("tiles traced:", n)
    lo, hi = 40, 56
    print("kt   " + " ".join(f"{x:>10s}" for x in names))
    for k in range(lo, hi):
        print(f"{k:4d} " + " ".join(f"{int(rel[s][k]):10d}" for s in range(8)))
    d = np.diff(rel[2][20:n - 5])
    print("QK issue period: median", np.median(d), "mean", d.mean())
    print("softmax: start->maxsync", np.median(rel[5][20:n - 5] - rel[4][20:n - 5]),
          "maxsync->P0", np.median(rel[6][20:n - 5] - rel[5][20:n - 5]),
          "S_FULL-wait(QK issue->sm start)", np.median(rel[4][20:n - 5] - rel[2][20:n - 5]),
          "P0->PV issue", np.median(rel[3][20:n - 5] - rel[6][20:n - 5]))


if __name__ == "__main__":
    main()
