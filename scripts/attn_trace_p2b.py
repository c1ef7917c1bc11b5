"""Profiling aid: merged, time-sorted event list of the attention kernel's phase 2 in CTA 0
(trace build: build.py trace=True with -DIL_TRACE_PHASE=2), over a window of items.  Events:
  Kp/Vp  producer issued K / V load lc      Kf  MMA passed K_FULL(lc) (QK follow)
  PVx    MMA passed the waits of PV of tile x (load lc)
  SA/SB  softmax saw S_FULL (tile count)    PA/PB  softmax stored P (arrived P_FULL)
  LA     softmax A: S loaded into registers  QA  MMA passed Q_FULL of item (A)   EA  epilogue A done"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_08523_b200 import _lib  # noqa: E402

_lib.LIB_PATH = _lib.LIB_PATH.replace(".so", os.environ.get("IL_TRACE_SUFFIX", "_trace") + ".so")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_08523_b200 import IL_F_GUARD, IL_F_PAIR, IL_F_VERIFY, Config, Pipeline  # noqa: E402
from workload import gen  # noqa: E402


def main():
    cfg, ds, pool, instr = bench.workload(3, 0, 1, n_queries=100 * 1024)
    c = Config(k=cfg.k, table_capacity=cfg.T, kv_pages=cfg.C, max_batch=cfg.B, max_prompt_tokens=cfg.max_prompt_tokens,
               max_pool=cfg.M, max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16,
               max_suffix_tokens=cfg.B * cfg.max_prompt_tokens, n_q_heads=cfg.Hq, n_kv_heads=cfg.Hkv, head_dim=cfg.d,
               flags=IL_F_PAIR | IL_F_VERIFY | IL_F_GUARD)
    pl = Pipeline(c, "cuda", fused_kv=True)
    pl.load_pool(pool, instr)
    nb = int(os.environ.get("NB", "85"))
    lib = _lib.load()
    plan = bench.plan_batches(cfg, nb, 0, 1)
    for j, (s, b) in enumerate(plan):                 # steady state: the cache is full after ~75
        if j == len(plan) - 1:                         # trace the last batch only
            torch.cuda.synchronize()
            _lib.check(lib.il_debug_trace_reset(), "trace reset")
        pl.stage_batch(gen.make_batch(ds, s, b))
        pl.step()
    torch.cuda.synchronize()
    raw = np.zeros(16 * 4096 + 1024 * 4 // 2 + 8, np.uint64)
    lib.il_debug_trace.argtypes = [C.c_void_p]
    _lib.check(lib.il_debug_trace(raw.ctypes.data_as(C.c_void_p)), "trace")
    tr = raw[:16 * 4096].reshape(16, 4096).astype(np.int64)
    names = {0: "Kp", 1: "Vp", 2: "Kf", 4: "SA", 5: "PA", 6: "SB", 7: "PB", 8: "LA", 13: "QA", 15: "EA"}
    ev = []
    for slot, nm in names.items():
        for idx in np.flatnonzero(tr[slot] > 0):
            ev.append((int(tr[slot][idx]), nm, int(idx)))
    for idx in np.flatnonzero(tr[3] > 0):
        ev.append((int(tr[3][idx]), "PV" + "AB"[idx & 1], int(idx >> 1)))
    ev.sort()
    t0 = ev[0][0]
    q = sorted(t for t, n, _ in ev if n == "QA")
    n_items = len(q)
    span = ev[-1][0] - t0
    print(f"phase 2, CTA 0 (last batch of {nb}): {n_items} A items; span {span} cycles, {span / max(n_items, 1):.0f} per item")
    lo = q[min(6, n_items - 1)]
    hi = q[min(12, n_items - 1)]
    prev = lo
    for t, n, i in ev:
        if lo - 3000 <= t <= hi:
            print(f"{t - lo:8d} (+{t - prev:5d})  {n:4s} {i}")
            prev = t


if __name__ == "__main__":
    main()
