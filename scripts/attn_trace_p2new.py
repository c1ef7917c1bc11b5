"""Profiling aid: merged, time-sorted event list of the phase-2 kernel (attn_p2.cuh) in CTA 0 of
the last steady-state batch (trace build: build.py trace=True, defines -DIL_TRACE_PHASE=2).
Events (x = stream): Kx / Vx producer issued the K / V load of step s; QKx / PVx issuer issued
QK / PV of step s; Sx / Px softmax saw S / stored P of step s; Qx Q TMA issued (item); Dx epilogue
done (item)."""
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
    for j, (s, b) in enumerate(plan):
        if j == len(plan) - 1:
            torch.cuda.synchronize()
            _lib.check(lib.il_debug_trace_reset(), "trace reset")
        pl.stage_batch(gen.make_batch(ds, s, b))
        pl.step()
    torch.cuda.synchronize()
    raw = np.zeros(16 * 4096 + 1024 * 4 // 2 + 8, np.uint64)
    lib.il_debug_trace.argtypes = [C.c_void_p]
    _lib.check(lib.il_debug_trace(raw.ctypes.data_as(C.c_void_p)), "trace")
    tr = raw[:16 * 4096].reshape(16, 4096).astype(np.int64)
    names = {0: "K0", 1: "V0", 2: "K1", 3: "V1", 4: "S0", 5: "S1", 6: "QK0", 7: "QK1", 8: "PV0", 9: "PV1",
             10: "P0", 11: "P1", 12: "Q0", 13: "Q1", 14: "D0", 15: "D1"}
    ev = []
    for slot, nm in names.items():
        for idx in np.flatnonzero(tr[slot] > 0):
            ev.append((int(tr[slot][idx]), nm, int(idx)))
    ev.sort()
    t0 = ev[0][0]
    span = ev[-1][0] - t0
    n_items = sum(1 for _, n, _ in ev if n == "D0")
    print(f"phase 2 (attn_p2), CTA 0: {n_items} stream-0 items; span {span} cycles, {span / max(n_items, 1):.0f} per item")
    # per stream: softmax time (S seen -> P stored) and wait (P stored -> next S seen), epilogue
    for x in (0, 1):
        S = {i: t for t, n, i in ev if n == f"S{x}"}
        P = {i: t for t, n, i in ev if n == f"P{x}"}
        QK = {i: t for t, n, i in ev if n == f"QK{x}"}
        ks = sorted(set(S) & set(P))
        sm = [P[k] - S[k] for k in ks]
        gap = [S[k + 1] - P[k] for k in ks if k + 1 in S]
        lat = [S[k] - QK[k] for k in ks if k in QK]
        print(f"stream {x}: steps {len(ks)}; softmax median {np.median(sm):.0f}; P -> next S median {np.median(gap):.0f} "
              f"(mean {np.mean(gap):.0f}); QK issue -> S seen median {np.median(lat):.0f}; span per step {span / max(len(ks), 1):.0f}")
    if os.environ.get("IL_P2_TRACE_SM"):              # softmax sub-steps of stream 0 (slots 0-3)
        S = tr[4]
        for nm, a, b in (("S seen -> LDTM done", S, tr[0]), ("LDTM -> max done", tr[0], tr[1]),
                         ("max -> exps done", tr[1], tr[2]), ("exps -> STTM done", tr[2], tr[3]),
                         ("STTM -> P arrive", tr[3], tr[10])):
            m = (a > 0) & (b > 0)
            print(f"  {nm:22s} median {np.median(b[m] - a[m]):7.0f}  mean {np.mean(b[m] - a[m]):7.0f}")
        return
    # per-event-type gap statistics
    w0 = sorted(t for t, n, _ in ev if n == "Q0")
    lo = w0[min(6, len(w0) - 1)]
    hi = w0[min(10, len(w0) - 1)]
    prev = lo
    for t, n, i in ev:
        if lo - 2000 <= t <= hi:
            print(f"{t - lo:8d} (+{t - prev:5d})  {n:4s} {i}")
            prev = t


if __name__ == "__main__":
    main()
