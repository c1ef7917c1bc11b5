"""Profiling aid (round 2): per-role clock64 timeline of the attention kernel in CTA 0, from the
trace build (python paper_2507_08523_b200/build.py --trace -> libinferlog_b200_trace.so), on
steady-state config-3 steps.  Prints cycles per KV load, the softmax phases per tile, and the
gaps between the roles' hand-offs."""
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
    cfg, ds, pool, instr = bench.workload(3, 0, 1, n_queries=12 * 1024)
    c = Config(k=cfg.k, table_capacity=cfg.T, kv_pages=cfg.C, max_batch=cfg.B, max_prompt_tokens=cfg.max_prompt_tokens,
               max_pool=cfg.M, max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16,
               max_suffix_tokens=cfg.B * cfg.max_prompt_tokens, n_q_heads=cfg.Hq, n_kv_heads=cfg.Hkv, head_dim=cfg.d,
               flags=IL_F_PAIR | IL_F_VERIFY | IL_F_GUARD)
    pl = Pipeline(c, "cuda")
    pl.load_pool(pool, instr)
    for s, b in bench.plan_batches(cfg, 8, 0, 1):
        pl.stage_batch(gen.make_batch(ds, s, b))
        pl.step()
    torch.cuda.synchronize()
    raw = np.zeros(16 * 4096 + 1024 * 4 // 2 + 8, np.uint64)
    lib = _lib.load()
    lib.il_debug_trace.argtypes = [C.c_void_p]
    _lib.check(lib.il_debug_trace(raw.ctypes.data_as(C.c_void_p)), "trace")
    tr = raw[:16 * 4096].reshape(16, 4096).astype(np.int64)
    t0 = tr[2][0]
    R = np.where(tr > 0, tr - t0, -1)
    nl = int((R[2] >= 0).sum())
    lo, hi = 40, min(nl - 10, 400)
    kf = R[2][lo:hi]
    print(f"loads seen by the MMA issuer: {nl}; steady window {lo}..{hi}")
    print(f"cycles per KV load (MMA K_FULL seen): median {np.median(np.diff(kf)):.0f} mean {np.mean(np.diff(kf)):.0f}")
    print(f"K load issued -> K_FULL seen by MMA: median {np.median(R[2][lo:hi] - R[0][lo:hi]):.0f}")
    for x, nm in ((0, "A"), (1, "B")):
        s_full, p_full = R[4 + 2 * x], R[5 + 2 * x]
        n = int((s_full >= 0).sum())
        a, b = 30, min(n - 5, 300)
        d = p_full[a:b] - s_full[a:b]
        idle = s_full[a + 1:b + 1] - p_full[a:b]
        print(f"softmax {nm}: tiles {n}; S seen -> P_FULL median {np.median(d):.0f}; P_FULL -> next S seen median {np.median(idle):.0f}")
    s4, s8, s9, s10, s11, s5 = R[4], R[8], R[9], R[10], R[11], R[5]
    a, b = 30, 300
    for nm, x, y in (("S seen->LDTM done", s4, s8), ("LDTM->max done", s8, s9), ("max->exp+P done", s9, s10),
                     ("P done->st waited", s10, s11), ("st waited->arrive", s11, s5)):
        v = (y[a:b] - x[a:b]); v = v[(x[a:b] >= 0) & (y[a:b] >= 0)]
        print(f"  softmax A {nm:20s} median {np.median(v) if len(v) else -1:.0f}")
    pv = R[3]
    print("PV issue times (A,B interleaved) first 24 of window:", (pv[2 * lo:2 * lo + 24] - pv[2 * lo]).tolist())
    print("K_FULL seen times (window start):", (R[2][lo:lo + 12] - R[2][lo]).tolist())
    print("S_FULL A seen:", (R[4][30:42] - R[2][lo]).tolist())
    print("P_FULL A:", (R[5][30:42] - R[2][lo]).tolist())
    print("S_FULL B seen:", (R[6][30:42] - R[2][lo]).tolist())
    print("P_FULL B:", (R[7][30:42] - R[2][lo]).tolist())
    d = np.diff(R[2][lo:hi])
    big = np.where(d > 3 * np.median(d))[0]
    print(f"load gaps > 3x median: {len(big)} of {len(d)}; their share of the window {d[big].sum() / d.sum():.1%}; "
          f"median big gap {np.median(d[big]) if len(big) else 0:.0f}")
    eq = R[13][:64]; ep = R[15][:64]
    print("item: Q_FULL A seen by MMA / epilogue A done (first 12):", list(zip((eq[:12] - R[2][lo]).tolist(), (ep[:12] - R[2][lo]).tolist())))
    hist = np.percentile(d, [10, 25, 50, 75, 90, 99])
    print("load interval percentiles 10/25/50/75/90/99:", hist.round().tolist())


if __name__ == "__main__":
    main()
