"""Profiling aid: per-load hand-off latencies of the attention kernel's phase 1 (CTA 0), from a
trace build (build.py --trace; optionally with -DIL_NO_SOFTMAX: IL_TRACE_SUFFIX=_tracensm).
Phase-1 loads target both Q tiles, so load l is tile step l of A and of B:
  K(l)    MMA issuer passed K_FULL(l) (QK of A and B follow)
  S_x(l)  softmax x saw S_FULL            P_x(l)  softmax x arrived P_FULL
  PV_x(l) MMA issuer passed its waits for PV(l) of tile x (the MMAs follow)"""
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
    K, PV, SA, PA, SB, PB = tr[2], tr[3], tr[4], tr[5], tr[6], tr[7]
    n = int((K > 0).sum())
    lo, hi = 30, min(n - 30, 300)
    l = np.arange(lo, hi)
    pva, pvb = PV[2 * l], PV[2 * l + 1]
    print(f"phase-1 loads in CTA 0: {n}; window {lo}..{hi}")
    med = lambda v: float(np.median(v))
    print(f"cycles per load (K_FULL passed): {med(np.diff(K[lo:hi])):.0f}")
    for nm, S, P, pv in (("A", SA, PA, pva), ("B", SB, PB, pvb)):
        print(f"tile {nm}: K(l)->S(l) {med(S[l] - K[l]):.0f} | S->P (softmax) {med(P[l] - S[l]):.0f} | "
              f"P(l)->PV(l) issued {med(pv - P[l]):.0f} | S(l)->S(l+1) {med(S[l + 1] - S[l]):.0f}")
    print(f"PV_A(l) -> K(l+1) {med(K[l + 1] - pva):.0f} | PV_B(l) -> PV_A(l+1) {med(PV[2 * l + 2] - pvb):.0f} | "
          f"PV_A(l) -> PV_B(l) {med(pvb - pva):.0f}")
    print("raw (rel. to K[lo]):")
    for j in range(lo, lo + 8):
        b0 = K[lo]
        print(f"  l={j}: K {K[j] - b0:7d}  S_A {SA[j] - b0:7d}  P_A {PA[j] - b0:7d}  PV_A {PV[2 * j] - b0:7d}  "
              f"S_B {SB[j] - b0:7d}  P_B {PB[j] - b0:7d}  PV_B {PV[2 * j + 1] - b0:7d}")


if __name__ == "__main__":
    main()
