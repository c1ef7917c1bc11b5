"""Profiling aid: phase-2 timeline of tile A in CTA 0 (trace build with -DIL_TRACE_PHASE=2):
per item, Q landed (MMA saw Q_FULL), each tile's S seen / P stored, the epilogue done."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv += []
import scripts.attn_trace3 as t3  # noqa: E402  (same driver: workload, trace read)


def main():
    from paper_2507_08523_b200 import _lib
    import torch
    import bench
    from paper_2507_08523_b200 import IL_F_GUARD, IL_F_PAIR, IL_F_VERIFY, Config, Pipeline
    from workload import gen
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
    K, SA, PA, SB, PB, Q, E = tr[2], tr[4], tr[5], tr[6], tr[7], tr[13], tr[15]
    nK = int((K > 0).sum()); nI = int((Q > 0).sum()); nSA = int((SA > 0).sum())
    t0 = K[0]
    dur = K[nK - 1] - K[0]
    print(f"phase 2, CTA 0: {nK} loads, {nI} items (A), {nSA} A tiles, {int((SB > 0).sum())} B tiles; span {dur} cycles; "
          f"{dur / max(nI, 1):.0f} cycles per item, {dur / max(nK, 1):.0f} per load")
    print("item: Q_A landed, epilogue A done, (epilogue - Q)")
    for k in range(2, min(14, nI)):
        print(f"  {k:3d}: {Q[k] - t0:8d} {E[k] - t0:8d} {E[k] - Q[k]:7d}")
    print("A tiles: S seen, P stored (rel.)")
    for j in range(4, min(24, nSA)):
        print(f"  {j:3d}: {SA[j] - t0:8d} {PA[j] - t0:8d}  softmax {PA[j] - SA[j]:6d}  gap to next S {SA[j + 1] - PA[j]:6d}")


if __name__ == "__main__":
    main()
