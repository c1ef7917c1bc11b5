"""Profiling aid: run config-3 steps with libinferlog_b200_trace.so (per-load clock64 stamps of
every role of the attention kernel in CTA 0) and print the steady-state timeline."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_08523_b200 import _lib  # noqa: E402

if not os.environ.get("IL_LIB_VARIANT"):          # a variant built with -DIL_ATTN_TRACE may be named instead
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
    raw = np.zeros(16 * 4096 + 1024 * 4 // 2 + 8, np.uint64)
    lib = _lib.load()
    lib.il_debug_trace.argtypes = [C.c_void_p]
    _lib.check(lib.il_debug_trace(raw.ctypes.data_as(C.c_void_p)), "trace")
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.save(os.path.join(ROOT, "gpurun_out", f"trace_{os.environ.get('IL_LIB_VARIANT', 'trace')}.npy"), raw)
    tr = raw[:16 * 4096].reshape(16, 4096).astype(np.int64)
    items = raw[16 * 4096:16 * 4096 + 2048].view(np.uint32).reshape(1024, 4)
    t0 = tr[2][0]
    rel = np.where(tr > 0, tr - t0, -1)
    n_it = int((items[:, 1] > 0).sum())
    print("items in CTA 0:", n_it, "loads:", int(items[:n_it, 1].sum()))
    print("first items (lc0, nload, nsh, nA|nB<<16):")
    for k in range(min(8, n_it)):
        print("  ", items[k, 0], items[k, 1], items[k, 2], items[k, 3] & 0xFFFF, items[k, 3] >> 16)
    nsh = items[:n_it, 2].astype(float); nl = items[:n_it, 1].astype(float)
    print(f"mean nsh {nsh.mean():.2f}, mean nload {nl.mean():.2f}, shared load share {nsh.sum() / nl.sum():.2%}")
    lo = int(items[2, 0]) if n_it > 3 else 0
    names = ["K-ready", "V-ready", "K_FULL", "PV(A)", "PV(B)", "smA-start", "smA-done", "smB-start", "smB-done"]
    print("lc    K-load  V-load  QK(K_FULL)  PV_A   PV_B")
    for l in range(lo, lo + 20):
        print(f"{l:4d} {rel[0][l]:8d} {rel[1][l]:8d} {rel[2][l]:8d} {rel[3][2*l] if 2*l < 4096 else -1:8d} {rel[3][2*l+1] if 2*l+1 < 4096 else -1:8d}")
    print("softmax tiles (A start, A done, B start, B done):")
    for k in range(64, 84):
        print(f"{k:4d} {rel[4][k]:8d} {rel[5][k]:8d} {rel[6][k]:8d} {rel[7][k]:8d}  durA {rel[5][k]-rel[4][k]:6d} durB {rel[7][k]-rel[6][k]:6d}")
    tot_cycles = rel[2][int(items[n_it - 1, 0])] - rel[2][int(items[1, 0])]
    loads = int(items[1:n_it - 1, 1].sum())
    print("cycles per load (steady):", tot_cycles / max(loads, 1))
    da = rel[5][20:400] - rel[4][20:400]; print("softmax A duration median", np.median(da))
    it_dec, it_q, it_last, it_epi = rel[12][:n_it], rel[13][:n_it], rel[14][:n_it], rel[15][:n_it]
    print("per item (cycles): decoded->Q landed, Q->last PV issued, last PV->epilogue done, epilogue->next decoded")
    for k in range(2, min(12, n_it - 1)):
        print(f"  item {k:3d} nload {int(items[k, 1]):3d}: {it_q[k] - it_dec[k]:7d} {it_last[k] - it_q[k]:7d} "
              f"{it_epi[k] - it_last[k]:7d} {it_dec[k + 1] - it_epi[k]:7d}")
    span = it_dec[n_it - 1] - it_dec[1]
    print("mean cycles per item:", span / max(n_it - 2, 1), " mean loads per item:", float(items[1:n_it - 1, 1].mean()))
    seg = [("S_FULL->ld done", 4, 8), ("ld->exchange done", 8, 9), ("exchange->exp done", 9, 10),
           ("exp->P stored", 10, 11), ("P stored->arrive", 11, 5)]
    for name, a, b in seg:
        print(f"  softmax A {name:22s} median {np.median(rel[b][20:400] - rel[a][20:400]):7.0f} cycles")


if __name__ == "__main__":
    main()
