"""Full-size parity: BASELINE.json configs[2] exactly as bench.py runs it (c3: 1,024 ~2k-token
prompts per batch, 200-demo pool, k = 5, T = 4,096, C = 73,728 pages, Llama-3-8B attention
shape, PAIR + verify + guard, cold-start ramp, then per-stage CUDA graphs replayed).  The integer
path (refine, hashes, hits, eviction, index and table state) is compared bit for bit with the
oracle after every batch, through the point where LRU eviction runs every batch; attention is
checked on sampled requests of the last batch against the fp64 oracle (Z27 tolerance)."""
import numpy as np
import pytest

import bench
import oracle as O
from tests.parity_util import StreamSpec, compare_batch, compare_state
from tests.test_parity_attn import check_request
from workload import gen

pytestmark = pytest.mark.gpu

N_FULL = 84          # full batches after the ramp: LRU eviction starts at about the 75th


def test_c3_fullsize_stream_graphs():
    import torch
    from paper_2507_08523_b200 import IL_F_GUARD, IL_F_PAIR, IL_F_VERIFY, Config, Pipeline

    cfg0 = gen.config(3)
    plan = bench.plan_batches(cfg0, N_FULL, 0, 1)
    n_q = plan[-1][0] + plan[-1][1]
    cfg, ds, pool, instr = bench.workload(3, 0, 1, n_queries=n_q)
    flags = IL_F_PAIR | IL_F_VERIFY | IL_F_GUARD
    ccfg = Config(k=cfg.k, table_capacity=cfg.T, kv_pages=cfg.C, max_batch=cfg.B,
                  max_prompt_tokens=cfg.max_prompt_tokens, max_pool=cfg.M,
                  max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16, max_log_tokens=256,
                  max_suffix_tokens=cfg.B * cfg.max_prompt_tokens, n_q_heads=cfg.Hq, n_kv_heads=cfg.Hkv,
                  head_dim=cfg.d, flags=flags)
    pl = Pipeline(ccfg, "cuda", qkv_seed=cfg.qkv_seed)
    pl.load_pool(pool, instr)
    o = O.Oracle(cfg.k, cfg.T, cfg.C, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD)
    o.pool_load(pool, instr)
    sp = StreamSpec(k=cfg.k, B=cfg.B, T=cfg.T, C=cfg.C, max_prompt_tokens=cfg.max_prompt_tokens,
                    Hq=cfg.Hq, Hkv=cfg.Hkv, d=cfg.d, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD)
    MB = (cfg.max_prompt_tokens + 15) // 16
    graphs = None
    evicting = 0
    for b, (start, B) in enumerate(plan):
        batch = gen.make_batch(ds, start, B)
        r = o.run_batch(batch, prompt_stride=cfg.max_prompt_tokens, max_blocks=MB)
        pl.stage_batch(batch)
        if graphs is None and B == cfg.B and b >= len(plan) - N_FULL + 2:
            graphs = pl.capture(cfg.B)                 # as bench.py: per-stage graphs after warm-up
        if graphs is not None and B == cfg.B:
            for n in pl.STAGES:
                graphs[n].replay()
        else:
            pl.step()
        pl.ctx.status_sync()
        torch.cuda.synchronize()
        compare_batch(r, pl, B, sp, where=f"c3 batch {b}")
        evicting += len(r.evicted) > 0
        if b % 12 == 11 or b >= len(plan) - 4:
            compare_state(o, pl, where=f"c3 batch {b}")
    assert evicting >= 3, "the stream should reach steady-state LRU eviction"
    # attention of sampled requests of the last batch (rows sampled inside long suffixes)
    rng = np.random.default_rng(7)
    picks = set(rng.choice(B, size=4, replace=False).tolist()) | {int(np.argmax(r.prompt_len - 16 * r.hit)), B - 1}
    for i in sorted(picks):
        check_request(pl, r, i, sp, cfg.qkv_seed, 1.0, max_rows=40)
