"""Full-size parity: BASELINE.json configs[2] exactly as bench.py runs it (c3: 1,024 ~2k-token
prompts per batch, 200-demo pool, k = 5, T = 4,096, C = 73,728 pages, Llama-3-8B attention
shape, PAIR + verify + guard, cold-start ramp, then per-stage CUDA graphs replayed).  The integer
path (refine, hashes, hits, eviction, index and table state) is compared bit for bit with the
oracle after every batch, through the point where LRU eviction runs every batch; attention is
checked on EVERY row of all 1,024 requests of the last (evicting) batch against the fp64 oracle
(Z27 tolerance)."""
import numpy as np
import pytest

import bench
import oracle as O
from tests.parity_util import StreamSpec, compare_batch, compare_state
from workload import gen

pytestmark = pytest.mark.gpu

N_FULL = 150         # at most this many full batches after the ramp; stop once 4 batches have evicted


def check_all_rows(pl, r, B, cfg, tol=1e-2):
    """Every suffix row of every request of the batch against the fp64 oracle (attention_np).
    Q/K/V come from the Z28 generator, evaluated once per distinct (token, position) pair of the
    batch (requests share the instruction and most demonstrations)."""
    toks = [r.prompt(i) for i in range(B)]
    Ls = np.array([len(t) for t in toks]); Ps = 16 * r.hit[:B].astype(np.int64)
    key = np.concatenate([t.astype(np.uint64) << np.uint64(32) | np.arange(len(t), dtype=np.uint64) for t in toks])
    uk, inv = np.unique(key, return_inverse=True)
    ut, up = (uk >> np.uint64(32)).astype(np.uint32), (uk & np.uint64(0xFFFFFFFF)).astype(np.int64)
    K = gen.bf16_bits_to_f64(gen.synth_bf16_bits(cfg.qkv_seed, "k", ut, up, cfg.Hkv, cfg.d))[inv]
    V = gen.bf16_bits_to_f64(gen.synth_bf16_bits(cfg.qkv_seed, "v", ut, up, cfg.Hkv, cfg.d))[inv]
    off = np.concatenate([[0], np.cumsum(Ls)])
    cu = pl.cu_q[:B + 1].cpu().numpy()
    got = pl.out[:int(cu[B])].float().cpu().numpy().astype(np.float64)
    worst = 0.0
    for i in range(B):
        P, L = int(Ps[i]), int(Ls[i])
        q = gen.bf16_bits_to_f64(gen.synth_bf16_bits(cfg.qkv_seed, "q", toks[i][P:], np.arange(P, L), cfg.Hq, cfg.d))
        ref = O.attention_np(q, K[off[i]:off[i + 1]], V[off[i]:off[i + 1]], P=P, scale=cfg.d ** -0.5)
        g_ = got[cu[i]:cu[i + 1]]
        err = np.abs(g_ - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
        assert err.max() <= tol, (i, P, L, float(err.max()))
        worst = max(worst, float(err.max()))
    return worst


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
                  max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16, max_log_tokens=255,
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
        if evicting >= 4:
            break
        batch = gen.make_batch(ds, start, B)
        r = o.run_batch(batch, prompt_stride=cfg.max_prompt_tokens, max_blocks=MB)
        pl.stage_batch(batch)
        if graphs is None and B == cfg.B and b >= 4:
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
        if b % 12 == 11 or evicting:
            compare_state(o, pl, where=f"c3 batch {b}")
    assert evicting >= 4, "the stream should reach steady-state LRU eviction"
    # attention of the last batch (an evicting one, replayed from the graphs): every row of every
    # request, so the dense phase-1 M-tiles that straddle request boundaries are all covered
    check_all_rows(pl, r, B, cfg)
