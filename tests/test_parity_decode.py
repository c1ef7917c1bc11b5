"""Paged decode (decode is the ~14.6% of request latency that is not prefill,
P:228): with Config.max_decode_tokens = D, il_prefix_match reserves ceil((L + D) / 16) - h pages per
request (the oracle's capacity accounting and eviction follow the same rule, or_set_decode), and
il_prefill_attn runs one row per request at position L_i + t for t = 0..D-1, writing the token's
K / V into the reserved pages and attending over the prompt plus the decode tokens before it.
Checked: integer parity (hits, evictions, index, table) with the reserve, and every decode row
of every request against the fp64 oracle on the whole sequence (Z28 cache transparency)."""
import numpy as np
import pytest
import torch

import oracle as O
from tests.parity_util import StreamSpec, batch_plan, compare_batch, compare_state, gpu_pipeline, make_stream, oracle_for
from workload import gen

pytestmark = pytest.mark.gpu


def _pipeline(sp, pool, instr, D):
    from paper_2507_08523_b200 import Config, Pipeline
    cfg = Config(k=sp.k, table_capacity=sp.T, kv_pages=sp.C, max_batch=sp.B, max_prompt_tokens=sp.max_prompt_tokens,
                 max_pool=sp.M, max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16,
                 n_q_heads=sp.Hq, n_kv_heads=sp.Hkv, head_dim=sp.d, flags=sp.flags, max_decode_tokens=D)
    pl = Pipeline(cfg, "cuda")
    pl.load_pool(pool, instr)
    return pl


@pytest.mark.parametrize("Hq,Hkv,d,D,cascade", [(4, 4, 64, 6, True), (32, 8, 128, 20, True),
                                                (12, 4, 128, 5, True), (64, 8, 128, 4, True),
                                                (16, 8, 64, 5, False), (32, 8, 128, 4, False)])
def test_decode_steps_after_cached_prefill(Hq, Hkv, d, D, cascade, monkeypatch):
    # il_decode_attn: the shared prefix on the tensor kernel's dense phase, each request's own keys
    # on the CUDA-core kernel (g = 1, 2, 3 (padded to 4), 4, 8); without the cascade the CUDA-core
    # kernel covers every key and writes the final rows and LSE
    if not cascade:
        monkeypatch.setenv("IL_CASCADE", "0")
    sp = StreamSpec(B=24, C=200, n_logs=2000, Hq=Hq, Hkv=Hkv, d=d,
                    flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD, ramp=(4,), n_batches=8)
    ds, pool, instr = make_stream(sp)
    o = oracle_for(sp, pool, instr)
    o.set_decode(D)
    pl = _pipeline(sp, pool, instr, D)
    evicting = 0
    for b, (start, B) in enumerate(batch_plan(sp, ds.n)):
        batch = gen.make_batch(ds, start, B)
        r = o.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=sp.max_prompt_tokens // 16)
        pl.stage_batch(batch)
        pl.refine(); pl.match(); pl.synth(); pl.attn()
        pl.ctx.status_sync()
        compare_batch(r, pl, B, sp, where=f"batch {b}")
        evicting += len(r.evicted) > 0
        # D decode tokens, every request, every row against fp64 on prompt + decode tokens
        dec = np.stack([gen.decode_tokens(batch.q_src, t) for t in range(D)], 1)      # [B][D]
        worst = 0.0
        for t in range(D):
            pl.decode_step(t, torch.from_numpy(dec[:, t].astype(np.int64)).to("cuda"))
            pl.ctx.status_sync()
            got = pl.dec_out[:B].float().cpu().numpy().astype(np.float64)
            glse = pl.dec_lse[:B].cpu().numpy().astype(np.float64)
            for i in range(B):
                L = int(r.prompt_len[i])
                toks = np.concatenate([r.prompt(i), dec[i, :t + 1]]).astype(np.uint32)
                pos = np.arange(L + t + 1)
                q = gen.bf16_bits_to_f64(gen.synth_bf16_bits(pl.qkv_seed, "q", toks[-1:], pos[-1:], Hq, d))
                k = gen.bf16_bits_to_f64(gen.synth_bf16_bits(pl.qkv_seed, "k", toks, pos, Hkv, d))
                v = gen.bf16_bits_to_f64(gen.synth_bf16_bits(pl.qkv_seed, "v", toks, pos, Hkv, d))
                ref, rl = O.attention(q, k, v, P=L + t, scale=d ** -0.5, want_lse=True)
                ref, rl = ref[0], rl[0]
                err = np.abs(got[i] - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)
                assert err.max() <= 1e-2, (b, t, i, float(err.max()))
                assert np.abs(glse[i] - rl).max() <= 1e-3 * max(1.0, np.abs(rl).max()), (b, t, i)
                worst = max(worst, float(err.max()))
        pl.commit()
        pl.ctx.status_sync()
        compare_state(o, pl, where=f"batch {b}")
    assert evicting >= 1
