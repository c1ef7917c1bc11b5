"""The cross-batch pipelined schedule (include/il.h, il_set_sm_split comment; bench.py's headline)
on the GPU vs the oracle: batch b's QKV stand-in + attention run on one stream while batch b's
commit and batch b+1's select / refine / match run on another, with two per-batch buffer slots.
Every batch's integer outputs must equal the oracle's bit for bit (the schedule changes when
kernels run, never what they compute), the prefix index and ICL Table after the stream too, and
the attention of sampled requests of every batch stays within Z27 of fp64 -- including requests
whose pages were freed or evicted (metadata) by the next batch's calls while their attention ran."""
import numpy as np
import pytest
import torch

import oracle as O
from tests.parity_util import StreamSpec, batch_plan, compare_state, gpu_config, make_stream, oracle_for
from workload import gen

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _run(sp: StreamSpec, n_batches: int, split: int = 0, split_synth: bool = False):
    from paper_2507_08523_b200 import Pipeline
    ds, pool, instr = make_stream(sp)
    o = oracle_for(sp, pool, instr)
    cfg = gpu_config(sp, pool)
    dev = torch.device("cuda")
    sA, sB = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    pl = Pipeline(cfg, dev, stream=sB, fused_kv=True, slots=2)
    with torch.cuda.stream(sB):
        pl.load_pool(pool, instr)
    if split:
        pl.ctx.set_sm_split(split)
    sp.n_batches = n_batches
    plan = batch_plan(sp, ds.n)
    MB = (sp.max_prompt_tokens + 15) // 16
    ref = [o.run_batch(gen.make_batch(ds, s, B), prompt_stride=sp.max_prompt_tokens, max_blocks=MB) for s, B in plan]
    ev_m = [torch.cuda.Event() for _ in plan]
    ev_a = [torch.cuda.Event() for _ in plan]
    saved = []
    torch.cuda.synchronize()
    for j, (s, B) in enumerate(plan):
        with torch.cuda.stream(sB):
            if j >= 2:
                sB.wait_event(ev_a[j - 2])
            pl.use(j % 2)
            pl.stage_batch(gen.make_batch(ds, s, B))
            pl.select(); pl.refine(); pl.match()
            if split_synth:
                pl.synth(part="q")                     # batch j's Q beside batch j-1's attention
            ev_m[j].record(sB)
            ints = {n: getattr(pl, n)[:B].clone() for n in ("topk", "final_ds", "info", "prompt_len", "hit",
                                                          "prefix_len", "block_hash")}
            ints["cu_q"] = pl.cu_q[:B + 1].clone()
        with torch.cuda.stream(sA):                    # (host order: il.h's call order; device order: streams)
            sA.wait_event(ev_m[j])
            pl.stream = sA
            pl.synth(part="kv" if split_synth else "qkv"); pl.attn()
            pl.stream = sB
            att = {"out": pl.out.clone(), "lse": pl.lse.clone()}
            ev_a[j].record(sA)
        with torch.cuda.stream(sB):
            pl.commit()                                # waits for match(j) only, not for the attention
        saved.append((ints, att))
    torch.cuda.synchronize()
    pl.ctx.status_sync(sB)
    rng = np.random.default_rng(5)
    worst = 0.0
    for j, ((ints, att), r) in enumerate(zip(saved, ref)):
        B = plan[j][1]
        u32 = lambda t: t.cpu().numpy().view(np.uint32)  # noqa: E731
        np.testing.assert_array_equal(u32(ints["topk"]), r.topk, err_msg=f"batch {j} topk")
        np.testing.assert_array_equal(u32(ints["final_ds"]), r.final_ds, err_msg=f"batch {j} final_ds")
        np.testing.assert_array_equal(u32(ints["prompt_len"]), r.prompt_len, err_msg=f"batch {j} prompt_len")
        np.testing.assert_array_equal(u32(ints["hit"]), r.hit, err_msg=f"batch {j} hit")
        bh = ints["block_hash"].cpu().numpy().view(np.uint64)
        for i in range(B):
            F = int(r.prompt_len[i]) // 16
            assert np.array_equal(bh[i, :F], r.block_hash[i, :F]), (j, i)
        suf = r.prompt_len.astype(np.int64) - 16 * r.hit.astype(np.int64)
        np.testing.assert_array_equal(ints["cu_q"].cpu().numpy(), np.concatenate([[0], np.cumsum(suf)]))
        cu = ints["cu_q"].cpu().numpy()
        picks = set(rng.choice(B, size=min(4, B), replace=False).tolist()) | {B - 1, int(np.argmin(r.hit))}
        for i in sorted(picks):
            L, P = int(r.prompt_len[i]), 16 * int(r.hit[i])
            toks, pos = r.prompt(i), np.arange(L)
            q = gen.bf16_bits_to_f64(gen.synth_bf16_bits(pl.qkv_seed, "q", toks[P:], pos[P:], sp.Hq, sp.d, pl.q_scale))
            k = gen.bf16_bits_to_f64(gen.synth_bf16_bits(pl.qkv_seed, "k", toks, pos, sp.Hkv, sp.d))
            v = gen.bf16_bits_to_f64(gen.synth_bf16_bits(pl.qkv_seed, "v", toks, pos, sp.Hkv, sp.d))
            want, wlse = O.attention(q, k, v, P=P, scale=sp.d ** -0.5, want_lse=True)
            got = att["out"][cu[i]:cu[i + 1]].float().cpu().numpy().astype(np.float64)
            glse = att["lse"][cu[i]:cu[i + 1]].cpu().numpy().astype(np.float64)
            err = np.abs(got - want).max(-1) / np.maximum(np.abs(want).max(-1), 1e-6)
            assert err.max() <= TOL, (j, i, float(err.max()))
            assert np.abs(glse - wlse).max() <= 1e-3 * max(1.0, np.abs(wlse).max()), (j, i)
            worst = max(worst, float(err.max()))
    pl.use(0)
    compare_state(o, pl, where="after the pipelined stream")
    return worst


@pytest.mark.parametrize("split_synth", [False, True])
def test_pipelined_stream_eviction_pressure(split_synth):
    # most batches evict: pages of batch b are evicted / freed by batch b+1's match while b's
    # attention may still run; split_synth: batch b+1's Q is written then too (its K / V after)
    sp = StreamSpec(C=700, B=32, T=64, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD, ramp=(4, 16))
    assert _run(sp, 60, split_synth=split_synth) <= TOL


def test_pipelined_c1_stream_and_sm_split():
    sp = StreamSpec(B=64, C=2200, ramp=(64,))
    assert _run(sp, 16) <= TOL
    sp = StreamSpec(B=64, C=1500, ramp=(64,))
    assert _run(sp, 16, split=132) <= TOL              # attention on 132 SMs, integer kernels sized for 16
