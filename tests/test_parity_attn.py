"""Prefill attention on the GPU vs the fp64 oracle (Z26-Z27), through the whole path: the
prefix K/V come from pages written by earlier batches, so this is also the cache-transparency
test (Z28: cached prefill == recompute)."""
import numpy as np
import pytest
import torch

import oracle as O
from tests.parity_util import StreamSpec, batch_plan, gpu_pipeline, make_stream, oracle_for
from workload import gen

pytestmark = pytest.mark.gpu

TOL = 1e-2     # north star: <= 1e-2 max relative error (row-normalised, Z27)


def bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.cpu().view(torch.int16).numpy().view(np.uint16)


def check_request(pl, r, i, sp, seed, q_scale, max_rows=None):
    L, h = int(r.prompt_len[i]), int(r.hit[i])
    P = 16 * h
    S = L - P
    toks = r.prompt(i)
    pos = np.arange(L)
    cu = pl.cu_q.cpu().numpy()
    r0 = int(cu[i])
    assert int(cu[i + 1]) - r0 == S
    # generator parity: the GPU's synthetic Q/K/V rows equal the numpy generator bit for bit
    qb = gen.synth_bf16_bits(seed, "q", toks[P:], pos[P:], sp.Hq, sp.d, q_scale)
    kb = gen.synth_bf16_bits(seed, "k", toks, pos, sp.Hkv, sp.d)
    vb = gen.synth_bf16_bits(seed, "v", toks, pos, sp.Hkv, sp.d)
    np.testing.assert_array_equal(bf16_bits(pl.q[r0:r0 + S]), qb)
    if getattr(pl, "fused_kv", False):
        # the projection stand-in wrote K / V into the request's pages: read them back by position
        bt = pl.block_table[i].cpu().numpy()
        pages = torch.from_numpy(bt[pos[P:] // 16].astype(np.int64)).to(pl.k_pages.device)
        slot = torch.from_numpy((pos[P:] % 16).astype(np.int64)).to(pl.k_pages.device)
        kp = pl.k_pages[pages, :, slot]                   # [S][Hkv][d]
        vp = pl.v_pages[pages, :, slot]
        np.testing.assert_array_equal(bf16_bits(kp), kb[P:])
        np.testing.assert_array_equal(bf16_bits(vp), vb[P:])
    else:
        np.testing.assert_array_equal(bf16_bits(pl.k_new[r0:r0 + S]), kb[P:])
        np.testing.assert_array_equal(bf16_bits(pl.v_new[r0:r0 + S]), vb[P:])
    rows = np.arange(S) if max_rows is None or S <= max_rows else np.unique(
        np.concatenate([np.arange(4), np.linspace(0, S - 1, max_rows).astype(int)]))
    ref, lse = O.attention(gen.bf16_bits_to_f64(qb)[rows[-1] * 0:], gen.bf16_bits_to_f64(kb),
                           gen.bf16_bits_to_f64(vb), P=P, scale=sp.d ** -0.5, want_lse=True)
    got = pl.out[r0:r0 + S].float().cpu().numpy().astype(np.float64)
    glse = pl.lse[r0:r0 + S].cpu().numpy().astype(np.float64)
    err = np.abs(got[rows] - ref[rows]).max(-1) / np.maximum(np.abs(ref[rows]).max(-1), 1e-6)
    assert err.max() <= TOL, (i, float(err.max()))
    assert np.abs(glse[rows] - lse[rows]).max() <= 1e-3 * max(1.0, np.abs(lse).max())
    return float(err.max())


def run(sp: StreamSpec, n_batches: int, seed=3000, q_scale=1.0, sample=6, max_rows=None, fused=False):
    ds, pool, instr = make_stream(sp)
    o = oracle_for(sp, pool, instr)
    pl = gpu_pipeline(sp, pool, instr)
    pl.fused_kv = fused
    pl.qkv_seed, pl.q_scale = seed, q_scale
    rng = np.random.default_rng(0)
    worst = 0.0
    sp.n_batches = n_batches
    for b, (start, B) in enumerate(batch_plan(sp, ds.n)):
        batch = gen.make_batch(ds, start, B)
        r = o.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=(sp.max_prompt_tokens + 15) // 16)
        pl.stage_batch(batch)
        pl.step()
        pl.ctx.status_sync()
        np.testing.assert_array_equal(pl.u32(pl.hit[:B]), r.hit)
        picks = set(rng.choice(B, size=min(sample, B), replace=False).tolist())
        picks |= {int(np.argmax(r.hit)), int(np.argmin(r.hit)), B - 1}
        for i in sorted(picks):
            worst = max(worst, check_request(pl, r, i, sp, seed, q_scale, max_rows))
    return worst


def test_attention_c1_shape():
    run(StreamSpec(B=24), n_batches=4)


@pytest.mark.parametrize("d", [64, 128])
def test_attention_fused_kv_into_pages(d):
    # il_synth_qkv_paged writes the suffix K / V into the pages, il_prefill_attn skips its append
    sp = StreamSpec(B=24, k=5, Hq=32 if d == 128 else 4, Hkv=8 if d == 128 else 4, d=d, max_prompt_tokens=1024)
    run(sp, n_batches=4, fused=True, sample=10)


def test_attention_llama_gqa_shape():
    run(StreamSpec(B=16, k=5, Hq=32, Hkv=8, d=128, max_prompt_tokens=1024), n_batches=3)


def test_attention_peaky_q():
    # Q scale 8 stresses the online-softmax rescaling (SURVEY d.1 'peaky')
    run(StreamSpec(B=16, k=5, Hq=32, Hkv=8, d=128, max_prompt_tokens=1024), n_batches=2, q_scale=8.0)


def test_attention_qwen_shape_k8():
    run(StreamSpec(B=12, k=8, Hq=40, Hkv=8, d=128, max_prompt_tokens=1536), n_batches=2)


def test_attention_long_prompts():
    sp = StreamSpec(n_logs=4096, n_templates=300, zipf=1.1, seed=4000, pool_seed=4001, k=5, B=8, n_instr=1836,
                    T=4096, C=4096, max_prompt_tokens=2560, Hq=32, Hkv=8, d=128, ramp=(1,))
    run(sp, n_batches=3, sample=3, max_rows=48)


def _long(B, ramp=(1,)):
    return StreamSpec(n_logs=4096, n_templates=300, zipf=1.1, seed=4000, pool_seed=4001, k=5, B=B, n_instr=1836,
                      T=4096, C=8192, max_prompt_tokens=2560, Hq=32, Hkv=8, d=128, ramp=ramp)


def test_attention_long_prompts_wide_batch():
    # B = 64: the cascade's dense phase-1 M-tiles span several requests each
    run(_long(64), n_batches=2, sample=10, max_rows=48)


def test_attention_long_prompts_no_cascade(monkeypatch):
    # IL_CASCADE=0: one phase over each request's whole prefix (the NC = 0 path)
    monkeypatch.setenv("IL_CASCADE", "0")
    run(_long(16), n_batches=2, sample=6, max_rows=48)


def test_attention_eviction_pressure_uneven_hits():
    # requests of one batch with fewer cached blocks than the batch-wide shared prefix bound (LRU
    # pressure, cold ramp): the cascade's shared range must shrink to the smallest hit count
    # (a request whose M-tiles started inside it would have no phase-2 KV tile)
    sp = StreamSpec(B=64, C=700, n_logs=3000, Hq=4, Hkv=4, d=128,
                    flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD, ramp=(4, 16))
    run(sp, n_batches=14, sample=8)
