"""Edge cases and error behaviour of the boundary on the GPU (include/il.h): empty batches,
host-detected argument errors, and device-latched capacity / length errors."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2507_08523_b200 import _lib as L
from tests.parity_util import StreamSpec, compare_batch, compare_state, gpu_pipeline, make_stream, oracle_for
from workload import gen

pytestmark = pytest.mark.gpu


def test_empty_batch_is_a_noop_for_the_path():
    sp = StreamSpec(B=24, C=2048)
    ds, pool, instr = make_stream(sp)
    o, pl = oracle_for(sp, pool, instr), gpu_pipeline(sp, pool, instr)
    batch = gen.make_batch(ds, 0, sp.B)
    r = o.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=sp.max_prompt_tokens // 16)
    pl.stage_batch(batch); pl.step(); pl.ctx.status_sync()
    compare_batch(r, pl, sp.B, sp, where="before")
    before = pl.ctx.index_dump(), pl.ctx.table_dump()
    for call in (pl.refine, pl.match, pl.synth, pl.attn):   # B = 0: every call returns IL_OK at once
        call(0)
    pl.ctx.status_sync()
    after = pl.ctx.index_dump(), pl.ctx.table_dump()
    for a, b in zip(before[0] + before[1], after[0] + after[1]):
        np.testing.assert_array_equal(a, b)


def test_host_detected_argument_errors():
    sp = StreamSpec(B=8, C=512)
    ds, pool, instr = make_stream(sp)
    pl = gpu_pipeline(sp, pool, instr)
    pl.stage_batch(gen.make_batch(ds, 0, sp.B))
    with pytest.raises(L.ILError) as e:                    # B > max_batch
        pl.refine(sp.B + 1)
    assert e.value.status == L.IL_ERR_ARG
    with pytest.raises(L.ILError) as e:                    # prompt rows not 16-byte aligned
        pl.ctx.refine_batch(sp.B, pl.q_off, pl.q_tok, pl.q_src, pl.topk, pl.final_ds, pl.info,
                            pl.prompt_tok.view(-1)[1:], pl.prompt_len)
    assert e.value.status == L.IL_ERR_ARG


def test_round2_call_argument_errors():
    """il_set_sm_split, il_decode_attn, il_synth_qkv_paged: host-detected misuse."""
    sp = StreamSpec(B=8, C=512)
    ds, pool, instr = make_stream(sp)
    pl = gpu_pipeline(sp, pool, instr)
    with pytest.raises(L.ILError) as e:                    # the attention grid must leave an SM
        pl.ctx.set_sm_split(10_000)
    assert e.value.status == L.IL_ERR_ARG
    pl.ctx.set_sm_split(0)
    B = sp.B
    with pytest.raises(L.ILError) as e:                    # decode before il_prefix_match
        pl.ctx.decode_attn(B, pl.prefix_len, pl.block_table, pl.q, None, None, pl.k_pages, pl.v_pages,
                           pl.out, None, 0.125)
    assert e.value.status == L.IL_ERR_STATE
    pl.stage_batch(gen.make_batch(ds, 0, B))
    pl.refine(); pl.match()
    with pytest.raises(L.ILError) as e:                    # k_new without v_new
        pl.ctx.decode_attn(B, pl.prefix_len, pl.block_table, pl.q, pl.k_new, None, pl.k_pages, pl.v_pages,
                           pl.out, None, 0.125)
    assert e.value.status == L.IL_ERR_ARG
    with pytest.raises(L.ILError) as e:                    # B > max_batch
        pl.ctx.decode_attn(B + 1, pl.prefix_len, pl.block_table, pl.q, None, None, pl.k_pages, pl.v_pages,
                           pl.out, None, 0.125)
    assert e.value.status == L.IL_ERR_ARG
    with pytest.raises(L.ILError) as e:                    # k pages without v pages
        pl.ctx.synth_qkv_paged(B, pl.prompt_tok, pl.cu_q, pl.prefix_len, pl.block_table, 1, 1.0, pl.q,
                               pl.k_pages, None)
    assert e.value.status == L.IL_ERR_ARG
    pl.commit()
    pl.ctx.status_sync()


def test_device_latched_capacity_error():
    # a cold batch needs more pages than the cache has: il_prefix_match latches IL_ERR_CAPACITY
    sp = StreamSpec(B=32, C=40)
    ds, pool, instr = make_stream(sp)
    pl = gpu_pipeline(sp, pool, instr)
    pl.stage_batch(gen.make_batch(ds, 0, sp.B))
    pl.refine(); pl.match()
    with pytest.raises(L.ILError) as e:
        pl.ctx.status_sync()
    assert e.value.status == L.IL_ERR_CAPACITY


def test_device_latched_prompt_too_long():
    # instruction + k demonstrations + query longer than max_prompt_tokens: latched IL_ERR_ARG
    sp = StreamSpec(B=8, C=512, n_instr=300, max_prompt_tokens=320)
    ds, pool, instr = make_stream(sp)
    pl = gpu_pipeline(sp, pool, instr)
    pl.stage_batch(gen.make_batch(ds, 0, sp.B))
    pl.refine()
    with pytest.raises(L.ILError) as e:
        pl.ctx.status_sync()
    assert e.value.status == L.IL_ERR_ARG


def test_suffix_overflow_latches_and_writes_nothing_past_the_buffers():
    """More suffix rows than max_suffix_tokens (a cold batch): il_prefix_match latches
    IL_ERR_CAPACITY and publishes an empty suffix (cu_q = 0), so synth / K,V append / attention
    write nothing past the caller's [max_suffix_tokens] buffers (canary rows stay intact)."""
    sp = StreamSpec(B=24, C=2048)
    ds, pool, instr = make_stream(sp)
    rows = 64
    pl = gpu_pipeline(sp, pool, instr, max_suffix_tokens=rows)
    canary = {}
    for name in ("q", "k_new", "v_new", "out"):
        t = getattr(pl, name)
        big = torch.full((rows + 256,) + tuple(t.shape[1:]), 7.0, dtype=t.dtype, device=t.device)
        setattr(pl, name, big[:rows])
        canary[name] = big
    pl.stage_batch(gen.make_batch(ds, 0, sp.B))
    pl.refine(); pl.match(); pl.synth(); pl.attn()
    with pytest.raises(L.ILError) as e:
        pl.ctx.status_sync()
    assert e.value.status == L.IL_ERR_CAPACITY
    assert int(pl.cu_q[sp.B].item()) == 0
    for name, big in canary.items():
        assert bool((big[rows:] == 7.0).all()), name
