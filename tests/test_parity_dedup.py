"""NEXT-1 in-batch dedup (IL_F_DEDUP; Z22b) on the GPU vs the oracle (OR_F_DEDUP).

Integer stages bit-exact (hits after dedup, evictions, index, table, prefix_len / cu_q), the
per-batch dedup counter against the oracle's hits with and without dedup, the attention of
requests whose block tables point at ANOTHER request's freshly computed pages (cold batches share
the instruction and demonstrations that way), and the data-parallel path (dedup per rank)."""
import numpy as np
import pytest

import oracle as O
from tests.parity_util import StreamSpec, batch_plan, gpu_pipeline, make_stream, oracle_for
from tests.test_parity_attn import run as run_attn
from tests.test_parity_dp import run_dp
from tests.test_parity_int import run_stream
from workload import gen

pytestmark = pytest.mark.gpu

DD = O.F_PAIR | O.F_VERIFY | O.F_DEDUP


def test_dedup_c1_stream_cold_start():
    run_stream(StreamSpec(flags=DD, ramp=(100,)))


def test_dedup_eviction_pressure_guard():
    sp = StreamSpec(C=700, B=32, T=64, flags=DD | O.F_GUARD, n_batches=200)
    rate, st = run_stream(sp, state_every=5)
    assert st["index_rebuilds"] >= 1


def test_dedup_c3_shape_and_naive():
    sp = StreamSpec(n_logs=4096, n_templates=300, zipf=1.1, seed=4000, M=200, pool_seed=4001, k=5, B=128,
                    n_instr=1836, T=4096, C=6000, max_prompt_tokens=2560, n_batches=6, ramp=(1, 8, 128),
                    flags=DD | O.F_GUARD)
    run_stream(sp, state_every=3)
    run_stream(StreamSpec(flags=O.F_VERIFY | O.F_DEDUP, n_batches=8))      # naive prefix caching + dedup
    run_stream(StreamSpec(B=1, n_batches=40, C=300, T=16, flags=DD))       # B = 1: nothing to share


def test_dedup_counter_matches_oracle():
    sp = StreamSpec(B=100, n_logs=800, C=4096, flags=DD)
    ds, pool, instr = make_stream(sp)
    o = oracle_for(sp, pool, instr)
    plain = O.Oracle(sp.k, sp.T, sp.C, metric=sp.metric, flags=O.F_PAIR | O.F_VERIFY, hash_seed=sp.hash_seed)
    plain.pool_load(pool, instr)
    pl = gpu_pipeline(sp, pool, instr)
    MB = (sp.max_prompt_tokens + 15) // 16
    seen = 0
    for b, (start, B) in enumerate(batch_plan(sp, ds.n)):
        if b == 3:
            break
        batch = gen.make_batch(ds, start, B)
        r = o.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=MB)
        # the same snapshot without dedup: only while both indices hold the same blocks (batch 0)
        r0 = plain.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=MB)
        pl.stage_batch(batch)
        pl.refine(); pl.match(); pl.commit()
        st = pl.ctx.stats()
        np.testing.assert_array_equal(pl.u32(pl.hit[:B]), r.hit)
        assert st["hit_blocks"] == int(r.hit.sum())
        if b == 0:
            assert st["dedup_blocks"] == int((r.hit - r0.hit).sum()) > 0
        seen += st["dedup_blocks"]
    assert seen > 0


@pytest.mark.parametrize("fused", [False, True])
def test_dedup_attention_reads_owner_pages(fused):
    # cold start: request 0 computes the instruction, every later request of batch 0 reads it
    # from request 0's pages (and shared demonstrations from their first user's)
    sp = StreamSpec(flags=DD, ramp=(100,), C=4096)
    assert run_attn(sp, n_batches=4, sample=10, fused=fused) <= 1e-2


def test_dedup_attention_long_prompts_gqa():
    sp = StreamSpec(n_logs=4096, n_templates=300, zipf=1.1, seed=4000, M=200, pool_seed=4001, k=5, B=64,
                    n_instr=1836, T=4096, C=6000, max_prompt_tokens=2560, Hq=8, Hkv=2, d=128, flags=DD,
                    ramp=(64,))
    assert run_attn(sp, n_batches=3, sample=4, max_rows=64, fused=True) <= 1e-2


def test_dedup_dp2_with_attention():
    sp = StreamSpec(B=96, C=1200, n_logs=2000, flags=DD, ramp=(96,))
    run_dp(sp, 2, 8, attention=True)
