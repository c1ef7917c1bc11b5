"""GPU vs oracle, bit-exact, over whole synthetic streams (integer stages a1-a7, a9)."""
import dataclasses

import numpy as np
import pytest

import oracle as O
from tests.parity_util import (StreamSpec, batch_plan, compare_batch, compare_state, gpu_pipeline, make_stream,
                               oracle_for)
from workload import gen

pytestmark = pytest.mark.gpu


def run_stream(sp: StreamSpec, state_every: int = 1):
    ds, pool, instr = make_stream(sp)
    o = oracle_for(sp, pool, instr)
    pl = gpu_pipeline(sp, pool, instr)
    hits = full = 0
    plan = batch_plan(sp, ds.n)
    nb = len(plan)
    for b, (start, B) in enumerate(plan):
        batch = gen.make_batch(ds, start, B)
        r = o.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=(sp.max_prompt_tokens + 15) // 16)
        pl.stage_batch(batch)
        pl.refine(); pl.match(); pl.commit()
        pl.ctx.status_sync()
        compare_batch(r, pl, B, sp, where=f"batch {b}")
        if b % state_every == 0 or b == nb - 1:
            compare_state(o, pl, where=f"after batch {b}")
        hits += int(r.hit.sum()); full += int((r.prompt_len // 16).sum())
    st = pl.ctx.stats()
    return hits / max(full, 1), st


def test_c1_stream_pair():
    rate, st = run_stream(StreamSpec())
    assert 0 < rate <= 1


def test_c1_stream_eviction_pressure_guard():
    # C small enough that almost every batch evicts; guard on; tombstone rebuilds happen
    sp = StreamSpec(C=700, B=32, T=64, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD, n_batches=240)
    rate, st = run_stream(sp, state_every=5)
    assert st["index_rebuilds"] >= 1


def test_naive_pc_and_jaccard_exclude_self():
    run_stream(StreamSpec(flags=O.F_VERIFY, n_batches=8))
    run_stream(StreamSpec(metric=O.SIM_JACCARD, flags=O.F_PAIR | O.F_VERIFY | O.F_EXCLUDE_SELF, n_batches=8))


def test_batch_size_one_and_ragged():
    # B = 1 is the paper's sequential semantics; B = 37 leaves a ragged last batch of the pool walk
    run_stream(StreamSpec(B=1, n_batches=150, C=300, T=16))
    run_stream(StreamSpec(B=37, n_batches=20, k=5, C=900, T=40, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD))


def test_k8_large_pool():
    # k = 8, 2,000-demo pool (config-4-like selection), many templates
    sp = StreamSpec(n_logs=6000, n_templates=300, zipf=1.3, M=2000, k=8, B=256, T=256, C=8192,
                    max_prompt_tokens=1024, n_batches=6)
    run_stream(sp, state_every=2)


def test_long_instruction_c3_shape():
    # ~2k-token prompts (1,836-token instruction, not block aligned): config-3 shape, small B
    sp = StreamSpec(n_logs=4096, n_templates=300, zipf=1.1, seed=4000, M=200, pool_seed=4001, k=5, B=128,
                    n_instr=1836, T=4096, C=6000, max_prompt_tokens=2560, n_batches=8, ramp=(1, 8),
                    flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD)
    run_stream(sp, state_every=4)


def test_graph_replay_stream_bit_exact():
    """Per-stage CUDA-graph replays (bench's launch mode) advance the device state exactly like
    eager calls: batch counter, index, table (all on the device)."""
    import torch
    sp = StreamSpec(B=64, C=1200, n_logs=2000, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD, ramp=(64,))
    ds, pool, instr = make_stream(sp)
    o = oracle_for(sp, pool, instr)
    pl = gpu_pipeline(sp, pool, instr)
    sp.n_batches = 12
    plan = batch_plan(sp, ds.n)
    for b, (start, B) in enumerate(plan):
        batch = gen.make_batch(ds, start, B)
        r = o.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=(sp.max_prompt_tokens + 15) // 16)
        pl.stage_batch(batch)
        if b == 0:
            pl.step(attention=False)                   # eager once (one-time attributes)
        else:
            if b == 1:
                graphs = pl.capture(B, stages=("refine", "match", "commit"))
            for n in ("refine", "match", "commit"):
                graphs[n].replay()
        torch.cuda.synchronize()
        pl.ctx.status_sync()
        compare_batch(r, pl, B, sp, where=f"graph batch {b}")
        compare_state(o, pl, where=f"graph batch {b}")
    assert pl.ctx.stats()["batch"] == len(plan)


def test_c4_full_pool_10k_k8():
    """BASELINE configs[3] selection at full size: a 10,000-demo pool, k = 8, B = 1,024, 1,000
    templates with Zipf 1.3 (bench.workload(4)); integer path bit-exact for 5 batches."""
    import bench
    cfg, ds, pool, instr = bench.workload(4, 0, 1, n_queries=6 * 1024)
    sp = StreamSpec(M=cfg.M, k=cfg.k, B=cfg.B, n_instr=cfg.n_instr, T=cfg.T, C=cfg.C,
                    max_prompt_tokens=cfg.max_prompt_tokens, Hq=cfg.Hq, Hkv=cfg.Hkv, d=cfg.d,
                    flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD)
    o = oracle_for(sp, pool, instr)
    pl = gpu_pipeline(sp, pool, instr)
    for b in range(5):
        batch = gen.make_batch(ds, b * cfg.B, cfg.B)
        r = o.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=sp.max_prompt_tokens // 16)
        pl.stage_batch(batch)
        pl.refine(); pl.match(); pl.commit()
        pl.ctx.status_sync()
        compare_batch(r, pl, cfg.B, sp, where=f"c4 batch {b}")
        compare_state(o, pl, where=f"c4 batch {b}")


def test_large_pool_jaccard_exclude_self():
    # inverted-index selection (pool > 1,024 demos) with Jaccard over token sets and self-exclusion
    sp = StreamSpec(n_logs=6000, n_templates=300, zipf=1.3, M=3000, k=5, B=128, T=256, C=4096,
                    max_prompt_tokens=1024, n_batches=4, metric=O.SIM_JACCARD,
                    flags=O.F_PAIR | O.F_VERIFY | O.F_EXCLUDE_SELF)
    run_stream(sp, state_every=2)


def test_multi_chunk_pool_20k():
    # 20,000 demos = two 16,384-demo chunks of the inverted index (accumulators per chunk, top-k
    # carried across chunks), cosine, k = 8
    sp = StreamSpec(n_logs=40000, n_templates=1000, zipf=1.3, M=20000, k=8, B=96, T=512, C=8192,
                    max_prompt_tokens=1536, n_batches=3)
    run_stream(sp, state_every=3)


def test_c5_pool_50k_selection():
    """BASELINE configs[4] selection: the 50,000-demo pool sampled from the full 10,485,760-log
    stream (bench.workload(5)), k = 5, four chunks of the inverted index; two batches of 128
    requests bit-exact (the oracle scores every demo of the pool for every query)."""
    import bench
    cfg, ds, pool, instr = bench.workload(5, 0, 1)
    sp = StreamSpec(M=cfg.M, k=cfg.k, B=128, n_instr=cfg.n_instr, T=cfg.T, C=8192,
                    max_prompt_tokens=cfg.max_prompt_tokens, Hq=cfg.Hq, Hkv=cfg.Hkv, d=cfg.d,
                    flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD)
    o = oracle_for(sp, pool, instr)
    pl = gpu_pipeline(sp, pool, instr)
    for b in range(2):
        batch = gen.make_batch(ds, b * sp.B, sp.B)
        r = o.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=sp.max_prompt_tokens // 16)
        pl.stage_batch(batch)
        pl.refine(); pl.match(); pl.commit()
        pl.ctx.status_sync()
        compare_batch(r, pl, sp.B, sp, where=f"c5 batch {b}")
        compare_state(o, pl, where=f"c5 batch {b}")
