"""Multi-GPU data parallelism vs the oracle's run_batch_dp, bit-exact.

Only one GPU exists on the test box, so the G ranks are G independent library contexts on the
same device; the per-batch record all-gather is what DataParallel.commit feeds to
il_commit_records (rank-major concatenation = global admission order; the collective itself is
covered over gloo in test_distributed_gloo.py).  Checked per rank after every batch: topk,
final DS, rule/PMC/guard, prompts, block hashes, hits, evictions, the rank's prefix index, and
the replicated ICL Table, and (il_commit_export / il_commit_apply) every request's box-level hit
count from the replicated residency map."""
import numpy as np
import pytest
import torch

import oracle as O
from tests.parity_util import StreamSpec, batch_plan, compare_batch, compare_state, make_stream
from workload import gen

pytestmark = pytest.mark.gpu


def _rank_pipeline(sp, pool, instr, G, rec_R=None):
    from paper_2507_08523_b200 import Config, Pipeline
    cfg = Config(k=sp.k, table_capacity=sp.T, kv_pages=sp.C, max_batch=sp.B // G,
                 max_prompt_tokens=sp.max_prompt_tokens, max_pool=sp.M,
                 max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16, max_log_tokens=255,
                 n_q_heads=sp.Hq, n_kv_heads=sp.Hkv, head_dim=sp.d, metric=sp.metric, flags=sp.flags,
                 hash_seed=sp.hash_seed, max_global_batch=sp.B,
                 # room for every block record of a batch (no FIFO backlog: the map is exact)
                 max_block_records=rec_R or 2 * (sp.B // G) * ((sp.max_prompt_tokens + 15) // 16))
    pl = Pipeline(cfg, "cuda")
    pl.load_pool(pool, instr)
    return pl


class _Slice:
    """Rows [lo, hi) of a global oracle result, shaped like a one-rank BatchResult."""
    def __init__(self, r, lo, hi, evicted):
        for f in ("topk", "final_ds", "info", "target_stamp", "prompt_len", "prompt_tok", "block_hash", "hit"):
            setattr(self, f, getattr(r, f)[lo:hi])
        self.evicted = evicted


def run_dp(sp: StreamSpec, G: int, n_batches: int, attention: bool = False, records: bool = True,
           rec_R=None):
    """records=True: the rank's record buffers (il_commit_export) concatenated rank-major, as the
    all-gather delivers them, applied on every rank with il_commit_apply (ICL table + residency
    map; box-level hits compared too).  records=False: il_commit_records over the concatenated
    ICL records (the table half alone)."""
    ds, pool, instr = make_stream(sp)
    ranks_o = []
    for _ in range(G):
        o = O.Oracle(sp.k, sp.T, sp.C, metric=sp.metric, flags=sp.flags, hash_seed=sp.hash_seed)
        o.pool_load(pool, instr)
        ranks_o.append(o)
    pls = [_rank_pipeline(sp, pool, instr, G, rec_R) for _ in range(G)]
    exact = rec_R is None
    max_backlog = 0
    k = sp.k
    fds_all = torch.zeros(sp.B, k, dtype=torch.int32, device="cuda")
    info_all = torch.zeros(sp.B, 16, dtype=torch.uint8, device="cuda")
    rb = pls[0].cfg.record_bytes()
    recs = torch.zeros(G, rb, dtype=torch.uint8, device="cuda")
    sp.n_batches = n_batches
    box_gain = 0
    for b, (start, B) in enumerate(batch_plan(sp, ds.n)):
        assert B % G == 0
        batch = gen.make_batch(ds, start, B)
        r = O.Oracle.run_batch_dp(ranks_o, batch, prompt_stride=sp.max_prompt_tokens,
                                  max_blocks=(sp.max_prompt_tokens + 15) // 16)
        n = B // G
        for g, pl in enumerate(pls):
            pl.stage_batch(gen.make_batch(ds, start + g * n, n))
            if records:
                pl.ctx.select_batch(n, pl.q_off, pl.q_tok, pl.q_src, pl.topk)   # a1-a2 ahead, as DataParallel
            pl.refine(); pl.match()
            if attention:
                pl.synth(); pl.attn()
            pl.ctx.commit_index()
            if records:
                pl.ctx.commit_export(recs[g])
        if records:
            for pl in pls:
                pl.ctx.commit_apply(recs, [n] * G)
        else:
            # the all-gather: rank-major rows = global admission order
            torch.cat([pl.final_ds[:n] for pl in pls], out=fds_all[:B])
            torch.cat([pl.info[:n] for pl in pls], out=info_all[:B])
            for pl in pls:
                pl.ctx.commit_records(B, fds_all, info_all)
        for g, pl in enumerate(pls):
            pl.ctx.status_sync()
            compare_batch(_Slice(r, g * n, (g + 1) * n, r.evicted_rank[g]), pl, n, sp, where=f"batch {b} rank {g}")
            compare_state(ranks_o[g], pl, where=f"batch {b} rank {g}")
            if records:
                st = pl.ctx.stats()
                max_backlog = max(max_backlog, st["record_backlog"])
                if not exact:                          # a lagging map: box hits stay >= local hits
                    assert (pl.ctx.box_hit_dump(n) >= pl.u32(pl.hit[:n])).all()
                    continue
                assert st["record_backlog"] == 0, (b, g, st["record_backlog"])
                if b > 0:                              # box hits of batch b read the map of batch b-1
                    np.testing.assert_array_equal(pl.ctx.box_hit_dump(n), r.box_hit[g * n:(g + 1) * n],
                                                  err_msg=f"batch {b} rank {g} box hits")
                    assert st["box_hit_blocks"] == int(r.box_hit[g * n:(g + 1) * n].sum())
                    assert st["hit_blocks"] == int(r.hit[g * n:(g + 1) * n].sum())
                    box_gain += int(r.box_hit[g * n:(g + 1) * n].sum() - r.hit[g * n:(g + 1) * n].sum())
    if records and G > 1 and exact:
        assert box_gain > 0, "remote residency should show in the box-level hits"
    if not exact:
        assert max_backlog > 0, "the small record window should have queued records"
    return pls


def test_dp2_no_guard():
    run_dp(StreamSpec(B=96, C=1700, n_logs=2000), G=2, n_batches=10)


def test_dp2_commit_records_table_half():
    run_dp(StreamSpec(B=96, C=1700, n_logs=2000, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD), G=2, n_batches=6,
           records=False)


def test_dp2_guard():
    run_dp(StreamSpec(B=96, C=1700, n_logs=2000, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD), G=2, n_batches=10)


def test_dp4_eviction_pressure_with_attention():
    sp = StreamSpec(B=64, C=700, n_logs=3000, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD, ramp=(4, 16))
    run_dp(sp, G=4, n_batches=14, attention=True)


def test_dp8_guard():
    # G = 8 ranks (the box size of SURVEY §8(e)), 16 requests per rank
    run_dp(StreamSpec(B=128, C=600, n_logs=3000, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD, ramp=(8, 64)),
           G=8, n_batches=10)


def test_dp4_small_record_window_backlog():
    # 8 block records per export: most batches queue records in the FIFO (backlog), the table,
    # index and hits stay exact, box-level hits stay >= local hits, nothing latches
    sp = StreamSpec(B=64, C=700, n_logs=3000, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD, ramp=(4, 16))
    run_dp(sp, G=4, n_batches=14, rec_R=8)
