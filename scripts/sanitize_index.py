"""compute-sanitizer driver: a small stream under eviction pressure through the
index paths -- k_hash_match, k_alloc_scan, cooperative k_evict, k_alloc_fill, lock-free
k_commit_insert / k_commit_own, cooperative k_rebuild (tombstone compaction), the ICL-Table
commit (k_tab_key / k_tab_find / k_tab_commit) -- and, with --attn, the attention call; every
batch is checked bit-exact against the CPU oracle, so a race that changes a result fails too.

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python scripts/sanitize_index.py [--attn] [--dedup]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from tests.parity_util import StreamSpec, batch_plan, compare_batch, compare_state, gpu_pipeline, make_stream, oracle_for  # noqa: E402
from workload import gen  # noqa: E402


def main_dp():
    """Two emulated ranks through il_commit_export / il_commit_apply (record FIFO, residency map
    with its cooperative rebuild, gathered ICL records), checked against run_batch_dp."""
    from tests.test_parity_dp import run_dp
    sp = StreamSpec(B=32, C=300, n_logs=2000, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD, ramp=(4, 16))
    run_dp(sp, G=2, n_batches=int(os.environ.get("NB", "20")), attention=False)
    print("sanitize_index --dp: bit-exact")


def main():
    if "--dp" in sys.argv:
        return main_dp()
    attn = "--attn" in sys.argv
    # 160 KV pages for 8 ~15-page prompts per batch: most batches evict, tombstones force rebuilds
    dedup = "--dedup" in sys.argv                     # IL_F_DEDUP: the in-batch table and owner pages
    sp = StreamSpec(C=160, B=8, T=32, n_logs=1200, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD | (O.F_DEDUP if dedup else 0),
                    n_batches=int(os.environ.get("NB", "60")), ramp=(2, 4))
    ds, pool, instr = make_stream(sp)
    o = oracle_for(sp, pool, instr)
    pl = gpu_pipeline(sp, pool, instr)
    ev = 0
    for b, (start, B) in enumerate(batch_plan(sp, ds.n)):
        batch = gen.make_batch(ds, start, B)
        r = o.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=sp.max_prompt_tokens // 16)
        pl.stage_batch(batch)
        pl.step(attention=attn)
        pl.ctx.status_sync()
        compare_batch(r, pl, B, sp, where=f"batch {b}")
        compare_state(o, pl, where=f"batch {b}")
        ev += len(r.evicted) > 0
    st = pl.ctx.stats()
    print(f"sanitize_index: {b + 1} batches bit-exact, {ev} evicting, {st['index_rebuilds']} index rebuilds, "
          f"attention={attn}, dedup={dedup}")


if __name__ == "__main__":
    main()
