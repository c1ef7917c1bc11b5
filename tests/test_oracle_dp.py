"""Pins of the oracle's data-parallel batch procedure (oracle/oracle.cpp
run_batch_dp): rank r owns the r-th contiguous admission slice and its own prefix index; the ICL
Table is replicated and receives every record in global admission order.

What fixes it independently of the implementation:
  - with the guard off, refinement reads only the table, so the G-rank run must reproduce the
    one-rank run request for request (topk, final DS, rule, PMC) and table for table;
  - the replicated tables stay identical on every rank;
  - a rank's index only ever holds blocks of prompts that rank processed, and a request's hits
    are a prefix of its own block chain that is resident in its rank's index;
  - with one request per rank per batch, each rank's index is SPEC's sequential kv_sim over
    that rank's prompts.
"""
import numpy as np
import pytest

import oracle as O
from tests.parity_util import StreamSpec, batch_plan, make_stream
from workload import gen


def _ranks(sp, pool, instr, G):
    out = []
    for _ in range(G):
        o = O.Oracle(sp.k, sp.T, sp.C, metric=sp.metric, flags=sp.flags, hash_seed=sp.hash_seed)
        o.pool_load(pool, instr)
        out.append(o)
    return out


def _run(sp, G, n_batches):
    ds, pool, instr = make_stream(sp)
    ranks = _ranks(sp, pool, instr, G)
    sp.n_batches = n_batches
    res = []
    for start, B in batch_plan(sp, ds.n):
        r = O.Oracle.run_batch_dp(ranks, gen.make_batch(ds, start, B), prompt_stride=sp.max_prompt_tokens,
                                  max_blocks=(sp.max_prompt_tokens + 15) // 16)
        res.append((B, r, [o.table_dump() for o in ranks], [o.index_dump() for o in ranks]))
    return res


SP = dict(B=96, C=1700, n_logs=2000)


@pytest.mark.parametrize("G", [2, 4])
def test_dp_refinement_equals_one_rank_without_guard(G):
    one = _run(StreamSpec(**SP), 1, 8)
    many = _run(StreamSpec(**SP), G, 8)
    for b, ((B, r1, t1, _), (_, rg, tg, _)) in enumerate(zip(one, many)):
        np.testing.assert_array_equal(r1.topk, rg.topk, err_msg=f"batch {b}")
        np.testing.assert_array_equal(r1.final_ds, rg.final_ds, err_msg=f"batch {b}")
        np.testing.assert_array_equal(r1.info, rg.info, err_msg=f"batch {b}")
        np.testing.assert_array_equal(r1.target_stamp, rg.target_stamp, err_msg=f"batch {b}")
        np.testing.assert_array_equal(r1.prompt_len, rg.prompt_len, err_msg=f"batch {b}")
        for t in tg:                                   # replicated, and equal to the one-rank table
            for a, c in zip(t1[0], t):
                np.testing.assert_array_equal(a, c, err_msg=f"batch {b}")


def test_dp_tables_stay_replicated_with_guard():
    sp = StreamSpec(**SP, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD)
    for b, (B, r, tabs, _) in enumerate(_run(sp, 2, 8)):
        for t in tabs[1:]:
            for a, c in zip(tabs[0], t):
                np.testing.assert_array_equal(a, c, err_msg=f"batch {b}")


def test_dp_rank_index_holds_only_its_own_blocks_and_hits_are_resident_prefixes():
    sp = StreamSpec(**SP)
    G = 2
    seen = [set() for _ in range(G)]
    prev_index = [set() for _ in range(G)]
    for b, (B, r, _, idx) in enumerate(_run(sp, G, 8)):
        for i in range(B):
            g = next(q for q in range(G) if q * B // G <= i < (q + 1) * B // G)
            L = int(r.prompt_len[i])
            nb = L // 16
            chain = r.block_hash[i, :nb]
            seen[g].update(int(x) for x in chain)
            h = int(r.hit[i])
            assert h <= max(0, (L - 1) // 16)
            # hits: leading blocks resident in this rank's index before the batch (snapshot, Z1)
            for j in range(h):
                assert int(chain[j]) in prev_index[g], (b, i, j)
            if h < min(nb, (L - 1) // 16):               # the longest resident prefix
                assert int(chain[h]) not in prev_index[g], (b, i, h)
        for g in range(G):
            hashes = set(int(x) for x in idx[g][0])
            assert hashes <= seen[g], f"rank {g} holds a block it never computed"
            prev_index[g] = hashes


@pytest.mark.parametrize("G", [2, 4])
def test_dp_one_request_per_rank_is_sequential_kv_sim_per_rank(G):
    """With one request per rank per batch (B = G) and an unbounded cache, each rank's prefix
    index is SPEC's sequential kv_sim over the prompts that rank processed: the hit
    of every request equals lookup (capped, Z20) then insert on a per-rank sequential oracle, and
    the resident sets agree.  Independent of run_batch_dp's own code path (or_lookup/or_insert)."""
    sp = StreamSpec(B=G, n_logs=600, C=1 << 20)
    ds, pool, instr = make_stream(sp)
    ranks = _ranks(sp, pool, instr, G)
    seq = _ranks(sp, pool, instr, G)
    for b in range(60):
        r = O.Oracle.run_batch_dp(ranks, gen.make_batch(ds, b * G, G), prompt_stride=sp.max_prompt_tokens,
                                  max_blocks=sp.max_prompt_tokens // 16)
        for g in range(G):
            p = r.prompt(g)
            assert seq[g].lookup(p, capped=True) == int(r.hit[g]), (b, g)
            seq[g].insert(p)
            assert (ranks[g].index_dump()[0] == seq[g].index_dump()[0]).all(), (b, g)


@pytest.mark.parametrize("G", [1, 2, 4])
def test_dp_residency_map_is_union_of_rank_indices_and_box_hits_are_box_prefixes(G):
    """§8(e) residency map: after every batch, on every rank, hash -> owner mask equals the union
    of the ranks' prefix indices (brute force from the index dumps); a request's box-level hit is
    the longest leading run of its blocks resident on ANY rank at the snapshot (brute force from
    the previous batch's dumps), capped as Z20; it is >= the rank-local hit and equal to it at G = 1."""
    sp = StreamSpec(B=96, C=1800 // G, n_logs=2000, flags=O.F_PAIR | O.F_VERIFY | O.F_GUARD)
    ds, pool, instr = make_stream(sp)
    ranks = _ranks(sp, pool, instr, G)
    prev_union = {}
    gained_on_others = 0
    for b in range(10):
        r = O.Oracle.run_batch_dp(ranks, gen.make_batch(ds, b * sp.B, sp.B), prompt_stride=sp.max_prompt_tokens,
                                  max_blocks=sp.max_prompt_tokens // 16)
        for i in range(sp.B):
            L = int(r.prompt_len[i])
            chain = [int(x) for x in r.block_hash[i, :L // 16]]
            run = 0
            while run < len(chain) and chain[run] in prev_union:
                run += 1
            want = min(max(run, int(r.hit[i])), max(L - 1, 0) // 16)
            assert int(r.box_hit[i]) == want, (b, i)
            assert r.box_hit[i] >= r.hit[i]
            if G == 1:
                assert r.box_hit[i] == r.hit[i]
            gained_on_others += int(r.box_hit[i] > r.hit[i])
        union = {}
        for g, o in enumerate(ranks):
            for x in o.index_dump()[0]:
                union[int(x)] = union.get(int(x), 0) | (1 << g)
        for o in ranks:
            h, m = o.box_map_dump()
            assert dict(zip((int(x) for x in h), (int(y) for y in m))) == union, b
        prev_union = union
    if G > 1:
        assert gained_on_others > 0          # remote residency is visible in the box-level hits
