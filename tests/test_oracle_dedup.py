"""Pins of the oracle's in-batch dedup (NEXT-1, OR_F_DEDUP; Z22b).

What fixes it independently of the owner table the oracle builds:
  - a full block that an earlier request of the batch also has at the same depth after the same
    prefix is computed once, so request i's effective hit count is the longest whole-block common
    prefix with ANY earlier request of the batch, or its snapshot hit count if longer, capped so
    that the last prompt token is computed (Z20):
        h_i = min(floor((L_i - 1) / 16), max(h_i^snapshot, max_{o < i} LCP_blocks(i, o)));
    brute force over all pairs, the snapshot hits taken from the run WITHOUT dedup (same tables,
    same index key set while nothing is evicted);
  - dedup changes which request computes a block, never which blocks become resident: without
    eviction the index holds the same hashes with and without dedup;
  - the pages a cold batch needs are sum_i ceil(L_i / 16) - h_i: exactly that many pages succeed,
    one fewer is IL_ERR_CAPACITY.
"""
import numpy as np
import pytest

import oracle as O
from tests.parity_util import StreamSpec, batch_plan, make_stream
from workload import gen

BS = 16


def _lcp_blocks(a: np.ndarray, b: np.ndarray) -> int:
    n = min(len(a), len(b)) // BS
    x = (a[:n * BS] != b[:n * BS]).reshape(n, BS).any(axis=1) if n else np.zeros(0, bool)
    bad = np.flatnonzero(x)
    return int(bad[0]) if len(bad) else n


def _oracle(sp, pool, instr, flags, C=None):
    o = O.Oracle(sp.k, sp.T, C if C is not None else sp.C, metric=sp.metric, flags=flags, hash_seed=sp.hash_seed)
    o.pool_load(pool, instr)
    return o


def _expected(r, B, h_snap):
    P = [r.prompt(i) for i in range(B)]
    out = np.zeros(B, np.int64)
    for i in range(B):
        best = int(h_snap[i])
        for o in range(i):
            best = max(best, _lcp_blocks(P[i], P[o]))
        out[i] = min((len(P[i]) - 1) // BS, best)
    return out


@pytest.mark.parametrize("cfg", [dict(B=100, n_logs=1200), dict(B=64, n_logs=900, k=5, max_prompt_tokens=768)])
def test_dedup_hits_are_batch_lcp(cfg):
    sp = StreamSpec(C=1 << 20, **cfg)
    ds, pool, instr = make_stream(sp)
    plain = _oracle(sp, pool, instr, sp.flags)
    dd = _oracle(sp, pool, instr, sp.flags | O.F_DEDUP)
    MB = (sp.max_prompt_tokens + 15) // 16
    gained = 0
    for b, (start, B) in enumerate(batch_plan(sp, ds.n)):
        batch = gen.make_batch(ds, start, B)
        r0 = plain.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=MB)
        r1 = dd.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=MB)
        np.testing.assert_array_equal(r0.final_ds, r1.final_ds, err_msg=f"batch {b}")
        np.testing.assert_array_equal(r0.prompt_len, r1.prompt_len, err_msg=f"batch {b}")
        exp = _expected(r1, B, r0.hit)
        np.testing.assert_array_equal(r1.hit.astype(np.int64), exp, err_msg=f"batch {b}")
        assert (r1.hit >= r0.hit).all()
        gained += int((r1.hit - r0.hit).sum())
        k0 = np.sort(plain.index_dump()[0])
        k1 = np.sort(dd.index_dump()[0])
        np.testing.assert_array_equal(k0, k1, err_msg=f"batch {b}: resident set")
    assert gained > 0                                  # the cold batch alone shares the instruction


def test_dedup_cold_batch_page_count():
    sp = StreamSpec(B=80, n_logs=400)
    ds, pool, instr = make_stream(sp)
    MB = (sp.max_prompt_tokens + 15) // 16
    batch = gen.make_batch(ds, 0, sp.B)
    probe = _oracle(sp, pool, instr, sp.flags | O.F_DEDUP, C=1 << 20)
    r = probe.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=MB)
    h = _expected(r, sp.B, np.zeros(sp.B, np.int64))
    need = int(sum((int(L) + BS - 1) // BS for L in r.prompt_len) - h.sum())
    plain_need = int(sum((int(L) + BS - 1) // BS for L in r.prompt_len))
    assert need < plain_need
    ok = _oracle(sp, pool, instr, sp.flags | O.F_DEDUP, C=need)
    ok.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=MB)
    short = _oracle(sp, pool, instr, sp.flags | O.F_DEDUP, C=need - 1)
    with pytest.raises(RuntimeError, match="rc=2"):
        short.run_batch(batch, prompt_stride=sp.max_prompt_tokens, max_blocks=MB)


def test_dedup_stays_within_a_rank():
    """Over G ranks a request shares only blocks an earlier request of its OWN slice computes (its
    pages are on that rank): the brute force runs per slice, the snapshot hits from the G-rank run
    without dedup."""
    sp = StreamSpec(B=96, n_logs=600, C=1 << 20)
    ds, pool, instr = make_stream(sp)
    G, MB = 2, (sp.max_prompt_tokens + 15) // 16
    plain = [_oracle(sp, pool, instr, sp.flags) for _ in range(G)]
    dd = [_oracle(sp, pool, instr, sp.flags | O.F_DEDUP) for _ in range(G)]
    for b, (start, B) in enumerate(batch_plan(sp, ds.n)):
        batch = gen.make_batch(ds, start, B)
        r0 = O.Oracle.run_batch_dp(plain, batch, prompt_stride=sp.max_prompt_tokens, max_blocks=MB)
        r1 = O.Oracle.run_batch_dp(dd, batch, prompt_stride=sp.max_prompt_tokens, max_blocks=MB)
        P = [r1.prompt(i) for i in range(B)]
        for r in range(G):
            lo, hi = r * B // G, (r + 1) * B // G
            for i in range(lo, hi):
                best = int(r0.hit[i])
                for o in range(lo, i):
                    best = max(best, _lcp_blocks(P[i], P[o]))
                assert int(r1.hit[i]) == min((len(P[i]) - 1) // BS, best), f"batch {b} request {i}"
