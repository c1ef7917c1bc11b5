"""Pins of the CPU oracle against what the paper, SPEC and mathematics fix (-m "not gpu").

Each test names the passage it pins.  None of them re-calls the oracle's own routine to
produce an expected value: expected values come from the paper's worked examples
(tests/golden/), closed forms, library routines (sklearn / torch) or brute force.
"""
import itertools
import json
import os
from collections import Counter, OrderedDict
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from tests.textfix import Interner, fragments, pool_from_demos
from workload import gen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ tokenizer fixture
def test_tokenize_fixture():
    g = load("spec_examples.json")["tokenize"]
    assert fragments(g["text"]) == g["fragments"]
    assert fragments("") == []


# ------------------------------------------------------------------ a1 similarity
def test_similarity_closed_forms():
    g = load("spec_examples.json")
    it = Interner()
    for case in g["jaccard"]:
        a = it(" ".join(case["a"])); b = it(" ".join(case["b"]))
        num, den, val = O.similarity(O.SIM_JACCARD, a, b)
        assert Fraction(num, den) == Fraction(*case["value"])
    c = g["cosine_collinear"]
    num, den, val = O.similarity(O.SIM_COSINE, it(" ".join(c["v"])), it(" ".join(c["two_v"])))
    assert num == den and val == pytest.approx(1.0)
    # both-empty conventions and one-empty (Z5)
    e = np.zeros(0, np.uint32)
    assert O.similarity(O.SIM_JACCARD, e, e)[2] == 1.0
    assert O.similarity(O.SIM_COSINE, e, e)[2] == 0.0
    assert O.similarity(O.SIM_JACCARD, e, it("a b"))[2] == 0.0
    assert O.similarity(O.SIM_COSINE, it("a"), e)[2] == 0.0


def test_similarity_vs_sklearn():
    from sklearn.metrics import jaccard_score
    from sklearn.metrics.pairwise import cosine_similarity
    rng = np.random.default_rng(0)
    for _ in range(300):
        a = rng.integers(16, 40, size=rng.integers(1, 25)).astype(np.uint32)
        b = rng.integers(16, 40, size=rng.integers(1, 25)).astype(np.uint32)
        va = np.bincount(a, minlength=40)[None]; vb = np.bincount(b, minlength=40)[None]
        cos = cosine_similarity(va, vb)[0, 0]
        jac = jaccard_score((va[0] > 0), (vb[0] > 0))
        assert O.similarity(O.SIM_COSINE, a, b)[2] == pytest.approx(cos, abs=1e-12)
        assert O.similarity(O.SIM_JACCARD, a, b)[2] == pytest.approx(jac, abs=1e-12)


# ------------------------------------------------------------------ a2 top-k
def _pool_from_token_lists(logs, tpl_ids=None):
    tpl_ids = list(range(len(logs))) if tpl_ids is None else tpl_ids
    lo = np.concatenate([[0], np.cumsum([len(x) for x in logs])]).astype(np.uint32)
    tok = np.concatenate([np.asarray(x, np.uint32) for x in logs]) if logs else np.zeros(0, np.uint32)
    tpls = [np.array([gen.PH, 16 + t], np.uint32) for t in tpl_ids]
    to = np.concatenate([[0], np.cumsum([len(x) for x in tpls])]).astype(np.uint32)
    return gen.Pool(lo, tok.astype(np.uint32), to, np.concatenate(tpls), np.array(tpl_ids, np.uint32),
                    np.arange(len(logs), dtype=np.uint32))


def test_select_identical_candidate_k1():
    it = Interner()
    logs = [it("alpha beta gamma"), it("delta eps"), it("alpha zeta")]
    o = O.Oracle(k=1, table_capacity=4, kv_pages=16)
    o.pool_load(_pool_from_token_lists(logs), gen.instruction(4, 0))
    assert list(o.select(it("delta eps"))) == [1]


def test_select_ascending_order():
    # jaccard scores of the three candidates vs q = {a,b,c,d,e,f,g,h,i,j}: 0.9, 0.5, 0.1
    it = Interner()
    q = it("a b c d e f g h i j")
    c09 = it("a b c d e f g h i")                 # 9/10
    c05 = it("a b c d e")                         # 5/10
    c01 = it("a")                                 # 1/10
    o = O.Oracle(k=2, table_capacity=4, kv_pages=16, metric=O.SIM_JACCARD)
    o.pool_load(_pool_from_token_lists([c09, c05, c01]), gen.instruction(4, 0))
    assert list(o.select(q)) == [1, 0]            # [0.5-cand, 0.9-cand]
    o3 = O.Oracle(k=4, table_capacity=4, kv_pages=16)
    with pytest.raises(ValueError):               # n > |candidates| -> argument error
        o3.pool_load(_pool_from_token_lists([c09, c05, c01]), gen.instruction(4, 0))


@pytest.mark.parametrize("metric", [O.SIM_COSINE, O.SIM_JACCARD])
def test_select_bruteforce_full_sort(metric):
    from sklearn.metrics import jaccard_score
    from sklearn.metrics.pairwise import cosine_similarity
    rng = np.random.default_rng(1 + metric)
    for trial in range(40):
        M, k = int(rng.integers(5, 40)), int(rng.integers(1, 6))
        logs = [rng.integers(16, 30, size=rng.integers(1, 8)) for _ in range(M)]
        o = O.Oracle(k=k, table_capacity=4, kv_pages=16, metric=metric)
        o.pool_load(_pool_from_token_lists(logs), gen.instruction(4, 0))
        q = rng.integers(16, 30, size=rng.integers(1, 8))
        vq = np.bincount(q, minlength=30)[None]
        sc = []
        for m in range(M):
            vm = np.bincount(logs[m], minlength=30)[None]
            sc.append(cosine_similarity(vq, vm)[0, 0] if metric == O.SIM_COSINE
                      else jaccard_score(vq[0] > 0, vm[0] > 0))
        sc = np.round(np.array(sc), 12)
        order = sorted(range(M), key=lambda m: (-sc[m], m))[:k]
        expect = sorted(order, key=lambda m: (sc[m], m))
        assert list(o.select(q)) == expect


def test_select_exclude_self():
    it = Interner()
    logs = [it("x y"), it("x y z"), it("w")]
    o = O.Oracle(k=1, table_capacity=4, kv_pages=16, flags=O.F_PAIR | O.F_VERIFY | O.F_EXCLUDE_SELF)
    o.pool_load(_pool_from_token_lists(logs), gen.instruction(4, 0))
    assert list(o.select(it("x y"), q_src=0)) == [1]   # S:174 flag: the query's own row is skipped
    assert list(o.select(it("x y"), q_src=7)) == [0]


# ------------------------------------------------------------------ a3 PMC
def _pmc_brute(cur_tpl, entry_tpl):
    """Largest p such that the multiset of entry_tpl[:p] is contained in multiset(cur_tpl)."""
    c = Counter(cur_tpl)
    best = 0
    for p in range(len(entry_tpl) + 1):
        if not (Counter(entry_tpl[:p]) - c):
            best = p
    return best


def test_pmc_fig_pair():
    g = load("fig_pair.json")
    it = Interner()
    pool = pool_from_demos(g["demos"], it)
    tid = pool.template_id
    cur = [int(tid[d]) for d in g["current"]]
    for e in g["table"]:
        assert O.pmc(cur, [int(tid[d]) for d in e["ds"]]) == g["expect"]["pmc"][e["name"]]
    assert O.pmc([4, 2, 9, 2, 7], [2, 7, 2, 9, 4]) == 5       # identical multiset -> k


def test_pmc_bruteforce_10k():
    rng = np.random.default_rng(2)
    for _ in range(10000):
        k = int(rng.integers(1, 9))
        cur = list(rng.integers(0, 5, size=k)); ent = list(rng.integers(0, 5, size=k))
        assert O.pmc(cur, ent) == _pmc_brute(cur, ent)


# ------------------------------------------------------------------ a4 refine
def _fig_pair_oracle():
    g = load("fig_pair.json")
    it = Interner()
    pool = pool_from_demos(g["demos"], it)
    o = O.Oracle(k=3, table_capacity=8, kv_pages=64)
    o.pool_load(pool, gen.instruction(8, 0))
    return g, it, pool, o


def test_match_modify_reorder_fig_pair():
    g, it, pool, o = _fig_pair_oracle()
    assert o.refine_one(g["current"])[1][3] == 0         # empty table -> absent
    for e in g["table"]:
        o.table_put(e["ds"], e["stamp"])
    fin, info, tstamp = o.refine_one(g["current"])
    assert list(fin) == g["expect"]["final"]
    assert info[0] == 2 and info[1] == g["expect"]["rule"] and info[3] == 1
    assert tstamp == 2                                     # DS2 is the target
    logs = [pool.log_tok[pool.log_off[d]:pool.log_off[d + 1]] for d in fin]
    assert [list(x) for x in logs] == [list(it(s)) for s in g["expect"]["final_logs"]]


def test_match_tie_prefers_recent():
    # two entries with equal PMC 3: the more recent wins
    it = Interner()
    demos = [{"log": f"t{j} v{i}", "template": f"t{j} <*>"} for j in range(4) for i in range(3)]
    o = O.Oracle(k=4, table_capacity=8, kv_pages=64)
    o.pool_load(pool_from_demos(demos, it), gen.instruction(8, 0))
    # demo ids: template j, variant i -> 3*j + i
    o.table_put([0, 3, 6, 9], 5)      # templates 0,1,2,3 -> PMC 3 against cur (0,1,2,2)
    o.table_put([1, 4, 7, 10], 9)
    cur = [2, 5, 8, 7]                # templates 0,1,2,2
    fin, info, ts = o.refine_one(cur)
    assert info[0] == 3 and ts == 9 and list(fin[:3]) == [1, 4, 7]


def test_modify_duplicate_templates_pair_by_occurrence():
    # a template appearing twice in both sets -> exactly two replacements, in occurrence order
    it = Interner()
    demos = [{"log": f"A v{i}", "template": "A <*>"} for i in range(4)] + \
            [{"log": f"B v{i}", "template": "B <*>"} for i in range(2)]
    o = O.Oracle(k=3, table_capacity=8, kv_pages=64)
    o.pool_load(pool_from_demos(demos, it), gen.instruction(8, 0))
    o.table_put([2, 3, 5], 1)         # A(v2), A(v3), B(v5)
    cur = [0, 4, 1]                   # A(v0), B(v4), A(v1)
    fin, info, _ = o.refine_one(cur)
    assert info[0] == 3 and info[1] == 1 and list(fin) == [2, 3, 5]   # PMC = k -> target verbatim
    o2 = O.Oracle(k=3, table_capacity=8, kv_pages=64)
    o2.pool_load(pool_from_demos(demos, it), gen.instruction(8, 0))
    o2.table_put([2, 3, 4], 1)        # A, A, then B(v4) — present in cur too: pmc 3
    o2.table_put([3, 2, 0], 2)        # A, A, A: pmc 2 (cur has only two A)
    fin, info, ts = o2.refine_one([0, 5, 1])    # A(v0), B(v5), A(v1)
    assert info[0] == 3 and ts == 1 and list(fin) == [2, 3, 4]
    o3 = O.Oracle(k=3, table_capacity=8, kv_pages=64)
    o3.pool_load(pool_from_demos(demos, it), gen.instruction(8, 0))
    o3.table_put([3, 2, 0], 2)
    fin, info, _ = o3.refine_one([0, 5, 1])
    # v3 replaces the FIRST A (position 0), v2 replaces the second A (position 2); B keeps order
    assert info[0] == 2 and info[1] == 3 and list(fin) == [3, 2, 5]


def test_reorder_identity_and_full():
    it = Interner()
    demos = [{"log": f"t{j} v{i}", "template": f"t{j} <*>"} for j in range(5) for i in range(2)]
    o = O.Oracle(k=3, table_capacity=8, kv_pages=64)
    o.pool_load(pool_from_demos(demos, it), gen.instruction(8, 0))
    o.table_put([8, 9, 8], 1)                       # template 4 only: pmc 0 vs cur below
    cur = [0, 2, 4]
    fin, info, _ = o.refine_one(cur)
    assert info[0] == 0 and info[1] == 2 and list(fin) == cur        # pmc 0 -> identity
    o.table_put([5, 3, 1], 2)                       # templates 2,1,0: pmc = k
    fin, info, _ = o.refine_one(cur)
    assert info[1] == 1 and list(fin) == [5, 3, 1]                   # pmc = N -> target order


def _matched_prefix(ds, table_ds):
    best = 0
    for e in table_ds:
        p = 0
        while p < len(ds) and ds[p] == e[p]:
            p += 1
        best = max(best, p)
    return best


def test_refine_invariants_10k():
    """SPEC acceptance 1: multiset preservation, prefix alignment,
    PMC == brute-force optimum over permutations x same-template substitutions (Z25 i), and
    the demo-unit never-worse invariant (north star)."""
    rng = np.random.default_rng(3)
    n_t, per = 4, 3
    demos = [{"log": f"t{j} v{i}", "template": f"t{j} <*>"} for j in range(n_t) for i in range(per)]
    it = Interner()
    pool = pool_from_demos(demos, it)
    tid = pool.template_id
    for trial in range(10000 // 20):
        k = int(rng.integers(1, 6))
        o = O.Oracle(k=k, table_capacity=64, kv_pages=64)
        o.pool_load(pool, gen.instruction(8, 0))
        table = []
        for s in range(int(rng.integers(0, 6))):
            e = list(rng.integers(0, n_t * per, size=k))
            if tuple(e) in {tuple(x) for x in table}:
                continue
            table.append(e); o.table_put(e, s + 1)
        for _ in range(20):
            cur = list(rng.integers(0, n_t * per, size=k))
            fin, info, _ = o.refine_one(cur)
            fin = list(fin)
            assert sorted(tid[fin]) == sorted(tid[cur])
            pm = int(info[0])
            if pm:
                tgt = [e for e in table if _pmc_brute(list(tid[cur]), list(tid[e])) == pm]
                assert any(fin[:pm] == e[:pm] for e in tgt)
            # brute-force optimum: best leading run of exact demo matches over every
            # permutation of cur with same-template substitutions
            best = 0
            for e in table:
                for perm in itertools.permutations(range(k)):
                    p = 0
                    while p < k and tid[cur[perm[p]]] == tid[e[p]]:
                        p += 1
                    best = max(best, p)
            assert pm == best
            assert _matched_prefix(fin, table) >= _matched_prefix(cur, table)


# ------------------------------------------------------------------ table management
def test_refine_table_spec_examples():
    it = Interner()
    demos = [{"log": f"t{j} v{i}", "template": f"t{j} <*>"} for j in range(6) for i in range(2)]
    pool = pool_from_demos(demos, it)
    o = O.Oracle(k=2, table_capacity=2, kv_pages=512)
    o.pool_load(pool, gen.instruction(8, 0))
    # feed queries identical to specific demos so the kNN picks them
    def run(rows):
        q = [pool.log_tok[pool.log_off[r]:pool.log_off[r + 1]] for r in rows]
        lo = np.concatenate([[0], np.cumsum([len(x) for x in q])]).astype(np.uint32)
        return o.run_batch(gen.Batch(lo, np.concatenate(q).astype(np.uint32), np.array(rows, np.uint32)))
    r = run([0])
    assert r.info[0, 0] == 0 and o.table_dump()[0].shape[0] == 1      # empty table: PMC 0, size 1
    ds0 = o.table_dump()[0][0].copy()
    r = run([0])
    assert r.info[0, 1] == 1 and o.table_dump()[0].shape[0] == 1      # same DS twice: rule 1, size 1
    r = run([4]); r = run([8])
    ds, _ = o.table_dump()
    assert ds.shape[0] == 2 and not any((row == ds0).all() for row in ds)   # head evicted


def test_batch1_equals_paper_ordereddict():
    """Z1-Z3 reduce to the paper's literal procedure when B = 1: an OrderedDict ICL Table
    (P:354), rule 1 moves the target to the tail, rules 2/3 append, the head is evicted at
    capacity.  Checked over a stream against a plain OrderedDict model."""
    cfg = gen.config(1)
    ds_ = gen.make_dataset("HDFS", 400, 14, 1.3, 1004)
    pool = gen.sample_pool(ds_, 60, 2004)
    T = 24
    o = O.Oracle(k=3, table_capacity=T, kv_pages=4096)
    o.pool_load(pool, gen.instruction(32, 0))
    tid = pool.template_id
    table = OrderedDict()
    for r in range(300):
        b = gen.make_batch(ds_, r, 1)
        res = o.run_batch(b)
        cur = [int(x) for x in res.topk[0]]
        # paper procedure
        best, best_p = None, 0
        for key in table:                                   # head -> tail
            p = _pmc_brute([tid[c] for c in cur], [tid[d] for d in key])
            if p > best_p or (p == best_p and p > 0):       # later = more recent
                best, best_p = key, p
        if best is None:
            final = tuple(cur); table[final] = None
        elif best_p == 3:
            final = best; table.move_to_end(best)
        else:
            rep = [False] * 3; head = []
            for j in range(best_p):
                q = next(qq for qq in range(3) if not rep[qq] and tid[cur[qq]] == tid[best[j]])
                rep[q] = True; head.append(best[j])
            final = tuple(head + [cur[q] for q in range(3) if not rep[q]])
            table[final] = None
        while len(table) > T:
            table.popitem(last=False)
        assert tuple(int(x) for x in res.final_ds[0]) == final
        assert res.info[0, 0] == best_p
        ds, _ = o.table_dump()
        assert [tuple(int(x) for x in row) for row in ds] == list(table.keys())


# ------------------------------------------------------------------ render
def test_render_layout_and_prefix_monotonicity():
    g, it, pool, o = _fig_pair_oracle()
    q = it("ARPT: 555")
    p1 = o.render([0, 1, 2], q)
    instr = gen.instruction(8, 0)
    lens = [pool.log_off[d + 1] - pool.log_off[d] + pool.tpl_off[d + 1] - pool.tpl_off[d] + 1 for d in [0, 1, 2]]
    # len(instr) + sum len(demo_i) + k*len(sep) + len(query), len(demo) = |log| + 1 + |tpl|
    assert len(p1) == len(instr) + sum(lens) + 3 * 1 + len(q)
    assert (p1[:len(instr)] == instr).all()
    p2 = o.render([0, 3, 2], q)                                        # differ at DS[1]
    first = len(instr) + lens[0] + 1
    assert (p1[:first] == p2[:first]).all() and p1[first] != p2[first]
    assert p1[first - 1] == gen.SEP


# ------------------------------------------------------------------ chain hash
def test_chain_hash_order_dependence_and_prefix():
    rng = np.random.default_rng(4)
    tok = rng.integers(16, 5000, size=16 * 6).astype(np.uint32)
    h = O.chain_hash(tok)
    assert len(h) == 6 and len(set(h.tolist())) == 6
    assert (O.chain_hash(tok) == h).all()                              # determinism
    assert (O.chain_hash(tok[:16 * 3 + 5])[:3] == h[:3]).all()         # a block's hash depends on its prefix only
    sw = tok.copy(); sw[16:32], sw[48:64] = tok[48:64], tok[16:32]     # swap blocks 1 and 3
    h2 = O.chain_hash(sw)
    assert h2[0] == h[0] and all(h2[j] != h[j] for j in range(1, 6))
    assert (O.chain_hash(tok, seed=1) != h).all()
    assert 0 not in h and 0xFFFFFFFFFFFFFFFF not in h                  # Z18 sentinels


# ------------------------------------------------------------------ lookup / insert
def _blocks(names, size=16):
    ids = {n: i for i, n in enumerate(sorted({x for x in names}))}
    return np.concatenate([np.full(size, 100 + ids[n], np.uint32) + np.arange(size, dtype=np.uint32) * 0
                           for n in names])


def test_fig_prefixcache():
    g = load("fig_prefixcache.json")
    allnames = sorted({b for r in g["requests"] for b in r["blocks"]})
    tokof = {n: (np.arange(16, dtype=np.uint32) + 1000 * (i + 1)) for i, n in enumerate(allnames)}
    o = O.Oracle(k=1, table_capacity=4, kv_pages=1024)
    o.pool_load(_pool_from_token_lists([[20]]), gen.instruction(4, 0))
    for r in g["requests"]:
        seq = np.concatenate([tokof[b] for b in r["blocks"]])
        assert o.lookup(seq) == r["expect_hit"], r["name"]
        o.insert(seq)


def test_lookup_bruteforce_500_traces():
    """S:317 oracle equivalence: unbounded capacity, <= 200 tokens/prompt, <= 50 prompts."""
    rng = np.random.default_rng(5)
    for trace in range(500):
        o = O.Oracle(k=1, table_capacity=4, kv_pages=1 << 20)
        o.pool_load(_pool_from_token_lists([[20]]), gen.instruction(4, 0))
        seen = []
        for _ in range(int(rng.integers(1, 12))):
            if seen and rng.random() < 0.6:
                base = seen[int(rng.integers(len(seen)))]
                cut = int(rng.integers(0, len(base) + 1))
                seq = np.concatenate([base[:cut], rng.integers(16, 20, size=rng.integers(0, 60))])
            else:
                seq = rng.integers(16, 20, size=rng.integers(0, 200))
            seq = seq[:200].astype(np.uint32)
            best = 0
            for s in seen:
                m = 0
                while (m + 1) * 16 <= min(len(s), len(seq)) and (s[m * 16:(m + 1) * 16] == seq[m * 16:(m + 1) * 16]).all():
                    m += 1
                best = max(best, m)
            h = o.lookup(seq)
            assert h == best and h <= len(seq) // 16
            o.insert(seq)
            seen.append(seq)


def test_insert_spec_examples():
    o = O.Oracle(k=1, table_capacity=4, kv_pages=2)
    o.pool_load(_pool_from_token_lists([[20]]), gen.instruction(4, 0))
    s32 = np.arange(100, 132, dtype=np.uint32)
    o.insert(s32)
    assert len(o.index_dump()[0]) == 2                                 # 32 tokens -> 2 blocks
    before = o.index_dump()[0].copy()
    o.insert(s32)
    assert (o.index_dump()[0] == before).all()                         # double insert: unchanged
    o2 = O.Oracle(k=1, table_capacity=4, kv_pages=2)
    o2.pool_load(_pool_from_token_lists([[20]]), gen.instruction(4, 0))
    seqs = [np.arange(16, dtype=np.uint32) + 200 * (i + 1) for i in range(3)]
    for s in seqs:
        o2.insert(s)
    assert o2.lookup(seqs[0]) == 0 and o2.lookup(seqs[1]) == 1 and o2.lookup(seqs[2]) == 1


def test_hit_rate_trace():
    g = load("spec_examples.json")["hit_rate_trace"]
    o = O.Oracle(k=1, table_capacity=4, kv_pages=1024)
    o.pool_load(_pool_from_token_lists([[20]]), gen.instruction(4, 0))
    base = np.arange(64, dtype=np.uint32) + 500
    o.insert(base)
    h1 = o.lookup(np.concatenate([base[:32], np.arange(32, dtype=np.uint32) + 9000]))
    h2 = o.lookup(base)
    h3 = o.lookup(np.arange(64, dtype=np.uint32) + 7000)
    assert [h1, h2, h3] == g["hits"]
    assert sum(g["hits"]) / sum(g["full"]) == g["rate"]


# ------------------------------------------------------------------ batch semantics
def _run_stream(cfgn, flags, n_batches=None, B=None, logs=None, T=None, C=None):
    cfg = gen.config(cfgn)
    name, n, nt, s, seed = cfg.datasets[0]
    ds_ = gen.make_dataset(name, logs or n, nt, s, seed)
    pool = gen.sample_pool(ds_, cfg.M, cfg.pool_seed)
    o = O.Oracle(k=cfg.k, table_capacity=T or cfg.T, kv_pages=C or cfg.C, flags=flags)
    o.pool_load(pool, gen.instruction(cfg.n_instr, cfg.instr_seed))
    B = B or cfg.B
    nb = n_batches or (ds_.n + B - 1) // B
    hits = full = 0
    res = []
    for b in range(nb):
        r = o.run_batch(gen.make_batch(ds_, b * B, min(B, ds_.n - b * B) if n_batches is None else B),
                        prompt_stride=cfg.max_prompt_tokens, max_blocks=cfg.max_prompt_tokens // 16)
        hits += int(r.hit.sum()); full += int((r.prompt_len // 16).sum())
        res.append(r)
    return o, res, hits / full


def test_hit_rate_uplift_pair_vs_naive():
    """SPEC acceptance 4 / paper P:706 (1.23x average, 2.1x HDFS): PAIR beats naive
    prefix caching on the hotspot-skewed stream by >= 1.10x (directional pin)."""
    _, _, pair = _run_stream(1, O.F_PAIR | O.F_VERIFY)
    _, _, naive = _run_stream(1, O.F_VERIFY)
    assert 0.0 <= naive <= 1.0 and 0.0 <= pair <= 1.0
    assert pair / naive >= 1.10, (pair, naive)


def test_batch_invariants_and_resident_set():
    """Hit blocks are never evicted in their batch, the resident set stays
    ancestor-closed (Z21), |resident| <= C, |table| <= T, hits <= F - or the Z20 cap."""
    o, res, _ = _run_stream(1, O.F_PAIR | O.F_VERIFY | O.F_GUARD, C=160, T=32, B=8, n_batches=120)
    h, st, dp, par = o.index_dump()
    assert len(h) <= 160
    hs = set(h.tolist())
    root_children = 0
    for x, p_, d in zip(h, par, dp):
        if d == 0:
            root_children += 1
        else:
            assert int(p_) in hs                      # ancestor-closed
    assert o.table_dump()[0].shape[0] <= 32
    for r in res:
        assert (r.hit <= np.maximum(r.prompt_len.astype(np.int64) - 1, 0) // 16).all()
        hit_hashes = {int(r.block_hash[i, j]) for i in range(len(r.hit)) for j in range(r.hit[i])}
        assert not hit_hashes & set(int(x) for x in r.evicted)     # S:319 LRU safety
    assert sum(len(r.evicted) for r in res) > 0                    # eviction was exercised
    # guard on: block form of never-worse holds per request against its snapshot:
    # re-run with guard and check hit(final) >= hit(cur) is implied by construction (Z25);
    # here we check the reverted flag is only set when a change happened.
    for r in res:
        rev = r.info[:, 2] == 1
        assert (r.final_ds[rev] == r.topk[rev]).all()


# ------------------------------------------------------------------ mix64 (Z17) vs published splitmix64
def test_mix64_published_splitmix64_outputs():
    """Z17 builds the chain hash from the splitmix64 finaliser.  splitmix64 (state += 0x9E3779B97F4A7C15,
    output = finaliser(state)) has published reference outputs: state 0 -> 0xE220A8397B1DCDAF first,
    and seed 1234567 -> 6457827717110365317, 3203168211198807973, 9817491932198370423,
    4593380528125082431, 16408922859458223821 (the generator's standard test vector).  A transposed
    shift or multiplier constant in the oracle's mix64 fails this."""
    g, M = 0x9E3779B97F4A7C15, (1 << 64) - 1
    assert O.mix64(g) == 0xE220A8397B1DCDAF
    st, out = 1234567, []
    for _ in range(5):
        st = (st + g) & M
        out.append(O.mix64(st))
    assert out == [6457827717110365317, 3203168211198807973, 9817491932198370423,
                   4593380528125082431, 16408922859458223821]
    assert O.mix64(0) == 0                                             # the finaliser fixes 0


# ------------------------------------------------------------------ batch procedure at B = 1 (Z1, Z21)
def _hdfs_stream(n_logs=600, M=60, k=3, n_instr=40):
    ds_ = gen.make_dataset("HDFS", n_logs, 14, 1.3, 1004)
    pool = gen.sample_pool(ds_, M, 2004)
    return ds_, pool, gen.instruction(n_instr, 0)


def test_batch1_run_batch_equals_sequential_lookup_insert():
    """c.4 "B = 1 == sequential SPEC refine + insert", prefix-cache half: with an
    unbounded cache, run_batch at B = 1 gives, request by request, the hit count SPEC's sequential
    kv_sim gives (lookup of the prompt, capped per Z20, then insert of the prompt), and both leave
    the same set of resident blocks."""
    ds_, pool, instr = _hdfs_stream()
    a = O.Oracle(k=3, table_capacity=24, kv_pages=1 << 20, flags=O.F_PAIR | O.F_VERIFY)
    seq = O.Oracle(k=3, table_capacity=24, kv_pages=1 << 20, flags=O.F_PAIR | O.F_VERIFY)
    a.pool_load(pool, instr); seq.pool_load(pool, instr)
    for r in range(250):
        res = a.run_batch(gen.make_batch(ds_, r, 1))
        p = res.prompt(0)
        assert seq.lookup(p, capped=True) == int(res.hit[0]), r
        seq.insert(p)
        assert (np.sort(a.index_dump()[0]) == np.sort(seq.index_dump()[0])).all(), r


class _Z21Model:
    """Literal reading Z21 + Z1 + Z22 over a plain dict:
    hash -> [stamp, depth, parent, tokens].  Stamps are (batch << 32 | admission index)."""

    def __init__(self, C, root, decode=0):
        self.C, self.root, self.res, self.b, self.decode = C, root, {}, 0, decode

    def hits(self, prompt, H):
        prev, h = self.root, 0
        for j, x in enumerate(H):
            e = self.res.get(x)
            if e is None or e[2] != prev or tuple(prompt[16 * j:16 * j + 16]) != e[3]:
                break
            h, prev = h + 1, x
        return min(h, max(len(prompt) - 1, 0) // 16)

    def batch(self, prompts, Hs):
        self.b += 1
        h = [self.hits(p, H) for p, H in zip(prompts, Hs)]            # snapshot (Z1)
        pinned = {Hs[i][j] for i in range(len(prompts)) for j in range(h[i])}
        for i in range(len(prompts)):                                   # touch in admission order
            for j in range(h[i]):
                self.res[Hs[i][j]][0] = (self.b << 32) | i
        need = sum((len(p) + self.decode + 15) // 16 - h[i] for i, p in enumerate(prompts))   # (+ decode reserve)
        free = self.C - len(self.res)
        victims = []
        if need > free:                                                 # LRU: (stamp, -depth, hash)
            order = sorted((e[0], -e[1], x) for x, e in self.res.items() if x not in pinned)
            victims = [x for _, _, x in order[:need - free]]
            for x in victims:
                del self.res[x]
        for i, p in enumerate(prompts):                                 # insert, first wins (Z22)
            for j in range(h[i], len(Hs[i])):
                x = Hs[i][j]
                if x in self.res:
                    self.res[x][0] = max(self.res[x][0], (self.b << 32) | i)
                else:
                    par = self.root if j == 0 else Hs[i][j - 1]
                    self.res[x] = [(self.b << 32) | i, j, par, tuple(p[16 * j:16 * j + 16])]
        return h, victims


@pytest.mark.parametrize("B,D", [(1, 0), (3, 0), (3, 7)])
def test_small_cache_stream_matches_literal_z21_lru(B, D):
    """Z21 with a small cache (C = 48 pages, every batch evicts): the oracle's hits, exact victim
    lists (in eviction order) and resident blocks with their stamps, depths and parents equal a
    literal LRU model keyed by (stamp, -depth, hash)."""
    ds_, pool, instr = _hdfs_stream(n_instr=24)
    C = 48
    o = O.Oracle(k=3, table_capacity=16, kv_pages=C, flags=O.F_PAIR | O.F_VERIFY)
    o.set_decode(D)                                                     # NEXT-4 decode reserve
    o.pool_load(pool, instr)
    probe = O.Oracle(k=1, table_capacity=4, kv_pages=4)              # ROOT = parent of a depth-0 block
    probe.pool_load(_pool_from_token_lists([[20]]), gen.instruction(4, 0))
    probe.insert(np.arange(16, dtype=np.uint32) + 100)
    m = _Z21Model(C, int(probe.index_dump()[3][0]), decode=D)
    n_evicting = 0
    for b in range(120):
        res = o.run_batch(gen.make_batch(ds_, b * B, B))
        prompts = [tuple(int(t) for t in res.prompt(i)) for i in range(B)]
        Hs = [[int(x) for x in res.block_hash[i, :len(prompts[i]) // 16]] for i in range(B)]
        h, victims = m.batch(prompts, Hs)
        assert [int(x) for x in res.hit] == h, b
        assert [int(x) for x in res.evicted] == victims, b
        n_evicting += bool(victims)
        hh, st, dp, par = o.index_dump()
        want = sorted(m.res.items())
        assert [int(x) for x in hh] == [x for x, _ in want], b
        assert [int(x) for x in st] == [e[0] for _, e in want], b
        assert [int(x) for x in dp] == [e[1] for _, e in want], b
        assert [int(x) for x in par] == [e[2] for _, e in want], b
    assert n_evicting >= 40
