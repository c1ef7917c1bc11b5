"""il_prefill_attn called directly (include/il.h) with hand-built block tables and full-mantissa
inputs, every output row checked against the fp64 oracle (Z26-Z27).

The stream tests (test_parity_attn.py) drive the kernel with the Z28 generator's 256-level grid;
here Q, K_new, V_new and the cached pages are N(0, 1) bf16 (all mantissa bits used), some rows
are scaled to large magnitudes (|q| ~ 30: near-one-hot softmax; |v| ~ 1e3), and the block tables
are built by hand: distinct random pages, or a leading run of pages shared by every request (the
batch-shared prefix the cascade splits off).  Cases: S = 1, P = 0, P not a multiple of 128,
S spanning several M-tiles, B = 1, GQA group g = 1..8, head dim 64 and 128."""
import numpy as np
import pytest
import torch

import oracle as O
from tests.parity_util import StreamSpec, make_stream
from workload import gen

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _bf16(x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16)


def run_case(Hq, Hkv, d, reqs, shared_blocks=0, seed=0, big_rows=True, C=2048):
    """reqs: list of (P, S) with P a multiple of 16.  Returns the worst row error."""
    from paper_2507_08523_b200 import Config, Pipeline
    rng = np.random.default_rng(seed)
    B = len(reqs)
    maxL = max(P + S for P, S in reqs)
    mpt = max(256, (maxL + 15) // 16 * 16)        # >= the pool instruction (128 tokens)
    tot_S = sum(S for _, S in reqs)
    sp = StreamSpec(n_logs=300, M=40, B=4)
    _, pool, instr = make_stream(sp)
    cfg = Config(k=3, table_capacity=16, kv_pages=C, max_batch=max(B, 4), max_prompt_tokens=mpt, max_pool=sp.M,
                 max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16, max_log_tokens=255,
                 max_suffix_tokens=tot_S, n_q_heads=Hq, n_kv_heads=Hkv, head_dim=d)
    pl = Pipeline(cfg, "cuda")
    pl.load_pool(pool, instr)
    pl.match(0)                                   # il_prefill_attn requires a preceding il_prefix_match
    MB = cfg.max_blocks
    # block tables: a shared leading run (same physical pages for every request), then distinct pages
    free = list(rng.permutation(C))
    shared = [free.pop() for _ in range(shared_blocks)]
    bt = np.full((max(B, 4), MB), -1, np.int32)
    for i, (P, S) in enumerate(reqs):
        nb = (P + S + 15) // 16
        sh = min(shared_blocks, P // 16)
        bt[i, :sh] = shared[:sh]
        for j in range(sh, nb):
            bt[i, j] = free.pop()
    # page contents: N(0,1) bf16 everywhere (prefix K/V are whatever the pages hold)
    kp = rng.normal(size=(C, Hkv, 16, d)); vp = rng.normal(size=(C, Hkv, 16, d))
    pl.k_pages.copy_(_bf16(kp)); pl.v_pages.copy_(_bf16(vp))
    kp = pl.k_pages.float().cpu().numpy().astype(np.float64); vp = pl.v_pages.float().cpu().numpy().astype(np.float64)
    q = rng.normal(size=(tot_S, Hq, d)); kn = rng.normal(size=(tot_S, Hkv, d)); vn = rng.normal(size=(tot_S, Hkv, d))
    if big_rows and tot_S > 2:
        q[rng.choice(tot_S, size=max(1, tot_S // 5), replace=False)] *= 30.0    # near one-hot softmax rows
        vn[rng.choice(tot_S, size=max(1, tot_S // 7), replace=False)] *= 1e3    # large-magnitude values
    qt, knt, vnt = _bf16(q), _bf16(kn), _bf16(vn)
    q = qt.float().numpy().astype(np.float64); kn = knt.float().numpy().astype(np.float64)
    vn = vnt.float().numpy().astype(np.float64)
    cu = np.concatenate([[0], np.cumsum([S for _, S in reqs])]).astype(np.int32)
    dev = pl.device
    cu_t = torch.from_numpy(cu).to(dev)
    pre_t = torch.tensor([P for P, _ in reqs], dtype=torch.int32, device=dev)
    bt_t = torch.from_numpy(bt).to(dev)
    out = torch.empty(tot_S, Hq, d, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(tot_S, Hq, dtype=torch.float32, device=dev)
    pl.ctx.prefill_attn(B, cu_t, pre_t, bt_t, qt.to(dev), knt.to(dev), vnt.to(dev), pl.k_pages, pl.v_pages,
                        out, lse, d ** -0.5)
    pl.ctx.status_sync()
    got = out.float().cpu().numpy().astype(np.float64)
    glse = lse.cpu().numpy().astype(np.float64)
    worst = 0.0
    for i, (P, S) in enumerate(reqs):
        pages = bt[i, :P // 16]
        kpre = kp[pages].transpose(0, 2, 1, 3).reshape(P, Hkv, d)          # [page][h][slot][d] -> [pos][h][d]
        vpre = vp[pages].transpose(0, 2, 1, 3).reshape(P, Hkv, d)
        K = np.concatenate([kpre, kn[cu[i]:cu[i + 1]]]); V = np.concatenate([vpre, vn[cu[i]:cu[i + 1]]])
        ref, rl = O.attention_np(q[cu[i]:cu[i + 1]], K, V, P=P, scale=d ** -0.5, want_lse=True)
        g_ = got[cu[i]:cu[i + 1]]
        err = np.abs(g_ - ref).max(-1) / np.maximum(np.abs(ref).max(-1), 1e-6)    # every (row, head)
        assert err.max() <= TOL, (i, P, S, float(err.max()), np.unravel_index(err.argmax(), err.shape))
        assert np.abs(glse[cu[i]:cu[i + 1]] - rl).max() <= 1e-3 * max(1.0, np.abs(rl).max()), (i, P, S)
        worst = max(worst, float(err.max()))
        # the suffix K/V rows were appended into the request's pages (K7a)
        kpg = pl.k_pages[torch.from_numpy(bt[i, P // 16:(P + S + 15) // 16].astype(np.int64)).to(dev)]
        kpg = kpg.float().cpu().numpy().transpose(0, 2, 1, 3).reshape(-1, Hkv, d)[:S]
        assert np.array_equal(kpg, kn[cu[i]:cu[i + 1]].astype(np.float32)), (i, "appended K rows")
    return worst


MIX = [(0, 1), (16, 1), (1840, 40), (0, 300), (2000, 129), (128, 17), (496, 250)]


@pytest.mark.parametrize("Hq,Hkv,d", [(32, 8, 128), (8, 8, 64), (8, 8, 128), (64, 8, 128), (40, 8, 128),
                                      (24, 8, 128), (56, 8, 128), (16, 8, 64), (4, 4, 64)])
def test_direct_mixed_requests(Hq, Hkv, d):
    run_case(Hq, Hkv, d, MIX, seed=Hq + d)


@pytest.mark.parametrize("Hq,Hkv,d", [(32, 8, 128), (16, 4, 64)])
def test_direct_shared_prefix_cascade(Hq, Hkv, d):
    # every request's first 100 blocks are the same physical pages (the cascade's dense phase)
    reqs = [(1600, 33), (1840, 1), (2048, 200), (1600, 64), (1760, 130)]
    run_case(Hq, Hkv, d, reqs, shared_blocks=100, seed=5)


@pytest.mark.parametrize("P,S", [(0, 1), (0, 129), (2032, 1), (1024, 512), (16, 2047)])
def test_direct_single_request(P, S):
    run_case(32, 8, 128, [(P, S)], seed=P + S)


def test_direct_many_short_requests():
    # 200 requests of S in 1..40 over P up to 1,200: the dense M-tiles straddle request boundaries
    rng = np.random.default_rng(11)
    reqs = [(16 * int(rng.integers(0, 76)), int(rng.integers(1, 41))) for _ in range(200)]
    run_case(32, 8, 128, reqs, seed=3, C=8192)


@pytest.mark.parametrize("p2", ["1", "0", "dense_p2", "dense2"])
@pytest.mark.parametrize("Hq,Hkv,d", [(32, 8, 128), (16, 4, 64)])
def test_direct_phase_orders(p2, Hq, Hkv, d, monkeypatch):
    # both cascade orders (read by il_prefill_attn at each call): the default -- the dense pass over
    # the shared prefix first (k_attn_sm100 phase 3), k_attn_p2 merging its partial in the
    # epilogue -- and IL_P2=0, each request's own part first on k_attn_sm100 (phase 2) continued by
    # the dense pass (phase 1); a shared prefix, short and multi-tile suffixes, one request without
    # a shared block beyond the prefix
    # ("dense_p2": the A / B variant IL_DENSE_P2=1, the dense pass on k_attn_p2 as well)
    if p2 == "dense_p2":
        monkeypatch.setenv("IL_DENSE_P2", "1")
    elif p2 == "dense2":                               # the CTA-pair dense pass (head dim 128; 64 falls back)
        monkeypatch.setenv("IL_DENSE2", "1")
    else:
        monkeypatch.setenv("IL_P2", p2)
    reqs = [(1600, 33), (1840, 1), (2048, 200), (1600, 64), (1760, 130), (1600, 1), (1616, 97)]
    run_case(Hq, Hkv, d, reqs, shared_blocks=100, seed=17)      # (the same inputs for every variant)
