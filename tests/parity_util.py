"""Helpers for GPU-vs-oracle parity tests: run one synthetic stream through both sides."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

import oracle as O
from workload import gen


@dataclass
class StreamSpec:
    n_logs: int = 2000
    n_templates: int = 14
    zipf: float = 1.3
    seed: int = 1004
    M: int = 200
    pool_seed: int = 2004
    k: int = 3
    B: int = 100
    n_instr: int = 128
    T: int = 512
    C: int = 4096
    max_prompt_tokens: int = 512
    Hq: int = 4
    Hkv: int = 4
    d: int = 64
    metric: int = O.SIM_COSINE
    flags: int = O.F_PAIR | O.F_VERIFY
    hash_seed: int = 0
    n_batches: int | None = None
    ramp: tuple = ()           # sizes of the first batches (cold-start warm-up), then B


def batch_plan(sp: StreamSpec, n_logs: int):
    """(start, size) of each batch: the ramp, then full batches of B over the stream."""
    plan, start = [], 0
    for r in sp.ramp:
        plan.append((start, r)); start += r
    nb = sp.n_batches if sp.n_batches is not None else (n_logs - start + sp.B - 1) // sp.B + len(plan)
    while len(plan) < nb:
        plan.append((start, sp.B)); start += sp.B
    return plan


def make_stream(sp: StreamSpec):
    ds = gen.make_dataset("S", sp.n_logs, sp.n_templates, sp.zipf, sp.seed)
    pool = gen.sample_pool(ds, sp.M, sp.pool_seed)
    instr = gen.instruction(sp.n_instr, 77)
    return ds, pool, instr


def gpu_config(sp: StreamSpec, pool, max_suffix_tokens: int = 0):
    from paper_2507_08523_b200 import Config
    return Config(k=sp.k, table_capacity=sp.T, kv_pages=sp.C, max_batch=sp.B,
                  max_prompt_tokens=sp.max_prompt_tokens, max_pool=sp.M,
                  max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16,
                  max_log_tokens=255, max_suffix_tokens=max_suffix_tokens,
                  n_q_heads=sp.Hq, n_kv_heads=sp.Hkv, head_dim=sp.d,
                  metric=sp.metric, flags=sp.flags, hash_seed=sp.hash_seed)


def gpu_pipeline(sp: StreamSpec, pool, instr, max_suffix_tokens: int = 0):
    from paper_2507_08523_b200 import Pipeline
    cfg = gpu_config(sp, pool, max_suffix_tokens)
    pl = Pipeline(cfg, "cuda")
    pl.load_pool(pool, instr)
    return pl


def oracle_for(sp: StreamSpec, pool, instr):
    o = O.Oracle(sp.k, sp.T, sp.C, metric=sp.metric, flags=sp.flags, hash_seed=sp.hash_seed)
    o.pool_load(pool, instr)
    return o


def compare_batch(r, pl, B, sp: StreamSpec, where=""):
    """Bit-exact comparison of one batch's integer outputs."""
    k, MB = sp.k, (sp.max_prompt_tokens + 15) // 16
    topk = pl.u32(pl.topk[:B])
    fin = pl.u32(pl.final_ds[:B])
    info = pl.info_np(B)
    np.testing.assert_array_equal(topk, r.topk, err_msg=f"{where} topk")
    np.testing.assert_array_equal(fin, r.final_ds, err_msg=f"{where} final_ds")
    np.testing.assert_array_equal(info["pmc"], r.info[:, 0], err_msg=f"{where} pmc")
    np.testing.assert_array_equal(info["rule"], r.info[:, 1], err_msg=f"{where} rule")
    np.testing.assert_array_equal(info["reverted"], r.info[:, 2], err_msg=f"{where} reverted")
    np.testing.assert_array_equal(info["matched"], r.info[:, 3], err_msg=f"{where} matched")
    np.testing.assert_array_equal(info["target_stamp"], r.target_stamp, err_msg=f"{where} target stamp")
    plen = pl.u32(pl.prompt_len[:B])
    np.testing.assert_array_equal(plen, r.prompt_len, err_msg=f"{where} prompt_len")
    ptok = pl.u32(pl.prompt_tok[:B])
    for i in range(B):
        L = plen[i]
        if not np.array_equal(ptok[i, :L], r.prompt_tok[i, :L]):
            raise AssertionError(f"{where} prompt tokens of request {i}")
    bh = pl.block_hash[:B].cpu().numpy().view(np.uint64)
    for i in range(B):
        F = plen[i] // 16
        if not np.array_equal(bh[i, :F], r.block_hash[i, :F]):
            raise AssertionError(f"{where} block hashes of request {i}")
    np.testing.assert_array_equal(pl.u32(pl.hit[:B]), r.hit, err_msg=f"{where} hit")
    ev = pl.ctx.evicted_dump()
    np.testing.assert_array_equal(ev, np.sort(r.evicted), err_msg=f"{where} evicted set")
    # derived outputs: prefix_len, cu_q
    np.testing.assert_array_equal(pl.prefix_len[:B].cpu().numpy(), 16 * r.hit.astype(np.int64))
    suf = r.prompt_len.astype(np.int64) - 16 * r.hit.astype(np.int64)
    np.testing.assert_array_equal(pl.cu_q[:B + 1].cpu().numpy(), np.concatenate([[0], np.cumsum(suf)]))


def compare_state(o, pl, where=""):
    oh, ost, odp, opar = o.index_dump()
    gh, gst, gdp, gpar = pl.ctx.index_dump()
    np.testing.assert_array_equal(gh, oh, err_msg=f"{where} index hashes")
    np.testing.assert_array_equal(gst, ost, err_msg=f"{where} index stamps")
    np.testing.assert_array_equal(gdp, odp, err_msg=f"{where} index depths")
    np.testing.assert_array_equal(gpar, opar, err_msg=f"{where} index parents")
    ods, ots = o.table_dump()
    gds, gts = pl.ctx.table_dump()
    np.testing.assert_array_equal(gts, ots, err_msg=f"{where} table stamps")
    np.testing.assert_array_equal(gds, ods, err_msg=f"{where} table entries")
