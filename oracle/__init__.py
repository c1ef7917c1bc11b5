"""ctypes wrapper of the CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE, NOT THE PRODUCT: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg / --impl reference arm may import this package.  It shares no code with
paper_2507_08523_b200/ (the CUDA path).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = [os.path.join(HERE, "oracle.cpp"), os.path.join(HERE, "oracle.h")]

SIM_COSINE, SIM_JACCARD = 0, 1
F_PAIR, F_GUARD, F_EXCLUDE_SELF, F_VERIFY, F_DEDUP = 1, 2, 4, 8, 16


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain g++ -O2 -fopenmp; no intrinsics)."""
    newest = max(os.path.getmtime(p) for p in SRC)
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < newest:
        tmp = LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, SRC[0]])
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        u32p, u64p, i32p, f64p = (C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                  C.POINTER(C.c_int32), C.POINTER(C.c_double))
        _lib.or_create.restype = P
        _lib.or_create.argtypes = [C.c_uint32] * 5 + [C.c_uint64]
        _lib.or_destroy.argtypes = [P]
        _lib.or_pool_load.argtypes = [P, C.c_uint32] + [u32p] * 7 + [C.c_uint32]
        _lib.or_run_batch.argtypes = ([P, C.c_uint32, u32p, u32p, u32p, u32p, u32p, i32p, u64p,
                                       u32p, u32p, C.c_uint32, u64p, C.c_uint32, u32p, u64p, u32p])
        _lib.or_run_batch_dp.argtypes = ([C.POINTER(P), C.c_uint32, C.c_uint32, u32p, u32p, u32p, u32p, u32p, i32p,
                                          u64p, u32p, u32p, C.c_uint32, u64p, C.c_uint32, u32p, u64p, u32p, u32p])
        _lib.or_set_decode.argtypes = [P, C.c_uint32]
        _lib.or_batch_index.restype = C.c_uint64
        _lib.or_batch_index.argtypes = [P]
        _lib.or_index_size.restype = C.c_uint32
        _lib.or_index_size.argtypes = [P]
        _lib.or_index_dump.argtypes = [P, u64p, u64p, u32p, u64p]
        _lib.or_table_size.restype = C.c_uint32
        _lib.or_table_size.argtypes = [P]
        _lib.or_table_dump.argtypes = [P, u32p, u64p]
        _lib.or_box_hits.argtypes = [P, u32p]
        _lib.or_box_map_size.restype = C.c_uint32
        _lib.or_box_map_size.argtypes = [P]
        _lib.or_box_map_dump.argtypes = [P, u64p, u32p]
        _lib.or_similarity.argtypes = [C.c_uint32, u32p, C.c_uint32, u32p, C.c_uint32, u64p, u64p, f64p]
        _lib.or_select.argtypes = [P, u32p, C.c_uint32, C.c_uint32, u32p]
        _lib.or_pmc.restype = C.c_uint32
        _lib.or_pmc.argtypes = [C.c_uint32, u32p, u32p]
        _lib.or_table_put.argtypes = [P, u32p, C.c_uint64]
        _lib.or_refine_one.argtypes = [P, u32p, u32p, i32p, u64p]
        _lib.or_render.argtypes = [P, u32p, u32p, C.c_uint32, u32p, u32p]
        _lib.or_mix64.restype = C.c_uint64
        _lib.or_mix64.argtypes = [C.c_uint64]
        _lib.or_chain_hash.argtypes = [C.c_uint64, u32p, C.c_uint32, u64p]
        _lib.or_lookup.restype = C.c_uint32
        _lib.or_lookup.argtypes = [P, u32p, C.c_uint32, C.c_uint32]
        _lib.or_insert.argtypes = [P, u32p, C.c_uint32]
        _lib.or_attention.argtypes = ([C.c_uint32] * 5 + [f64p, f64p, f64p, C.c_double, f64p, f64p])
    return _lib


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


@dataclass
class BatchResult:
    topk: np.ndarray          # [B][k]
    final_ds: np.ndarray      # [B][k]
    info: np.ndarray          # [B][4] pmc, rule, reverted, matched
    target_stamp: np.ndarray  # [B]
    prompt_len: np.ndarray    # [B]
    prompt_tok: np.ndarray    # [B][stride]
    block_hash: np.ndarray    # [B][max_blocks]
    hit: np.ndarray           # [B]
    evicted: np.ndarray       # [n] hashes

    def prompt(self, i: int) -> np.ndarray:
        return self.prompt_tok[i, :self.prompt_len[i]]


class Oracle:
    """One oracle context = one GPU context's worth of state (table + prefix index)."""

    def __init__(self, k: int, table_capacity: int, kv_pages: int, metric: int = SIM_COSINE,
                 flags: int = F_PAIR | F_VERIFY, hash_seed: int = 0):
        self.k, self.T, self.C, self.flags, self.seed = k, table_capacity, kv_pages, flags, hash_seed
        self.h = lib().or_create(k, table_capacity, kv_pages, metric, flags, hash_seed)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_destroy(self.h)
            self.h = None

    def set_decode(self, d: int) -> None:
        lib().or_set_decode(self.h, d)

    def pool_load(self, pool, instr) -> None:
        arrs = [_u32(pool.log_off), _u32(pool.log_tok), _u32(pool.tpl_off), _u32(pool.tpl_tok),
                _u32(pool.template_id), _u32(pool.src_index), _u32(instr)]
        rc = lib().or_pool_load(self.h, len(pool.template_id), *[_p(a, C.c_uint32) for a in arrs],
                                len(instr))
        if rc:
            raise ValueError(f"or_pool_load rc={rc}")

    def run_batch(self, batch, prompt_stride: int = 4096, max_blocks: int = 256,
                  max_evict: int = 1 << 20) -> BatchResult:
        B, k = batch.B, self.k
        topk = np.zeros((B, k), np.uint32); fin = np.zeros((B, k), np.uint32)
        info = np.zeros((B, 4), np.int32); tst = np.zeros(B, np.uint64)
        plen = np.zeros(B, np.uint32); ptok = np.zeros((B, prompt_stride), np.uint32)
        bh = np.zeros((B, max_blocks), np.uint64); hit = np.zeros(B, np.uint32)
        ev = np.zeros(max_evict, np.uint64); nev = np.array([max_evict], np.uint32)
        qo, qt, qs = _u32(batch.q_off), _u32(batch.q_tok), _u32(batch.q_src)
        rc = lib().or_run_batch(self.h, B, _p(qo, C.c_uint32), _p(qt, C.c_uint32), _p(qs, C.c_uint32),
                                _p(topk, C.c_uint32), _p(fin, C.c_uint32), _p(info, C.c_int32),
                                _p(tst, C.c_uint64), _p(plen, C.c_uint32), _p(ptok, C.c_uint32),
                                prompt_stride, _p(bh, C.c_uint64), max_blocks, _p(hit, C.c_uint32),
                                _p(ev, C.c_uint64), _p(nev, C.c_uint32))
        if rc:
            raise RuntimeError(f"or_run_batch rc={rc}")
        return BatchResult(topk, fin, info, tst, plen, ptok, bh, hit, ev[:nev[0]].copy())

    @staticmethod
    def run_batch_dp(ranks: list, batch, prompt_stride: int = 4096, max_blocks: int = 256,
                     max_evict: int = 1 << 20) -> BatchResult:
        """One global batch over len(ranks) data-parallel oracle contexts: rank r
        owns the r-th contiguous slice and its own prefix index; the replicated ICL Tables receive
        every record in global admission order."""
        G, B, k = len(ranks), batch.B, ranks[0].k
        topk = np.zeros((B, k), np.uint32); fin = np.zeros((B, k), np.uint32)
        info = np.zeros((B, 4), np.int32); tst = np.zeros(B, np.uint64)
        plen = np.zeros(B, np.uint32); ptok = np.zeros((B, prompt_stride), np.uint32)
        bh = np.zeros((B, max_blocks), np.uint64); hit = np.zeros(B, np.uint32)
        ev = np.zeros(max_evict, np.uint64); nev = np.array([max_evict], np.uint32)
        qo, qt, qs = _u32(batch.q_off), _u32(batch.q_tok), _u32(batch.q_src)
        hs = (C.c_void_p * G)(*[o.h for o in ranks])
        nrank = np.zeros(G, np.uint32)
        rc = lib().or_run_batch_dp(hs, G, B, _p(qo, C.c_uint32), _p(qt, C.c_uint32), _p(qs, C.c_uint32),
                                   _p(topk, C.c_uint32), _p(fin, C.c_uint32), _p(info, C.c_int32),
                                   _p(tst, C.c_uint64), _p(plen, C.c_uint32), _p(ptok, C.c_uint32),
                                   prompt_stride, _p(bh, C.c_uint64), max_blocks, _p(hit, C.c_uint32),
                                   _p(ev, C.c_uint64), _p(nev, C.c_uint32), _p(nrank, C.c_uint32))
        if rc:
            raise RuntimeError(f"or_run_batch_dp rc={rc}")
        res = BatchResult(topk, fin, info, tst, plen, ptok, bh, hit, ev[:nev[0]].copy())
        res.box_hit = np.zeros(B, np.uint32)
        lib().or_box_hits(ranks[0].h, _p(res.box_hit, C.c_uint32))
        off = np.concatenate([[0], np.cumsum(nrank.astype(np.int64))])
        res.evicted_rank = [res.evicted[off[r]:off[r + 1]] for r in range(G)]
        return res

    @property
    def batch_index(self) -> int:
        return int(lib().or_batch_index(self.h))

    def index_dump(self):
        n = lib().or_index_size(self.h)
        h = np.zeros(n, np.uint64); st = np.zeros(n, np.uint64)
        dp = np.zeros(n, np.uint32); par = np.zeros(n, np.uint64)
        lib().or_index_dump(self.h, _p(h, C.c_uint64), _p(st, C.c_uint64), _p(dp, C.c_uint32),
                            _p(par, C.c_uint64))
        return h, st, dp, par

    def box_map_dump(self):
        n = lib().or_box_map_size(self.h)
        h = np.zeros(n, np.uint64); m = np.zeros(n, np.uint32)
        lib().or_box_map_dump(self.h, _p(h, C.c_uint64), _p(m, C.c_uint32))
        return h, m

    def table_dump(self):
        n = lib().or_table_size(self.h)
        ds = np.zeros((n, self.k), np.uint32); st = np.zeros(n, np.uint64)
        lib().or_table_dump(self.h, _p(ds, C.c_uint32), _p(st, C.c_uint64))
        return ds, st

    # ---- pieces ----
    def select(self, q, q_src: int = 0xFFFFFFFF) -> np.ndarray:
        q = _u32(q); out = np.zeros(self.k, np.uint32)
        rc = lib().or_select(self.h, _p(q, C.c_uint32), len(q), q_src, _p(out, C.c_uint32))
        if rc:
            raise ValueError("argument error: k > candidates")
        return out

    def table_put(self, ds, stamp: int) -> None:
        ds = _u32(ds)
        lib().or_table_put(self.h, _p(ds, C.c_uint32), stamp)

    def refine_one(self, cur_ds):
        cur = _u32(cur_ds); fin = np.zeros(self.k, np.uint32); info = np.zeros(4, np.int32)
        ts = np.zeros(1, np.uint64)
        lib().or_refine_one(self.h, _p(cur, C.c_uint32), _p(fin, C.c_uint32), _p(info, C.c_int32),
                            _p(ts, C.c_uint64))
        return fin, info, int(ts[0])

    def render(self, ds, q) -> np.ndarray:
        ds, q = _u32(ds), _u32(q)
        out = np.zeros(1 << 16, np.uint32); n = np.zeros(1, np.uint32)
        lib().or_render(self.h, _p(ds, C.c_uint32), _p(q, C.c_uint32), len(q), _p(out, C.c_uint32),
                        _p(n, C.c_uint32))
        return out[:n[0]].copy()

    def lookup(self, tok, capped: bool = False) -> int:
        t = _u32(tok)
        return int(lib().or_lookup(self.h, _p(t, C.c_uint32), len(t), int(capped)))

    def insert(self, tok) -> None:
        t = _u32(tok)
        lib().or_insert(self.h, _p(t, C.c_uint32), len(t))


def similarity(metric: int, a, b):
    a, b = _u32(a), _u32(b)
    num = np.zeros(1, np.uint64); den = np.zeros(1, np.uint64); val = np.zeros(1, np.float64)
    lib().or_similarity(metric, _p(a, C.c_uint32), len(a), _p(b, C.c_uint32), len(b),
                        _p(num, C.c_uint64), _p(den, C.c_uint64), _p(val, C.c_double))
    return int(num[0]), int(den[0]), float(val[0])


def pmc(cur_tpl, entry_tpl) -> int:
    c, e = _u32(cur_tpl), _u32(entry_tpl)
    return int(lib().or_pmc(len(c), _p(c, C.c_uint32), _p(e, C.c_uint32)))


def mix64(x: int) -> int:
    return int(lib().or_mix64(x & 0xFFFFFFFFFFFFFFFF))


def chain_hash(tok, seed: int = 0) -> np.ndarray:
    t = _u32(tok); out = np.zeros(max(1, len(t) // 16), np.uint64)
    lib().or_chain_hash(seed, _p(t, C.c_uint32), len(t), _p(out, C.c_uint64))
    return out[:len(t) // 16].copy()


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, P: int, scale: float,
              want_lse: bool = False):
    """q [S][Hq][d], k/v [L][Hkv][d] (float64) -> out [S][Hq][d] (+ lse [S][Hq])."""
    q = np.ascontiguousarray(q, np.float64); k = np.ascontiguousarray(k, np.float64)
    v = np.ascontiguousarray(v, np.float64)
    S, Hq, d = q.shape
    L, Hkv, _ = k.shape
    assert S == L - P
    out = np.zeros_like(q); lse = np.zeros((S, Hq), np.float64)
    lib().or_attention(Hq, Hkv, d, L, P, _p(q, C.c_double), _p(k, C.c_double), _p(v, C.c_double),
                       scale, _p(out, C.c_double), _p(lse, C.c_double))
    return (out, lse) if want_lse else out


def attention_np(q: np.ndarray, k: np.ndarray, v: np.ndarray, P: int, scale: float,
                 want_lse: bool = False):
    """The same definition as attention() written with fp64 numpy
    matmuls as library steps, for checking every row of large batches in seconds:
        logits[h, s, j] = (q[s, h] . k[j, h // g]) * scale   for j <= P + s (causal), else -inf
        out[s, h] = sum_j softmax_j(logits[h, s, :]) v[j, h // g];  lse = log sum_j exp(logits)
    with the row max subtracted before exp.  No blocking or reordering beyond the definition;
    pinned to the same closed forms as attention() and to it (tests/test_oracle_attention.py)."""
    q = np.asarray(q, np.float64); k = np.asarray(k, np.float64); v = np.asarray(v, np.float64)
    S, Hq, d = q.shape
    L, Hkv, _ = k.shape
    assert S == L - P
    g = Hq // Hkv
    qh = q.reshape(S, Hkv, g, d).transpose(1, 2, 0, 3).reshape(Hkv, g * S, d)     # rows (hh, s)
    logits = np.matmul(qh, k.transpose(1, 2, 0)) * scale                        # [Hkv][g*S][L]
    pos = np.tile(np.arange(S), g) + P
    logits = np.where(np.arange(L)[None, None, :] <= pos[None, :, None], logits, -np.inf)
    mx = logits.max(-1, keepdims=True)
    w = np.exp(logits - mx)
    den = w.sum(-1, keepdims=True)
    o = np.matmul(w / den, v.transpose(1, 0, 2))                                # [Hkv][g*S][d]
    out = o.reshape(Hkv, g, S, d).transpose(2, 0, 1, 3).reshape(S, Hq, d)
    if not want_lse:
        return out
    lse = (mx + np.log(den))[..., 0].reshape(Hkv, g, S).transpose(2, 0, 1).reshape(S, Hq)
    return out, lse
