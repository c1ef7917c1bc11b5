"""Seeded synthetic Loghub-shaped workloads in the token-id domain.

This module is the ONLY code shared by the CUDA path's callers (tests, bench) and the
oracle's callers. It holds input generation only: no similarity, no top-k, no PAIR,
no hashing, no attention. Nothing here is the method's arithmetic.

Recipe:
  * templates: length U[4,20]; each position constant w.p. 0.75 else a ``<*>`` slot (>=1
    slot); constants drawn Zipf(1.0) over a 2,000-id dataset vocabulary, so templates
    share words and similarity is non-trivial.  Template tokens = constants + PH.
  * popularity: Zipf(s) over templates (template 0 hottest) — the hotspot structure of
    PAPER.md P:256-257 (fig:hotspot).
  * logs: each slot of each template owns a value pool of U[1,1000] values; a value is a
    run of U[1, w] tokens (w ~ U[1,8] per slot) drawn from a per-slot alphabet of U[4,40]
    fresh ids — numbers, IPs and block ids are several BPE tokens long and share digit
    chunks — so logs of one template differ in length and in partial overlap.  A
    log is its template with each slot replaced by a value drawn uniformly from the slot's
    pool (exact repeats happen).
  * pool: seeded uniform sample of M logs without replacement ("samples 200 logs
    from each log dataset"), kept in dataset-row order.
  * queries: every log in dataset order, cycled; batch b = next B queries
    (closed-loop concurrency B).
  * instruction: I fixed tokens from a separate id range ("Common Instruction").
  * Q/K/V: a counter-based generator of (seed, token, absolute position, head, dim),
    SURVEY §8(c) Z28, so a cached page equals recomputation (cache transparency).

Token ids: 0 PAD, 1 SEP, 2 TPL, 3 PH (the ``<*>`` placeholder), 4..15 spare; real >= 16.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

PAD, SEP, TPL, PH = 0, 1, 2, 3
VOCAB_BASE = 16          # dataset vocabulary ids live in [16, 16 + vocab)
INSTR_BASE = 1 << 20     # instruction ids
VALUE_BASE = 1 << 22     # slot-value ids (numbers, IPs, block ids ...)

# The 16 Loghub-2k systems named in PAPER.md P:599-614, with approximate public template
# counts (NOT given in PAPER.md: tunable knobs).
LOGHUB16 = [
    ("Android", 166), ("Apache", 6), ("BGL", 120), ("Hadoop", 114), ("HDFS", 14),
    ("HealthApp", 75), ("HPC", 46), ("Linux", 118), ("Mac", 341), ("OpenSSH", 27),
    ("OpenStack", 43), ("Proxifier", 8), ("Spark", 36), ("Thunderbird", 149),
    ("Windows", 50), ("Zookeeper", 50),
]


@dataclass
class Dataset:
    name: str
    templates: list            # list[np.ndarray uint32] template tokens (PH at slots)
    log_off: np.ndarray        # [n+1] uint32 CSR offsets
    log_tok: np.ndarray        # [sum] uint32
    log_tpl: np.ndarray        # [n] uint32 template id of each log

    @property
    def n(self) -> int:
        return len(self.log_tpl)

    def log(self, r: int) -> np.ndarray:
        return self.log_tok[self.log_off[r]:self.log_off[r + 1]]


@dataclass
class Pool:
    """The candidate set: per-demo log tokens, template tokens, template id, row."""
    log_off: np.ndarray
    log_tok: np.ndarray
    tpl_off: np.ndarray
    tpl_tok: np.ndarray
    template_id: np.ndarray
    src_index: np.ndarray

    @property
    def n(self) -> int:
        return len(self.template_id)


@dataclass
class Batch:
    q_off: np.ndarray   # [B+1] uint32
    q_tok: np.ndarray   # [sum] uint32
    q_src: np.ndarray   # [B] uint32 dataset row of each query

    @property
    def B(self) -> int:
        return len(self.q_src)


def _zipf_probs(n: int, s: float) -> np.ndarray:
    w = 1.0 / np.arange(1, n + 1, dtype=np.float64) ** s
    return w / w.sum()


LOG_CHUNK = 4096


def make_dataset(name: str, n_logs: int, n_templates: int, zipf_s: float, seed: int,
                 vocab: int = 2000, len_range=(4, 20), p_const: float = 0.75,
                 value_pool_range=(1, 1000), value_base: int = VALUE_BASE,
                 max_value_len: int = 8) -> Dataset:
    rng = np.random.default_rng(seed)
    word_p = _zipf_probs(vocab, 1.0)
    templates, slot_pools, seen = [], [], set()
    next_value = value_base
    while len(templates) < n_templates:
        ell = int(rng.integers(len_range[0], len_range[1] + 1))
        is_slot = rng.random(ell) >= p_const
        if not is_slot.any():
            is_slot[int(rng.integers(ell))] = True
        words = VOCAB_BASE + rng.choice(vocab, size=ell, p=word_p)
        tpl = np.where(is_slot, PH, words).astype(np.uint32)
        key = tpl.tobytes()
        if key in seen:            # template_id is a pure function of template text
            continue
        seen.add(key)
        pools = []
        for pos in np.flatnonzero(is_slot):
            sz = int(rng.integers(value_pool_range[0], value_pool_range[1] + 1))
            w = int(rng.integers(1, max_value_len + 1))
            alpha = int(rng.integers(4, 41))
            vlen = rng.integers(1, w + 1, size=sz).astype(np.int64)
            vflat = (next_value + rng.integers(0, alpha, size=int(vlen.sum()))).astype(np.uint32)
            pools.append((int(pos), vlen, vflat))         # value v = vflat[voff[v]:voff[v+1]]
            next_value += alpha
        templates.append(tpl)
        slot_pools.append(pools)
    pop = _zipf_probs(n_templates, zipf_s)
    # Logs come in chunks of doubling size (4,096, 4,096, 8,192, 16,384, ...), each drawn whole from
    # its own generator (seed, chunk): the first m logs are the same for every n_logs >= m, so a
    # longer run (more bench steps) replays the same stream prefix.
    offs, toks, tpls, base, c0, k = [], [], [], 0, 0, 0
    while c0 < n_logs:
        size = LOG_CHUNK if k == 0 else LOG_CHUNK << (k - 1)
        crng = np.random.default_rng([seed, k])
        lt = crng.choice(n_templates, size=size, p=pop).astype(np.uint32)
        lo, lk = _assemble_logs(crng, templates, slot_pools, lt)
        m = min(size, n_logs - c0)
        offs.append(lo[:m].astype(np.int64) + base)
        toks.append(lk[:int(lo[m])])
        tpls.append(lt[:m])
        base += int(lo[m]); c0 += size; k += 1
    log_off = np.concatenate(offs + [np.array([base], np.int64)]).astype(np.uint32)
    return Dataset(name, templates, log_off, np.concatenate(toks), np.concatenate(tpls))


def _ragged_arange(lens: np.ndarray) -> np.ndarray:
    """concatenate(arange(l) for l in lens), vectorised."""
    tot = int(lens.sum())
    starts = np.cumsum(lens) - lens
    return np.arange(tot, dtype=np.int64) - np.repeat(starts, lens)


def _assemble_logs(rng, templates, slot_pools, log_tpl):
    """Every log = its template with each slot replaced by a value drawn uniformly from that
    slot's pool.  Vectorised per (template, slot): the value draws of all logs of a template are
    one rng call per slot, in template order, and the ragged pieces are scattered into one flat
    token array (a 10M-log stream takes seconds, not minutes)."""
    n = len(log_tpl)
    lens = np.zeros(n, np.int64)
    plan = []
    order = np.argsort(log_tpl, kind="stable")            # logs grouped by template, row order kept
    bounds = np.concatenate([[0], np.cumsum(np.bincount(log_tpl, minlength=len(templates)))])
    for t, (tpl, pools) in enumerate(zip(templates, slot_pools)):
        idx = order[bounds[t]:bounds[t + 1]]
        if len(idx) == 0:
            plan.append(None)
            continue
        choice = []
        for pos, vlen, vflat in pools:
            voff = np.concatenate([[0], np.cumsum(vlen)])
            v = rng.integers(len(vlen), size=len(idx))
            choice.append((pos, vlen, voff, vflat, v))
        lens[idx] = (len(tpl) - len(pools)) + sum(c[1][c[4]] for c in choice)
        plan.append((idx, choice))
    log_off = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=log_off[1:])
    log_tok = np.empty(int(log_off[-1]), np.uint32)
    for t, pl in enumerate(plan):
        if pl is None:
            continue
        idx, choice = pl
        tpl = templates[t]
        cur = log_off[idx].copy()                       # write cursor of each log of template t
        prev = 0
        for pos, vlen, voff, vflat, v in choice + [(len(tpl), None, None, None, None)]:
            seg = tpl[prev:pos]                         # constant piece before this slot
            if len(seg):
                log_tok[cur[:, None] + np.arange(len(seg))[None, :]] = seg[None, :]
                cur += len(seg)
            if vlen is not None:                        # the slot's value, ragged
                L = vlen[v]
                r = _ragged_arange(L)
                log_tok[np.repeat(cur, L) + r] = vflat[np.repeat(voff[v], L) + r]
                cur += L
            prev = pos + 1
    return log_off.astype(np.uint32), log_tok


def sample_pool(ds: Dataset, M: int, seed: int, n_rows: int | None = None) -> Pool:
    """M distinct logs of the first n_rows (default: all) rows, seeded."""
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(min(n_rows or ds.n, ds.n), size=M, replace=False)).astype(np.uint32)
    log_lens = np.array([ds.log_off[r + 1] - ds.log_off[r] for r in rows], dtype=np.int64)
    tpls = [ds.templates[ds.log_tpl[r]] for r in rows]
    log_off = np.zeros(M + 1, dtype=np.int64); np.cumsum(log_lens, out=log_off[1:])
    tpl_off = np.zeros(M + 1, dtype=np.int64); np.cumsum([len(t) for t in tpls], out=tpl_off[1:])
    log_tok = np.concatenate([ds.log(int(r)) for r in rows]).astype(np.uint32)
    tpl_tok = np.concatenate(tpls).astype(np.uint32)
    return Pool(log_off.astype(np.uint32), log_tok, tpl_off.astype(np.uint32), tpl_tok,
                ds.log_tpl[rows].astype(np.uint32), rows)


def instruction(n_instr: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return (INSTR_BASE + rng.integers(0, 1 << 16, size=n_instr)).astype(np.uint32)


DECODE_BASE = 1 << 23    # synthetic decode-token ids


def decode_tokens(q_src: np.ndarray, t: int) -> np.ndarray:
    """Token t decoded for each request (a deterministic stand-in for the model's output, e.g. the
    parsed template's tokens): a function of the query row and t only."""
    return (DECODE_BASE + (np.asarray(q_src, np.uint64) * 2654435761 + np.uint64(t) * 40503) % 65536).astype(np.uint32)


def dedup_rows(ds: Dataset) -> np.ndarray:
    """The LILAC / LogBatcher stream shape: a parsing cache answers repeated logs, so
    only the first occurrence of each distinct log reaches the LLM; the rows of those first
    occurrences in dataset order."""
    seen, rows = set(), []
    for r in range(ds.n):
        key = ds.log(r).tobytes()
        if key not in seen:
            seen.add(key)
            rows.append(r)
    return np.asarray(rows, np.int64)


def make_batch_rows(ds: Dataset, rows: np.ndarray) -> Batch:
    """A batch of the given dataset rows (in the given order)."""
    rows = np.asarray(rows, np.int64)
    lens = ds.log_off[rows + 1].astype(np.int64) - ds.log_off[rows].astype(np.int64)
    q_off = np.zeros(len(rows) + 1, dtype=np.int64); np.cumsum(lens, out=q_off[1:])
    q_tok = np.concatenate([ds.log(int(r)) for r in rows]) if len(rows) else np.zeros(0, np.uint32)
    return Batch(q_off.astype(np.uint32), q_tok.astype(np.uint32), rows.astype(np.uint32))


def make_batch(ds: Dataset, start: int, B: int) -> Batch:
    """Queries start..start+B-1 in dataset order, cycled."""
    rows = (np.arange(start, start + B, dtype=np.int64) % ds.n).astype(np.uint32)
    lens = (ds.log_off[rows + 1].astype(np.int64) - ds.log_off[rows].astype(np.int64))
    q_off = np.zeros(B + 1, dtype=np.int64); np.cumsum(lens, out=q_off[1:])
    q_tok = np.concatenate([ds.log(int(r)) for r in rows]) if B else np.zeros(0, np.uint32)
    return Batch(q_off.astype(np.uint32), q_tok.astype(np.uint32), rows)


# ----------------------------------------------------------------------------------------
# Workload configurations (BASELINE.json configs)
# ----------------------------------------------------------------------------------------
@dataclass
class Config:
    name: str
    datasets: list            # list of (name, n_logs, n_templates, zipf_s, seed)
    M: int
    k: int
    B: int
    n_instr: int
    T: int
    C: int
    Hq: int
    Hkv: int
    d: int
    pool_seed: int
    qkv_seed: int = 3000
    instr_seed: int = 77
    max_prompt_tokens: int = 1024
    extra: dict = field(default_factory=dict)


def config(n: int) -> Config:
    if n == 1:
        return Config("c1-tiny-hdfs", [("HDFS", 2000, 14, 1.3, 1004)], M=200, k=3, B=100,
                      n_instr=128, T=512, C=4096, Hq=4, Hkv=4, d=64, pool_seed=2004,
                      max_prompt_tokens=512)
    if n == 2:
        return Config("c2-loghub16", [(nm, 2000, nt, 1.1, 1000 + j)
                                      for j, (nm, nt) in enumerate(LOGHUB16)],
                      M=200, k=5, B=256, n_instr=128, T=4096, C=73728, Hq=32, Hkv=8, d=128,
                      pool_seed=2000, max_prompt_tokens=1024)
    if n == 3:
        return Config("c3-2k-prompts", [("C3", 32768, 300, 1.1, 4000)], M=200, k=5, B=1024,
                      n_instr=1836, T=4096, C=73728, Hq=32, Hkv=8, d=128, pool_seed=4001,
                      max_prompt_tokens=2560)
    if n == 4:
        return Config("c4-qwen14b-skewed", [("C4", 102400, 1000, 1.3, 5000)], M=10000, k=8,
                      B=1024, n_instr=128, T=2048, C=45056, Hq=40, Hkv=8, d=128,
                      pool_seed=5001, max_prompt_tokens=1536)
    if n == 5:
        # Loghub-2.0 scale (BASELINE configs[4]): a ~10M-log stream, 5,000 templates, a 50k-demo pool;
        # 8 GPUs x 1,024 requests per global batch (k and the attention shape are unspecified there:
        # the paper's default k = 5, and the Llama shape)
        return Config("c5-loghub2-scale", [("C5", 10_485_760, 5000, 1.1, 6000)], M=50000, k=5, B=1024,
                      n_instr=128, T=4096, C=73728, Hq=32, Hkv=8, d=128, pool_seed=6001,
                      max_prompt_tokens=1024)
    raise ValueError(f"unknown config {n}")


# ----------------------------------------------------------------------------------------
# Q/K/V counter-based generator.  A pure function of
# (seed, token, absolute position, head, dim): the GPU helper il_synth_qkv implements the
# same generator independently.
# ----------------------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30); x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27); x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


QKV_TENSOR_SALT = {"q": 0x51, "k": 0x4B, "v": 0x56}


def tensor_seed(seed: int, which: str) -> int:
    return int(_mix(np.array([(seed << 8) ^ QKV_TENSOR_SALT[which]], dtype=np.uint64))[0])


def _fmix32(h: np.ndarray) -> np.ndarray:
    """murmur3 32-bit finaliser (uint32 arrays, wrapping)."""
    h = h ^ (h >> np.uint32(16))
    h = (h * np.uint32(0x85EBCA6B)).astype(np.uint32)
    h = h ^ (h >> np.uint32(13))
    h = (h * np.uint32(0xC2B2AE35)).astype(np.uint32)
    return h ^ (h >> np.uint32(16))


def synth_bf16_bits(seed: int, which: str, tokens: np.ndarray, positions: np.ndarray,
                    n_heads: int, d: int, scale: float = 1.0) -> np.ndarray:
    """[n][n_heads][d] uint16 bf16 bit patterns (Z28): per (token, position) a 64-bit
    row key r = mix(mix(seed_t ^ token) ^ position); per 4 dims (e = head * 64 + dim // 4)
    v = fmix32((lo32(r) ^ e * 0x9E3779B9) + hi32(r)); u = byte dim % 4 of v; f = 1 + u / 256;
    x = (f - 1.5) * (2 * scale) in float32 (= (u - 128) / 128 * scale, exact in bf16); RNE to bf16."""
    s = np.uint64(tensor_seed(seed, which))
    t = tokens.astype(np.uint64)[:, None, None]
    p = positions.astype(np.uint64)[:, None, None]
    r = _mix(_mix(s ^ t) ^ p)
    lo = (r & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    hi = (r >> np.uint64(32)).astype(np.uint32)
    dim = np.arange(d, dtype=np.uint32)
    e = (np.arange(n_heads, dtype=np.uint32)[None, :, None] * np.uint32(64) + (dim // np.uint32(4))[None, None, :])
    with np.errstate(over="ignore"):
        v = _fmix32(((lo ^ (e * np.uint32(0x9E3779B9)).astype(np.uint32)) + hi).astype(np.uint32))
    u = (v >> (np.uint32(8) * (dim & np.uint32(3)))[None, None, :]) & np.uint32(0xFF)
    f = (np.uint32(0x3F800000) | (u.astype(np.uint32) << np.uint32(15))).view(np.float32)
    x = (f - np.float32(1.5)) * np.float32(2.0 * scale)
    b = x.view(np.uint32).astype(np.uint64)
    rnd = ((b >> np.uint64(16)) & np.uint64(1)) + np.uint64(0x7FFF)
    return ((b + rnd) >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
