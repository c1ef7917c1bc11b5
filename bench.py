#!/usr/bin/env python
"""Benchmark: ICL requests/s of the InferLog hot path (refine + cached prefill) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A step = one batch of B concurrent requests through the whole path:
il_refine_batch (kNN + PAIR + render) -> il_prefix_match (chain hash, longest cached prefix,
LRU evict, page allocation) -> il_synth_qkv (stands in for the QKV projection of the
suffix tokens) -> il_prefill_attn (K/V append + paged prefill attention) -> il_commit.
Rank 0 prints one JSON line.  --impl reference times the CPU oracle (oracle/) instead.
Multi-GPU (torchrun): each rank runs its own slice of every global batch (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workload import gen  # noqa: E402

METRIC = "ICL requests/s (refine+cached prefill), prefix-hit %, % HBM/TC roofline"
UNIT = "requests/s"


# INT32 lane-op peak for the integer stages' ALU fractions (1 membership test /
# compare = 1 lane-op): the ALU pipe retires one warp instruction per 2 clocks per SMSP
# (B200_PROFILING.md, "fma vs alu split": rt_SMSP = 2) = 64 lanes / clk / SM, x 148 SMs x the max
# SM clock; scripts/alu_microbench.cu measures it (profiles/r02_alu_microbench.txt)
INT32_LANES_PER_CLK_SM = 64


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm": d["hbm_gbs"], "tc": d["bf16_tflops"], "tc_sustained": d.get("bf16_tflops_sustained"),
                "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm": 6650.0, "tc": 1590.0, "tc_sustained": 1400.0, "src": "fallback (B200_PROFILING.md)"}


def ncu_traffic(args=None):
    """dram read+write bytes per launch of the attention kernel from the committed ncu summary
    (profiles/attn_ncu_summary.json, written from one `ncu --set full` capture of the DEFAULT
    run: c3, PAIR, fused K/V, no decode), or None for any other workload."""
    if args is not None and (args.config != 3 or args.naive or args.no_fused_kv or args.decode or args.dedup
                             or args.batch_dedup):
        return None, "no ncu capture of this workload (profiles/attn_ncu_summary.json is the default c3 run's)"
    p = os.path.join(ROOT, "profiles", "attn_ncu_summary.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("dram_bytes_per_launch"), d.get("source")
    return None, None


# Steady state: after the cold-start ramp, untimed full batches run until the KV cache is full and
# a batch evicts (LRU, Z21), so every warm-up and timed step runs in the eviction regime.  At most
# this many fill batches (c3 starts evicting after ~70).
MAX_FILL = {1: 400, 2: 200, 3: 200, 4: 200, 5: 200}


def pipelined_on(args) -> bool:
    """The cross-batch pipelined schedule (il.h il_set_sm_split comment) is timed unless --serial,
    --no-graph or --decode."""
    return not (args.serial or args.no_graph or args.decode)


def n_queries_for(cfg, args, world: int) -> int:
    """Stream length both arms use (the same dataset instance): ramp + fill + warm-up + timed
    (2K serial steps, + 2K pipelined ones)."""
    n_timed = 2 * args.steps * (2 if pipelined_on(args) else 1)
    n = (MAX_FILL[args.config] + args.warmup + n_timed + 1) * cfg.B * world + 65 * world
    return int(n * 1.25) if getattr(args, "dedup", False) else n      # (the dedup'd stream is shorter)


class Stream:
    """The query stream: dataset rows in order, or with --dedup the LILAC / LogBatcher
    shape: only the first occurrence of each distinct log is queried."""

    def __init__(self, ds, dedup: bool):
        self.ds = ds
        self.rows = gen.dedup_rows(ds) if dedup else None

    def batch(self, start: int, B: int):
        if self.rows is None:
            return gen.make_batch(self.ds, start, B)
        return gen.make_batch_rows(self.ds, self.rows[np.arange(start, start + B) % len(self.rows)])

    @property
    def n(self) -> int:
        return self.ds.n if self.rows is None else len(self.rows)


def workload(cfg_n: int, rank: int, world: int, n_queries: int = 0):
    """Config dataset, grown (same generator, same seed) to at least n_queries logs so that no
    query repeats inside the run: the paper parses every log once.  (Config 2's 16
    datasets run through run_c2.)"""
    cfg = gen.config(cfg_n)
    name, n, nt, s, seed = cfg.datasets[0]
    ds = gen.make_dataset(name, max(n, n_queries), nt, s, seed)
    pool = gen.sample_pool(ds, cfg.M, cfg.pool_seed, n_rows=n)   # (from the configured size: the same
                                                                  # pool whatever the run length)
    instr = gen.instruction(cfg.n_instr, cfg.instr_seed)
    return cfg, ds, pool, instr


def plan_batches(cfg, n_full: int, rank: int, world: int, ramp=(1, 64)):
    """Cold-start ramp (each rank its own), then full batches: global batch g covers queries
    [off + g*B*world, ...), rank r takes the r-th slice of B (weak scaling)."""
    plan, off = [], 0
    for r in ramp:
        plan.append((off + rank * r, r)); off += r * world
    for g in range(n_full):
        plan.append((off + (g * world + rank) * cfg.B, cfg.B))
    return plan


def flops_bytes(plen, hit, bt, Hq, Hkv, d):
    """Algorithmic work of prefill attention for one batch:
    FLOPs = sum_i 4 d Hq (S_i P_i + S_i (S_i + 1) / 2); bytes = Q + O + K_new + V_new of the
    suffix rows (write + read of the appended K/V) + one read of every distinct cached page."""
    L = plen.astype(np.int64); H = hit.astype(np.int64); P = 16 * H; S = L - P
    flops = float(np.sum(4 * d * Hq * (S * P + S * (S + 1) // 2)))
    mask = np.arange(bt.shape[1])[None, :] < H[:, None]
    n_pages = len(np.unique(bt[mask]))
    byts = float(np.sum(2 * d * S * (2 * Hq + 4 * Hkv))) + 4.0 * d * Hkv * 16 * n_pages
    return flops, byts


class ClockSampler:
    def __init__(self, gpu_index: int):
        self.p = None
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.first = self.p.stdout.readline()          # sampling has started
        except Exception:
            self.p = None
            self.first = ""

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out = self.first + self.p.communicate()[0]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0])); mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def config_dict(cfg, args, world, ds):
    """The `config` of the JSON line; both arms print the same one."""
    return {"workload": cfg.name, "baseline_config": f"configs[{args.config - 1}]",
            "requests_per_gpu_per_step": cfg.B, "k": cfg.k, "pool": cfg.M, "instr_tokens": cfg.n_instr,
            "table_capacity": cfg.T, "kv_pages": cfg.C, "heads_q_kv_d": [cfg.Hq, cfg.Hkv, cfg.d],
            "layers": 1, "flags": ("naive-PC" if args.naive else ("PAIR+verify" + ("" if args.no_guard else "+guard")))
            + ("+batch-dedup" if args.batch_dedup else ""),
            "l2": ("serial steps: flushed (256 MiB write) before each step; pipelined steps (the headline): no flush, "
                   "the attention alone moves ~1.2 GB of DRAM per step at c3 (ncu), ~10x the 126 MB L2"
                   if pipelined_on(args) else "flushed (256 MiB write) between timed steps"),
            "parallelism": f"dp{world} (request shards)",
            "stream": f"{ds.n} distinct logs, no query repeats within the run",
            "steady_state": "LRU eviction in every timed step" if not args.no_fill else "no fill",
            "int_dtype": "u32/u64 bit-exact", "attn": "bf16 in, fp32 accumulate"}


# ---------------------------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2507_08523_b200 import IL_F_DEDUP, IL_F_GUARD, IL_F_PAIR, IL_F_VERIFY, Config, Pipeline

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg0 = gen.config(args.config)
    cfg, ds, pool, instr = workload(args.config, rank, world, n_queries=n_queries_for(cfg0, args, world))
    stream_q = Stream(ds, args.dedup)
    flags = IL_F_PAIR | IL_F_VERIFY | (IL_F_GUARD if not args.no_guard else 0)
    if args.naive:
        flags = IL_F_VERIFY
    if args.batch_dedup:
        flags |= IL_F_DEDUP
    ccfg = Config(k=cfg.k, table_capacity=cfg.T, kv_pages=cfg.C, max_batch=cfg.B,
                  max_prompt_tokens=cfg.max_prompt_tokens, max_pool=cfg.M,
                  max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16, max_log_tokens=255,
                  max_suffix_tokens=cfg.B * cfg.max_prompt_tokens, n_q_heads=cfg.Hq, n_kv_heads=cfg.Hkv,
                  head_dim=cfg.d, flags=flags, max_global_batch=cfg.B * world, max_decode_tokens=args.decode)
    # (IL_BENCH_PRIO=1: the integer stream at high priority, so its kernels take the SMs the
    # attention grids free at their boundaries -- A / B knob)
    stream = torch.cuda.Stream(dev, priority=-1) if os.environ.get("IL_BENCH_PRIO") else torch.cuda.Stream(dev)
    piped = pipelined_on(args)
    # (IL_SPLIT_SYNTH=1: batch j+1's Q on the integer stream, its K / V after batch j's attention --
    # measured slower, 1.10-1.11 vs 1.06 ms per step: the integer stream only has the attention's gaps)
    split_synth = piped and not args.no_fused_kv and bool(os.environ.get("IL_SPLIT_SYNTH"))
    select_ahead = os.environ.get("IL_SELECT_AHEAD", "1") == "1"    # (0: select in batch order)
    # (two per-batch buffer slots for the pipelined schedule: batch b's attention reads slot b % 2
    # while batch b+1's integer stages write the other)
    pl = Pipeline(ccfg, dev, qkv_seed=cfg.qkv_seed, stream=stream, fused_kv=not args.no_fused_kv,
                  slots=2 if piped else 1)
    # N > 1: rank r runs the r-th slice of every global batch; the pool is
    # broadcast from rank 0; per batch one record buffer per rank (ICL records + prefix-index
    # updates) is all-gathered (NCCL) on a side stream, overlapping the next batch's selection
    dp = None
    if world > 1:
        from paper_2507_08523_b200.distributed import DataParallel
        dp = DataParallel(pl)
    with torch.cuda.stream(stream):
        (dp or pl).load_pool(pool, instr)
    step = dp.step if dp else pl.step
    if args.decode and dp is not None:
        raise SystemExit("--decode is measured at N = 1 only")
    if args.decode and dp is None:
        def step():                                    # eager step with the decode tokens
            pl.refine(); pl.match(); pl.synth(); pl.attn()
            for t in range(args.decode):
                pl.decode_step(t, dec_tok[t], lse=False)
            pl.commit()
    K, W = args.steps, args.warmup
    n_fill_max = 0 if args.no_fill else MAX_FILL[args.config]
    n_timed = 2 * K * (2 if piped else 1)
    plan = plan_batches(cfg, n_fill_max + W + n_timed, rank, world)
    n_ramp = len(plan) - (n_fill_max + W + n_timed)

    dec_tok = torch.zeros(args.decode, cfg.B, dtype=torch.int64, device=dev) if args.decode else None

    def dec_of(bt):                                    # the batch's decode tokens [D][B] (NEXT-4 stand-ins)
        return torch.from_numpy(np.stack([gen.decode_tokens(bt.q_src, t) for t in range(max(args.decode, 1))])
                                .astype(np.int64))

    def to_dev(bt):
        return (torch.from_numpy(bt.q_off.view(np.int32)).to(dev), torch.from_numpy(bt.q_tok.view(np.int32)).to(dev),
                torch.from_numpy(bt.q_src.view(np.int32)).to(dev), bt.B, dec_of(bt).to(dev))

    def to_pinned(bt):
        return (tuple(torch.from_numpy(a.view(np.int32)).pin_memory() for a in (bt.q_off, bt.q_tok, bt.q_src))
                + (bt.B, dec_of(bt).pin_memory()))

    def set_inputs(x):
        pl.load_inputs(*x[:4])                         # device-to-device into the resident input buffers
        if dec_tok is not None:
            dec_tok[:, :x[3]].copy_(x[4])

    # ---- cold-start ramp, then fill until a batch evicts (untimed; all ranks stop together)
    stats_dev = torch.zeros(128, dtype=torch.uint8, device=dev)
    j = 0
    with torch.cuda.stream(stream):
        for j in range(n_ramp + n_fill_max):
            set_inputs(to_dev(stream_q.batch(*plan[j])))
            step()
            if j < n_ramp:
                continue
            pl.ctx.stats_async(stats_dev, stream=stream)
            ev_now = pl.ctx.stats_from_bytes(stats_dev.cpu().numpy())["evicted_blocks"]
            flag = torch.tensor([1 if ev_now > 0 else 0], device=dev)
            if world > 1:
                dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            if int(flag.item()):
                break
    n_fill = j + 1 - n_ramp if n_fill_max else 0
    plan = plan[:n_ramp + n_fill] + plan[n_ramp + n_fill_max:]
    stream.synchronize()
    batches = [stream_q.batch(s, b) for s, b in plan[n_ramp + n_fill:]]

    # Timed steps alternate: even = device-timed (inputs already resident in HBM), odd = end to
    # end (pinned host inputs copied in, refined DS / info / hits copied out inside the timed
    # region), so both see the same part of the stream.
    warm_in = [to_dev(bt) for bt in batches[:W]]
    timed = batches[W:W + 2 * K]
    dev_in = [to_dev(bt) if j % 2 == 0 else None for j, bt in enumerate(timed)]
    host_in = [to_pinned(bt) if j % 2 == 1 else None for j, bt in enumerate(timed)]
    # the pipelined schedule's batches: K device-resident, then K from pinned host memory
    piped_dev = [to_dev(bt) for bt in batches[W + 2 * K:W + 3 * K]] if piped else []
    piped_host = [to_pinned(bt) for bt in batches[W + 3 * K:W + 4 * K]] if piped else []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    out_fin = torch.empty(cfg.B, cfg.k, dtype=torch.int32).pin_memory()
    out_hit = torch.empty(cfg.B, dtype=torch.int32).pin_memory()
    out_info = torch.empty(cfg.B, 16, dtype=torch.uint8).pin_memory()
    # per-step accounting kept on the device (no host sync inside the timed region)
    rec_len = torch.zeros(K, cfg.B, dtype=torch.int32, device=dev)
    rec_hit = torch.zeros(K, cfg.B, dtype=torch.int32, device=dev)
    rec_bt = torch.zeros(K, cfg.B, ccfg.max_blocks, dtype=torch.int32, device=dev)
    rec_info = torch.zeros(K, cfg.B, 16, dtype=torch.uint8, device=dev)
    rec_stats = torch.zeros(2 * K, 128, dtype=torch.uint8, device=dev)   # il_stats after every timed step

    # ---- warm-up (W full steps in the eviction regime), not timed
    with torch.cuda.stream(stream):
        for x in warm_in:
            set_inputs(x)
            step()
    stream.synchronize()
    pl.ctx.status_sync(stream)

    # The stages of one step.  N = 1: il_refine_batch .. il_commit.  N > 1: il_select_batch (a1-a2,
    # overlapping the previous batch's record all-gather), then il_commit_apply of the gathered
    # records + il_refine_batch, .., il_commit_index + il_commit_export; the all-gather itself
    # (NCCL, side stream) and the wait for it stay outside the stages.
    if args.decode:
        def decode_all():
            for t in range(args.decode):
                pl.decode_step(t, dec_tok[t], lse=False)
    if dp is None:
        stage_fns = {"select": pl.select, "refine": pl.refine, "match": pl.match, "synth": pl.synth,
                     "attn": pl.attn, "commit": pl.commit}
        if args.decode:
            stage_fns = {k: v for k, v in list(stage_fns.items())[:5]}
            stage_fns["decode"] = decode_all
            stage_fns["commit"] = pl.commit
    else:
        stage_fns = {"select": dp.select, "refine": lambda: (dp.apply_records(), pl.refine()),
                     "match": pl.match, "synth": pl.synth, "attn": pl.attn, "commit": dp.export}
    stage_names = list(stage_fns)
    # CUDA graphs: each stage captured once for B (one replay per stage, no per-kernel launch gaps;
    # every library call of the step is inside a graph, so the host-side call-order state stays
    # consistent).  Capture does not run the kernels: the warm-up's pending records are applied by
    # the first replay of the "refine" stage.
    graphs, per_step_launches = None, None
    if not args.no_graph:
        l0 = pl.launches()
        pl.B = cfg.B
        graphs = {}
        for slot in range(2 if piped else 1):          # one set of stage graphs per buffer slot
            pl.use(slot)
            for name in stage_names:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    stage_fns[name]()
                graphs[slot, name] = g
                if slot == 0 and name == "commit":
                    per_step_launches = pl.launches() - l0
                if piped and name == "synth" and split_synth:
                    for part in ("q", "kv"):           # the pipelined schedule's split of the stand-in
                        g = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(g, stream=stream):
                            pl.synth(part=part)
                        graphs[slot, "synth_" + part] = g
                    l0 += 2                           # (not extra launches of a step)
        pl.use(0)
        stream.synchronize()

    def run_stage(name):
        if dp is not None and name == "refine":
            dp.wait_gathered()                         # (eager: an event wait, never captured)
        if graphs is not None:
            graphs[pl.slot, name].replay()
        else:
            stage_fns[name]()
        if dp is not None and name == "commit":
            dp.gather()                                # all-gather on the comm stream (eager)

    def run_step():
        for n in stage_names:
            run_stage(n)

    evs, e2e_evs = [], []
    h2d = d2h = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    t_wall = time.perf_counter()
    launches0 = pl.launches()
    prof = None
    if os.environ.get("IL_BENCH_PROFILE"):             # diagnostics only: kernel timeline of the timed loop
        from torch.profiler import ProfilerActivity, profile
        prof = profile(activities=[ProfilerActivity.CUDA])
        prof.__enter__()
    with torch.cuda.stream(stream):
        for j in range(2 * K):
            flush.zero_()
            if j % 2 == 0:
                set_inputs(dev_in[j])
                e = [ev() for _ in range(len(stage_names) + 1)]
                for i, n in enumerate(stage_names):
                    e[i].record(stream)
                    run_stage(n)
                e[-1].record(stream)
                pl.ctx.stats_async(rec_stats[j], stream=stream)
                evs.append(e)
                B = dev_in[j][3]
                rec_len[j // 2, :B].copy_(pl.prompt_len[:B]); rec_hit[j // 2, :B].copy_(pl.hit[:B])
                rec_bt[j // 2, :B].copy_(pl.block_table[:B])
                rec_info[j // 2, :B].copy_(pl.info[:B])
            else:
                qo, qt, qs, B, dt = host_in[j]
                e0, e1 = ev(), ev()
                e0.record(stream)
                pl.q_off[:B + 1].copy_(qo, non_blocking=True)        # pinned host -> resident buffers
                pl.q_tok[:qt.numel()].copy_(qt, non_blocking=True)
                pl.q_src[:B].copy_(qs, non_blocking=True)
                if dec_tok is not None:
                    dec_tok[:, :B].copy_(dt, non_blocking=True)
                pl.B = B
                run_step()
                out_fin[:B].copy_(pl.final_ds[:B], non_blocking=True)
                out_hit[:B].copy_(pl.hit[:B], non_blocking=True)
                out_info[:B].copy_(pl.info[:B], non_blocking=True)
                e1.record(stream)
                pl.ctx.stats_async(rec_stats[j], stream=stream)
                e2e_evs.append((e0, e1))
                h2d = 4 * (qo.numel() + qt.numel() + qs.numel()) + (8 * dt.numel() if dec_tok is not None else 0)
                d2h = 4 * B * cfg.k + 4 * B + 16 * B
    torch.cuda.synchronize()

    # ---- the pipelined schedule (il.h, il_set_sm_split comment): batch j's synth + attention on
    # stream sA overlap batch j's commit and batch j+1's select / refine / match on `stream`; buffer
    # slot j % 2; batch j+2 reuses slot j % 2 only after batch j's attention.  No L2 flush: the
    # inputs each batch streams (its Q / K / V and the KV pages it reads, ~1.4 GB at c3) exceed the
    # 126 MB L2 (the serial steps flush, outside their events).  Device-resident inputs (value),
    # then pinned host inputs with the integer results copied back (e2e).  Timed from before the
    # first batch to after the last.
    sA = torch.cuda.Stream(dev)
    pipe = {}

    def run_pipelined(inputs, host):
        n = len(inputs)
        ev_m = [torch.cuda.Event() for _ in range(n)]
        ev_a = [torch.cuda.Event() for _ in range(n)]
        e0, e1 = ev(), ev()
        e0.record(stream)
        sA.wait_stream(stream)
        # select_ahead: batch j+1's a1-a2 (il_select_batch reads only the pool) is issued right after
        # batch j's match, ahead of batch j's commit, so it runs beside batch j's QKV stand-in instead
        # of after batch j's attention (the integer stream only gets the SMs the attention leaves)
        ahead = select_ahead and stage_names[0] == "select"

        def stage_in(jj, xx):
            pl.use(jj % 2)
            if host:
                qo, qt, qs, B = xx[:4]
                pl.q_off[:B + 1].copy_(qo, non_blocking=True)
                pl.q_tok[:qt.numel()].copy_(qt, non_blocking=True)
                pl.q_src[:B].copy_(qs, non_blocking=True)
                pl.B = B
            else:
                set_inputs(xx)

        if ahead:
            with torch.cuda.stream(stream):
                stage_in(0, inputs[0])
                run_stage("select")
        for j, x in enumerate(inputs):
            with torch.cuda.stream(stream):
                if j >= 2:
                    stream.wait_event(ev_a[j - 2])     # slot j % 2 is free again
                if ahead:
                    pl.use(j % 2)
                    pl.B = x[3]
                else:
                    stage_in(j, x)
                for name in stage_names[:-3]:          # select, refine, match
                    if not (ahead and name == "select"):
                        run_stage(name)
                if split_synth:
                    graphs[j % 2, "synth_q"].replay()  # Q of batch j: no page writes
                ev_m[j].record(stream)
                if host:
                    out_fin[:x[3]].copy_(pl.final_ds[:x[3]], non_blocking=True)
                    out_hit[:x[3]].copy_(pl.hit[:x[3]], non_blocking=True)
                    out_info[:x[3]].copy_(pl.info[:x[3]], non_blocking=True)
                if ahead and j + 1 < n:                # batch j+1's inputs + a1-a2 into slot (j+1) % 2
                    stage_in(j + 1, inputs[j + 1])     # (batch j-1's attention reads none of them)
                    run_stage("select")
                    pl.use(j % 2)
                    pl.B = x[3]
            with torch.cuda.stream(sA):
                sA.wait_event(ev_m[j])
                for name in (("synth_kv" if split_synth else "synth"), "attn"):
                    graphs[j % 2, name].replay()
                ev_a[j].record(sA)
            with torch.cuda.stream(stream):
                run_stage("commit")                    # after match(j) on `stream`, beside the attention
        stream.wait_stream(sA)
        e1.record(stream)
        return e0, e1

    if piped:
        assert stage_names[-3:] == ["synth", "attn", "commit"], stage_names
        for key, inputs, host in (("device", piped_dev, False), ("e2e", piped_host, True)):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            pipe[key] = run_pipelined(inputs, host)
            torch.cuda.synchronize()
        pl.use(0)
    if dp is not None:
        with torch.cuda.stream(stream):
            dp.flush()                                 # the last batch's records (after the timed region)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall
    if prof is not None:
        prof.__exit__(None, None, None)
        evs_p = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
        t0p, prev = evs_p[0].time_range.start, None
        for e in evs_p[-int(os.environ.get("IL_BENCH_PROFILE_N", "90")):]:
            gap = (e.time_range.start - prev) if prev else 0
            print(f"{e.time_range.start - t0p:10.1f} us dur {e.time_range.elapsed_us():8.1f} gap {gap:7.1f} {e.name[:60]}",
                  file=sys.stderr)
            prev = e.time_range.end
    clk = clocks.stop()
    launches = pl.launches() - launches0 - 2 * K      # minus the per-step k_stats (accounting, not the path)
    if graphs is not None:                             # replays do not pass through the host counter
        launches += per_step_launches * (2 * K + (2 * K if piped else 0)) + (2 * K if split_synth else 0)
    st_steps = [pl.ctx.stats_from_bytes(r) for r in rec_stats.cpu().numpy()]
    evicted = [s_["evicted_blocks"] for s_ in st_steps]
    # hit accounting of every timed step (device counters), summed over ranks: rank-local hits and
    # box-level hits (this rank's index or the residency map, §8(e))
    hb = torch.tensor([sum(s_[f] for s_ in st_steps) for f in ("hit_blocks", "box_hit_blocks", "full_blocks")],
                      dtype=torch.float64, device=dev)
    backlog = max(s_["record_backlog"] for s_ in st_steps)
    if world > 1:
        dist.all_reduce(hb)
    pl.ctx.status_sync(stream)
    if world > 1:
        dist.barrier()
    step_ms = [e[0].elapsed_time(e[-1]) for e in evs]
    stage_ms = {n: [e[i].elapsed_time(e[i + 1]) for e in evs] for i, n in enumerate(stage_names)}
    e2e_ms = [a.elapsed_time(b) for a, b in e2e_evs]
    work, hits, fulls, hit_tok, all_tok, mwork, mtouch = [], 0, 0, 0, 0, [], []
    L_all, H_all, BT_all = rec_len.cpu().numpy(), rec_hit.cpu().numpy(), rec_bt.cpu().numpy()
    from paper_2507_08523_b200.context import INFO_DTYPE
    inf_all = rec_info.cpu().numpy()
    rules, pmcs = np.zeros(4, np.int64), np.zeros(cfg.k + 1, np.int64)
    for j in range(K):
        B = dev_in[2 * j][3]
        L, H = L_all[j, :B].astype(np.int64), H_all[j, :B].astype(np.int64)
        work.append(flops_bytes(L_all[j, :B], H_all[j, :B], BT_all[j, :B], cfg.Hq, cfg.Hkv, cfg.d))
        hits += int(H.sum()); fulls += int((L // 16).sum())
        hit_tok += int(16 * H.sum()); all_tok += int(L.sum())
        # SURVEY §8(d).2 a6 algorithmic bytes: prompt tokens + block hashes + block table, one
        # 32-byte probe per looked-up block (hits + the first miss) and a 64-byte verification
        # read per hit page (the instruction's blocks are probed once per batch)
        F = L // 16
        mwork.append(float((4 * L + 8 * F + 4 * ((L + 15) // 16)).sum() + 32 * (H + 1).sum() + 64 * H.sum()))
        # the bytes this implementation must move: the instruction's blocks are hashed and probed
        # once per batch (exact shortcut), so per request only the tokens past the instruction are
        # read and only its own blocks probed / verified
        nI = cfg.n_instr // 16
        hI = np.minimum(H, nI)
        mtouch.append(float((4 * np.maximum(L - 16 * nI, 0) + 8 * F + 4 * ((L + 15) // 16)).sum()
                            + 32 * (H - hI + 1).sum() + 64 * (H - hI).sum()))
        inf = inf_all[j, :B].reshape(-1).view(INFO_DTYPE)
        rules += np.bincount(inf["rule"], minlength=4)[:4]
        pmcs += np.bincount(np.minimum(inf["pmc"], cfg.k), minlength=cfg.k + 1)[:cfg.k + 1]

    # ---- reduce over ranks (max time)
    ms = float(np.mean(step_ms)); e2e = float(np.mean(e2e_ms))
    pms = pe2e = 0.0
    if piped:
        pms = pipe["device"][0].elapsed_time(pipe["device"][1]) / K
        pe2e = pipe["e2e"][0].elapsed_time(pipe["e2e"][1]) / K
    if world > 1:
        t = torch.tensor([ms, e2e, pms, pe2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, e2e, pms, pe2e = (float(x) for x in t)
    serial_ms, serial_e2e = ms, e2e
    if piped:                                          # the headline is the pipelined schedule
        ms, e2e = pms, pe2e
    if rank != 0:
        return
    pk = peaks()
    fl = np.array([w[0] for w in work]); by = np.array([w[1] for w in work])
    at = np.array(stage_ms["attn"]) * 1e-3
    t_tc = fl / (pk["tc"] * 1e12); t_hbm = by / (pk["hbm"] * 1e9)
    bound = "tensor" if t_tc.sum() >= t_hbm.sum() else "hbm"
    if bound == "tensor":
        achieved = float(fl.sum() / at.sum() / 1e12); peak = pk["tc"]; unitr = "TFLOP/s"
    else:
        achieved = float(by.sum() / at.sum() / 1e9); peak = pk["hbm"]; unitr = "GB/s"
    B_all = cfg.B * world
    # per-stage roofline: the match stage against HBM with its algorithmic bytes;
    # the integer stages with no HBM-sized work are latency bound and reported as times only
    mt = np.array(stage_ms["match"]) * 1e-3
    mw = np.array(mwork)
    clk_hz = (clk.get("sm_max_mhz") or 1965.0) * 1e6
    int32_peak = INT32_LANES_PER_CLK_SM * 148 * clk_hz            # lane-ops / s
    pool_u = int(sum(len(np.unique(pool.log_tok[pool.log_off[m]:pool.log_off[m + 1]])) for m in range(pool.n)))
    stage_roof = {
        "match": {"bound": "hbm (algorithmic); latency in practice", "bytes_per_step": float(mw.mean()),
                  "achieved": float(mw.sum() / mt.sum() / 1e9), "peak": pk["hbm"], "unit": "GB/s",
                  "frac": float(mw.sum() / mt.sum() / 1e9 / pk["hbm"]),
                  "bytes_touched_per_step": float(np.mean(mtouch)),
                  "frac_touched": float(np.sum(mtouch) / mt.sum() / 1e9 / pk["hbm"]),
                  "note": "bytes = SURVEY 8(d).2 formula (every prompt token read); bytes_touched = what this "
                          "implementation moves (instruction blocks hashed and probed once per batch)"},
        "attn": {"bound": bound, "frac": achieved / peak},
        **({"select": {"bound": "ALU (INT32 lane-ops)", "ms": float(np.mean(stage_ms["select"])),
                       "membership_tests_per_step": float(cfg.B * pool_u), "int32_peak_lane_ops_per_s": int32_peak,
                       "frac": float(cfg.B * pool_u / (np.mean(stage_ms["select"]) * 1e-3) / int32_peak),
                       "note": "a1+a2: B x sum_m u_m membership tests (SURVEY 8(d).2) / (64 lanes/clk/SM x 148 x clock)"}}
           if "select" in stage_ms else {}),
        "refine": {"bound": "ALU (PMC) / HBM write (render)", "ms": float(np.mean(stage_ms["refine"])),
                   "pmc_compares_per_step": float(cfg.B * np.mean([s_["table_entries"] for s_ in st_steps]) * cfg.k ** 2),
                   "pmc_frac_of_int32": float(cfg.B * np.mean([s_["table_entries"] for s_ in st_steps]) * cfg.k ** 2
                                              / (np.mean(stage_ms["refine"]) * 1e-3) / int32_peak),
                   "render_bytes_per_step": float(np.mean([4 * L_all[j, :dev_in[2 * j][3]].astype(np.int64).sum() for j in range(K)])),
                   "render_frac_of_hbm": float(np.mean([4 * L_all[j, :dev_in[2 * j][3]].astype(np.int64).sum() for j in range(K)])
                                               / (np.mean(stage_ms["refine"]) * 1e-3) / (pk["hbm"] * 1e9)),
                   "note": "a3 (PMC vs the ICL Table) + a4 (rules, guard) + a5 (render): compares / INT32 lane-op peak, "
                           "prompt bytes written / HBM peak, both over the whole stage time"},
        "commit": {"bound": "latency", "ms": float(np.mean(stage_ms["commit"]))},
        "synth": {"bound": "ALU (stand-in generator, not the method)", "ms": float(np.mean(stage_ms["synth"]))},
    }
    t_star_step = float(np.maximum(t_tc, t_hbm).mean() * 1e3 + mw.mean() / (pk["hbm"] * 1e9) * 1e3)
    def decode_roof():
        """Decode is HBM-bound: per decode step the K / V of every request's own blocks (past the
        batch-shared instruction blocks, read once) are read: algorithmic bytes = (shared blocks +
        sum_i own blocks) x 16 x Hkv x d x 2 B x 2 (K and V), averaged over the D steps."""
        nI = cfg.n_instr // 16
        tot = 0.0
        for j in range(K):
            Bj = dev_in[2 * j][3]
            Lj = L_all[j, :Bj].astype(np.int64)
            for t in range(args.decode):
                blocks = nI + np.maximum((Lj + t + 1 + 15) // 16 - nI, 0).sum()
                tot += blocks * 16 * cfg.Hkv * cfg.d * 2 * 2
        per_step = tot / (K * args.decode)
        t_step = np.mean(stage_ms["decode"]) * 1e-3 / args.decode
        return {"bound": "hbm", "bytes_per_decode_step": per_step, "achieved_gbs": per_step / t_step / 1e9,
                "frac_of_hbm": per_step / t_step / (pk["hbm"] * 1e9)}

    line = {
        "metric": METRIC, "value": B_all / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "config": config_dict(cfg, args, world, ds),
        "steady_state": {"ramp_batches": n_ramp, "fill_batches": n_fill,
                         "evicted_blocks_per_step": {"mean": float(np.mean(evicted)), "min": int(np.min(evicted)),
                                                     "max": int(np.max(evicted))},
                         "evicting_steps": f"{sum(1 for x in evicted if x > 0)}/{len(evicted)}",
                         "resident_blocks": int(st_steps[-1]["resident_blocks"]),
                         "note": "untimed full batches after the ramp until the KV cache is full and a batch "
                                 "evicts; every timed step then runs LRU eviction (rank 0's counts)"},
        "decode": None if not args.decode else {
            "tokens_per_request": args.decode, "ms_per_step": float(np.mean(stage_ms["decode"])),
            "tokens_per_s": B_all * args.decode / (np.mean(stage_ms["decode"]) * 1e-3),
            **decode_roof(),
            "note": "SURVEY 8(f) NEXT-4: after the cached prefill, D decode steps per request, one row per request "
                    "through il_prefill_attn at positions L_i + t into the pages il_prefix_match reserved (Q/K/V from "
                    "the synthetic projection); part of ms_per_step, as the stage 'decode'"},
        "stream_shape": "dedup (first occurrence of each distinct log; LILAC / LogBatcher, P:637-675): "
                        f"{stream_q.n} of {ds.n} logs" if args.dedup else "every log once (S:148)",
        "prefix_hit_pct": 100.0 * hits / max(fulls, 1),
        "box_level": None if dp is None else {
            "hit_pct_rank_local": 100.0 * float(hb[0]) / max(float(hb[2]), 1.0),
            "hit_pct_box": 100.0 * float(hb[1]) / max(float(hb[2]), 1.0),
            "note": "all ranks, all timed steps: leading blocks resident in the rank's own index vs in any rank's "
                    "(the replicated residency map built from the all-gathered block records)",
            "record_bytes_per_rank": dp.rec_bytes, "record_backlog_max": int(backlog),
            "collective": "one all_gather_into_tensor of the record buffers per batch, overlapping il_select_batch"},
        "prefix_hit_pct_tokens": 100.0 * hit_tok / max(all_tok, 1),
        "pair": {"rule_counts": {"1_target": int(rules[1]), "2_unchanged": int(rules[2]), "3_modified": int(rules[3])},
                 "pmc_histogram": [int(x) for x in pmcs]},
        "stage_ms": {n: float(np.mean(v)) for n, v in stage_ms.items()},
        "stage_roofline": stage_roof,
        "roofline_requests_per_s": B_all / (t_star_step * 1e-3) if t_star_step else None,
        "attention_stack_equivalent_32_layers": {
            "value": B_all / ((sum(np.mean(v) for n, v in stage_ms.items() if n != "attn")
                               + 32 * np.mean(stage_ms["attn"])) * 1e-3),
            "unit": UNIT, "note": "B / (t_integer + t_synth + 32 x t_attention): one attention layer is what runs; 32 is the Llama-3-8B depth"},
        "roofline": {"kernel": "il_prefill_attn (attention; the suffix K/V written into the pages by the QKV-"
                               "projection stand-in's epilogue)" if not args.no_fused_kv else
                               "il_prefill_attn (K/V append + attention)", "bound": bound, "achieved": achieved,
                     "peak": peak, "unit": unitr, "frac": achieved / peak, "traffic": ncu_traffic(args)[0],
                     "traffic_src": ncu_traffic(args)[1],
                     "peak_src": pk["src"] + (" burst bf16" if bound == "tensor" else ""),
                     "flops_per_step": float(fl.mean()), "bytes_per_step": float(by.mean()),
                     "t_star_ms": float(np.maximum(t_tc, t_hbm).mean() * 1e3)},
        "e2e": {"value": B_all / (e2e * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e},
        "schedule": {
            "kind": "pipelined" if piped else "serial",
            "note": ("value / e2e: batch b's QKV stand-in + attention (one stream) overlap batch b's commit and batch "
                     "b+1's select / refine / match (another stream), two per-batch buffer slots, the attention on "
                     "every SM (il_set_sm_split measured slower: the latency-bound integer stages need the whole "
                     "GPU); stage_ms, roofline and the per-step accounting come from the serial steps"
                     if piped else "one batch at a time on one stream"),
            "serial": {"value": B_all / (serial_ms * 1e-3), "ms_per_step": serial_ms,
                       "e2e_value": B_all / (serial_e2e * 1e-3), "e2e_ms_per_step": serial_e2e},
            **({"pipelined": {"value": B_all / (pms * 1e-3), "ms_per_step": pms,
                              "e2e_value": B_all / (pe2e * 1e-3), "e2e_ms_per_step": pe2e}} if piped else {})},
        "gpu_launches": int(launches),
        "timed_steps": {"serial_device": K, "serial_e2e": K, "serial_order": "alternating",
                        **({"pipelined_device": K, "pipelined_e2e": K} if piped else {}),
                        "launch": "eager" if graphs is None else "per-stage CUDA graphs"},
        "clocks": clk,
        "wall_s_timed": wall,
    }
    if not args.no_cpu_baseline and world == 1:        # (the contract: rank 0 at N = 1 only)
        line["cpu_baseline"] = cpu_baseline(args, cfg, ds, pool, instr, plan, n_ramp + n_fill + W, flags)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
def run_c2(args, rank, world, local_rank):
    """BASELINE configs[1]: all 16 Loghub-2k-shaped datasets, each from a FRESH pool,
    ICL Table and prefix cache, all 2,000 logs of the dataset as 8 batches of up to 256 concurrent
    requests (the paper's per-dataset cold run), with PAIR and again with naive prefix
    caching (PAIR off, the paper's baseline PC).  Every batch is device-timed with CUDA
    events on the launching stream (L2 flushed before each).  value = total requests / total time
    of the PAIR runs; per dataset: requests/s, block- and token-weighted hits, PAIR / naive hit
    ratio.  One GPU; ranks > 0 exit (the datasets are independent problems)."""
    import torch
    from paper_2507_08523_b200 import IL_F_DEDUP, IL_F_GUARD, IL_F_PAIR, IL_F_VERIFY, Config, Pipeline
    if rank != 0:
        return
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = gen.config(2)
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    per, tot_req, tot_ms = [], 0, 0.0
    clocks = ClockSampler(local_rank)
    launches = 0
    # the first dataset once more in front, untimed: one-time costs (module load, first launches)
    for d_ix, (name, n, nt, zs, seed) in enumerate([cfg.datasets[0]] + list(cfg.datasets)):
        warm = d_ix == 0
        ds = gen.make_dataset(name, n, nt, zs, seed)
        pool = gen.sample_pool(ds, cfg.M, cfg.pool_seed)
        instr = gen.instruction(cfg.n_instr, cfg.instr_seed)
        row = {"dataset": name, "templates": nt}
        for mode, flags in (("pair", IL_F_PAIR | IL_F_VERIFY | (0 if args.no_guard else IL_F_GUARD)),
                            ("naive", IL_F_VERIFY)):
            ccfg = Config(k=cfg.k, table_capacity=cfg.T, kv_pages=cfg.C, max_batch=cfg.B,
                          max_prompt_tokens=cfg.max_prompt_tokens, max_pool=cfg.M,
                          max_pool_tokens=int(max(pool.log_off[-1], pool.tpl_off[-1])) + 16, max_log_tokens=255,
                          max_suffix_tokens=cfg.B * cfg.max_prompt_tokens, n_q_heads=cfg.Hq, n_kv_heads=cfg.Hkv,
                          head_dim=cfg.d, flags=flags | (IL_F_DEDUP if args.batch_dedup else 0))
            pl = Pipeline(ccfg, dev, qkv_seed=cfg.qkv_seed, stream=stream)
            with torch.cuda.stream(stream):
                pl.load_pool(pool, instr)
            batches = [gen.make_batch(ds, s0, min(cfg.B, ds.n - s0)) for s0 in range(0, ds.n, cfg.B)]
            ins = [(torch.from_numpy(b.q_off.view(np.int32)).to(dev), torch.from_numpy(b.q_tok.view(np.int32)).to(dev),
                    torch.from_numpy(b.q_src.view(np.int32)).to(dev), b.B) for b in batches]
            l0 = pl.launches()
            evs, hits, fulls, htok, atok = [], 0, 0, 0, 0
            stats = torch.zeros(len(ins), 128, dtype=torch.uint8, device=dev)
            lens = []
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                for j, x in enumerate(ins):
                    flush.zero_()
                    pl.load_inputs(*x)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    pl.step()
                    e1.record(stream)
                    pl.ctx.stats_async(stats[j], stream=stream)
                    evs.append((e0, e1))
                    lens.append((pl.prompt_len[:x[3]].clone(), pl.hit[:x[3]].clone()))
            torch.cuda.synchronize()
            pl.ctx.status_sync(stream)
            launches += pl.launches() - l0 - len(ins)
            ms = sum(a.elapsed_time(b) for a, b in evs)
            for L_, H_ in lens:
                L_ = L_.cpu().numpy().astype(np.int64); H_ = H_.cpu().numpy().astype(np.int64)
                hits += int(H_.sum()); fulls += int((L_ // 16).sum()); htok += int(16 * H_.sum()); atok += int(L_.sum())
            row[mode] = {"requests_per_s": ds.n / (ms * 1e-3), "ms": ms, "block_hit_pct": 100.0 * hits / max(fulls, 1),
                         "token_hit_pct": 100.0 * htok / max(atok, 1)}
            if args.batch_dedup:                       # hits above include the in-batch shared blocks
                dd = sum(pl.ctx.stats_from_bytes(stats[j].cpu().numpy())["dedup_blocks"] for j in range(len(ins)))
                row[mode]["dedup_blocks"] = int(dd)
                row[mode]["cache_block_hit_pct"] = 100.0 * (hits - dd) / max(fulls, 1)
            if mode == "pair" and not warm:
                tot_req += ds.n; tot_ms += ms
            del pl
        row["pair_over_naive_block_hit"] = row["pair"]["block_hit_pct"] / max(row["naive"]["block_hit_pct"], 1e-9)
        if not warm:
            per.append(row)
    clk = clocks.stop()
    hp = [r["pair"]["block_hit_pct"] for r in per]; hn = [r["naive"]["block_hit_pct"] for r in per]
    line = {"metric": METRIC, "value": tot_req / (tot_ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": len(per),
            "warmup": 0, "ms_per_step": tot_ms / max(sum(len(range(0, 2000, cfg.B)) for _ in per), 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": cfg.name, "baseline_config": "configs[1]", "datasets": 16,
                       "requests_per_dataset": 2000, "batch": cfg.B, "k": cfg.k, "pool": cfg.M,
                       "table_capacity": cfg.T, "kv_pages": cfg.C, "heads_q_kv_d": [cfg.Hq, cfg.Hkv, cfg.d],
                       "protocol": "per dataset: fresh pool/table/cache, cold start, every log once (P:515); "
                                   "a step = one batch; L2 flushed before every batch"},
            "block_hit_pct_mean": {"pair": float(np.mean(hp)), "naive": float(np.mean(hn)),
                                   "ratio_of_means": float(np.mean(hp) / max(np.mean(hn), 1e-9))},
            "per_dataset": per, "gpu_launches": int(launches), "clocks": clk}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
def oracle_sample(cfg, ds, pool, instr, plan, n_warm, flags, n_attn: int, n_steps: int = 1):
    """The CPU oracle as it stands: replay the warm-up batches (untimed), then time the integer
    path over full batches and fp64 attention over a sample of their requests."""
    import oracle as O
    o = O.Oracle(cfg.k, cfg.T, cfg.C, flags=flags)
    o.pool_load(pool, instr)
    for s, b in plan[:n_warm]:
        o.run_batch(gen.make_batch(ds, s, b), prompt_stride=cfg.max_prompt_tokens, max_blocks=cfg.max_prompt_tokens // 16)
    t_int = t_att = 0.0
    n_int = n_att = 0
    rng = np.random.default_rng(0)
    for s, b in plan[n_warm:n_warm + n_steps]:
        t0 = time.perf_counter()
        r = o.run_batch(gen.make_batch(ds, s, b), prompt_stride=cfg.max_prompt_tokens,
                        max_blocks=cfg.max_prompt_tokens // 16)
        t_int += time.perf_counter() - t0
        n_int += b
        for i in rng.choice(b, size=min(n_attn, b), replace=False):
            L, P = int(r.prompt_len[i]), 16 * int(r.hit[i])
            toks, pos = r.prompt(i), np.arange(L)
            q = gen.bf16_bits_to_f64(gen.synth_bf16_bits(cfg.qkv_seed, "q", toks[P:], pos[P:], cfg.Hq, cfg.d))
            k = gen.bf16_bits_to_f64(gen.synth_bf16_bits(cfg.qkv_seed, "k", toks, pos, cfg.Hkv, cfg.d))
            v = gen.bf16_bits_to_f64(gen.synth_bf16_bits(cfg.qkv_seed, "v", toks, pos, cfg.Hkv, cfg.d))
            t0 = time.perf_counter()
            O.attention(q, k, v, P=P, scale=cfg.d ** -0.5)
            t_att += time.perf_counter() - t0
            n_att += 1
    per_req = t_int / n_int + t_att / max(n_att, 1)
    return 1.0 / per_req, t_int, n_int, t_att, n_att


def cpu_baseline(args, cfg, ds, pool, instr, plan, n_warm, flags):
    cores = len(os.sched_getaffinity(0))
    # every host core (torchrun sets OMP_NUM_THREADS=1 per rank; only rank 0 runs the oracle);
    # set before the oracle library and its OpenMP runtime are first loaded
    os.environ["OMP_NUM_THREADS"] = str(cores)
    v, t_int, n_int, t_att, n_att = oracle_sample(cfg, ds, pool, instr, plan, n_warm, flags,
                                                  n_attn=max(1, args.cpu_baseline_attn // args.cpu_baseline_batches),
                                                  n_steps=args.cpu_baseline_batches)
    return {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"integer path of {n_int} requests ({args.cpu_baseline_batches} full batches after {n_warm} warm-up batches) in {t_int:.2f} s "
                      f"+ fp64 attention of {n_att} sampled requests in {t_att:.2f} s; requests/s = 1 / per-request time",
            "cpu": cpu_model()}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank, world):
    """The CPU oracle on the GPU arm's workload: the same dataset instance, the same global batches
    in the same order (ramp, fill until the first evicting batch, warm-up, then the 2K batches
    the GPU arm alternates over), the same procedure (run_batch_dp over `world` oracle ranks =
    the GPU arm's request shards).  A timed step = the integer path of one whole global batch
    (the one the GPU arm device-times at that step) + fp64 attention of a random sample of its
    requests; ms_per_step is that measured time.  value = requests/s from the measured
    per-request costs (integer path per request + attention per sampled request): "sampled"."""
    if rank != 0:
        return
    cfg0 = gen.config(args.config)
    cfg, ds, pool, instr = workload(args.config, 0, world, n_queries=n_queries_for(cfg0, args, world))
    import oracle as O
    flags = O.F_VERIFY if args.naive else (O.F_PAIR | O.F_VERIFY | (0 if args.no_guard else O.F_GUARD))
    if args.batch_dedup:
        flags |= O.F_DEDUP
    K, W = args.steps, args.warmup
    n_fill_max = 0 if args.no_fill else MAX_FILL[args.config]
    n_timed = 2 * K * (2 if pipelined_on(args) else 1)
    plans = [plan_batches(cfg, n_fill_max + W + n_timed, r, world) for r in range(world)]
    n_ramp = len(plans[0]) - (n_fill_max + W + n_timed)
    cores = len(os.sched_getaffinity(0))
    # every host core (torchrun sets OMP_NUM_THREADS=1 per rank; only rank 0 runs the oracle);
    # set before the oracle library and its OpenMP runtime are first loaded
    os.environ["OMP_NUM_THREADS"] = str(cores)
    ranks = []
    for _ in range(world):
        o = O.Oracle(cfg.k, cfg.T, cfg.C, flags=flags)
        o.pool_load(pool, instr)
        ranks.append(o)

    def global_batch(j):
        parts = [gen.make_batch(ds, *plans[r][j]) for r in range(world)]
        if world == 1:
            return parts[0]
        q_off = np.concatenate([[0], np.cumsum(np.concatenate([np.diff(p.q_off.astype(np.int64)) for p in parts]))])
        return gen.Batch(q_off.astype(np.uint32), np.concatenate([p.q_tok for p in parts]),
                         np.concatenate([p.q_src for p in parts]))

    def run(j):
        bt = global_batch(j)
        kw = dict(prompt_stride=cfg.max_prompt_tokens, max_blocks=cfg.max_prompt_tokens // 16)
        r = ranks[0].run_batch(bt, **kw) if world == 1 else O.Oracle.run_batch_dp(ranks, bt, **kw)
        return bt, r

    t_prep = time.perf_counter()
    j, n_fill = 0, 0
    while j < n_ramp + n_fill_max:                      # ramp + fill, untimed
        _, r = run(j)
        j += 1
        if j > n_ramp and len(r.evicted) > 0:
            break
    n_fill = j - n_ramp if n_fill_max else 0
    order = list(range(n_ramp + n_fill_max, n_ramp + n_fill_max + W + n_timed))
    for jj in order[:W]:
        run(jj)
    # the GPU arm's headline steps: with the pipelined schedule, the K device-resident batches after
    # its 2K serial ones (replayed here untimed, integer path only); else its alternating serial steps
    timed_ix = list(range(2 * K, 3 * K)) if pipelined_on(args) else list(range(0, 2 * K, 2))
    for step in range(timed_ix[0]):
        if step not in timed_ix:
            run(order[W + step])
    t_prep = time.perf_counter() - t_prep
    rng = np.random.default_rng(0)
    steps_ms, per_req = [], []
    n_att_tot = 0
    for step in range(timed_ix[0], timed_ix[-1] + 1):
        jj = order[W + step]
        if step not in timed_ix:                          # the GPU arm's serial e2e steps: keep the state in step
            run(jj)
            continue
        t0 = time.perf_counter()
        bt, r = run(jj)
        t_int = time.perf_counter() - t0
        Bg = bt.B
        t_att, n_att = 0.0, 0
        for i in rng.choice(Bg, size=min(args.cpu_attn_sample, Bg), replace=False):
            L, P = int(r.prompt_len[i]), 16 * int(r.hit[i])
            toks, pos = r.prompt(i), np.arange(L)
            q = gen.bf16_bits_to_f64(gen.synth_bf16_bits(cfg.qkv_seed, "q", toks[P:], pos[P:], cfg.Hq, cfg.d))
            kk = gen.bf16_bits_to_f64(gen.synth_bf16_bits(cfg.qkv_seed, "k", toks, pos, cfg.Hkv, cfg.d))
            vv = gen.bf16_bits_to_f64(gen.synth_bf16_bits(cfg.qkv_seed, "v", toks, pos, cfg.Hkv, cfg.d))
            t1 = time.perf_counter()
            O.attention(q, kk, vv, P=P, scale=cfg.d ** -0.5)
            t_att += time.perf_counter() - t1
            n_att += 1
        n_att_tot += n_att
        steps_ms.append(1e3 * (time.perf_counter() - t0))
        per_req.append(t_int / Bg + t_att / max(n_att, 1))
    v = 1.0 / float(np.mean(per_req))
    sample = (f"per step: integer path of the whole global batch of {cfg.B * world} requests (the batch the GPU "
              f"arm device-times at that step) + fp64 attention of {args.cpu_attn_sample} sampled requests; "
              f"requests/s = 1 / (integer time per request + attention time per sampled request) [sampled]; "
              f"{n_ramp} ramp + {n_fill} fill + {W} warm-up batches replayed untimed first ({t_prep:.1f} s)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": float(np.mean(steps_ms)), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfg, args, world, ds),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                         "cpu": cpu_model()},
        "sampled": {"requests_per_step_integer": cfg.B * world, "requests_per_step_attention": args.cpu_attn_sample,
                    "attention_requests_timed": n_att_tot},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-guard", action="store_true")
    ap.add_argument("--naive", action="store_true", help="PAIR off (naive prefix caching)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of per-stage CUDA graphs")
    ap.add_argument("--no-fill", action="store_true", help="time right after the ramp (cache not yet full)")
    ap.add_argument("--serial", action="store_true",
                    help="time one batch at a time only (no cross-batch pipelining of attention vs integer stages)")
    ap.add_argument("--decode", type=int, default=0, help="decode tokens per request after the prefill (NEXT-4)")
    ap.add_argument("--no-fused-kv", action="store_true",
                    help="K / V to k_new / v_new and il_prefill_attn's append pass (instead of the projection "
                         "stand-in writing the pages)")
    ap.add_argument("--dedup", action="store_true", help="query only the first occurrence of each distinct log")
    ap.add_argument("--batch-dedup", action="store_true",
                    help="IL_F_DEDUP (NEXT-1): a block an earlier request of the batch computes is not computed again")
    ap.add_argument("--cpu-attn-sample", type=int, default=32, help="--impl reference: fp64 attention requests per step")
    ap.add_argument("--cpu-baseline-attn", type=int, default=400, help="cpu_baseline: fp64 attention requests sampled")
    ap.add_argument("--cpu-baseline-batches", type=int, default=4, help="cpu_baseline: full batches of the integer path")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("IL_BENCH_ONE_DEVICE"):
        # plumbing check on a one-GPU box only (never a reported number): every rank on cuda:0,
        # collectives over gloo (NCCL refuses two ranks on one GPU)
        local_rank = 0
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if os.environ.get("IL_BENCH_ONE_DEVICE"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.config == 2:
        run_c2(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
