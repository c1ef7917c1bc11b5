#!/bin/bash
# phase-2 kernel (attn_p2.cuh): parity first, then A / B against the round-2 phase 2
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_attn_direct.py -m gpu -x -q > gpurun_out/p2_direct.log 2>&1; echo direct=$?; tail -15 gpurun_out/p2_direct.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p2_all.log 2>&1; echo all=$?; tail -15 gpurun_out/p2_all.log
for v in 1 0; do
  IL_P2=$v timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/p2_bench_$v.json 2> gpurun_out/p2_bench_$v.err; echo bench$v=$?
  python -c "
import json; d=json.load(open('gpurun_out/p2_bench_$v.json'))
print('IL_P2=$v', 'attn', round(d['stage_ms']['attn'],4), 'ms/step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'value', round(d['value']))"
done
