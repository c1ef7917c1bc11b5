#!/bin/bash
# last headline runs of the session (select-ahead pipelined schedule): full GPU tests, bench, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final6_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/final6_tests.log
timeout 900 python bench.py > gpurun_out/final6_bench.json 2> gpurun_out/final6_bench.err; echo bench=$?
timeout 900 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/final6_c4.json 2>/dev/null; echo c4=$?
timeout 900 python bench.py --config 5 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/final6_c5.json 2>/dev/null; echo c5=$?
python -c "
import json
for f in ('final6_bench', 'final6_c4', 'final6_c5'):
    d=json.load(open('gpurun_out/%s.json' % f))
    print(f, 'value', round(d['value']), 'e2e', round(d['e2e']['value']), 'ms', round(d['ms_per_step'],4), 'serial', round(d['schedule']['serial']['value']), 'attn', round(d['stage_ms']['attn'],4), 'frac', round(d['roofline']['frac'],3), d['clocks'])"
