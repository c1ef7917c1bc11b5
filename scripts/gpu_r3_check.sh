#!/bin/bash
# full GPU suite + default bench + launch list on the current build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'attn', round(d['stage_ms']['attn'],4), 'frac', round(d['roofline']['frac'],3), 'serial', round(d['schedule']['serial']['value']), 'clocks', d['clocks'])"
IL_P2=0 timeout 600 python bench.py --no-cpu-baseline --serial > gpurun_out/bench_oldp2.json 2> /dev/null; echo oldp2=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_oldp2.json'))
print('IL_P2=0 attn', round(d['stage_ms']['attn'],4), 'frac', round(d['roofline']['frac'],3))"
