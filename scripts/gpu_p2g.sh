#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_attn_direct.py tests/test_parity_attn.py tests/test_parity_fullsize.py -m gpu -x -q > gpurun_out/p2_direct.log 2>&1; echo tests=$?; tail -3 gpurun_out/p2_direct.log
bash scripts/gpu_p2f.sh
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/p2_bench.json 2> gpurun_out/p2_bench.err; echo bench=$?
python -c "
import json; d=json.load(open('gpurun_out/p2_bench.json'))
print('attn', round(d['stage_ms']['attn'],4), 'ms/step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'value', round(d['value']), 'serial', round(d['schedule']['serial']['value']))"
