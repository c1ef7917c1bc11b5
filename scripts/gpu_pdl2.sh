#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_attn_direct.py tests/test_parity_attn.py tests/test_parity_pipelined.py -m gpu -x -q > gpurun_out/pdl2_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/pdl2_tests.log
for v in 0 1 0 1; do
  IL_PDL=$v timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/pdl2_$v.json 2> /dev/null
  python -c "
import json; d=json.load(open('gpurun_out/pdl2_$v.json'))
print('pdl=$v', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'serial', round(d['schedule']['serial']['value']), 'attn', round(d['stage_ms']['attn'],4), 'frac', round(d['roofline']['frac'],3))"
done
