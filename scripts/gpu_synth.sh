#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_attn.py tests/test_parity_fullsize.py tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/synth_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/synth_tests.log
for v in prev cur prev cur; do
  unset IL_LIB_VARIANT
  if [ $v = prev ]; then export IL_LIB_VARIANT=prev; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/synth_$v.json 2> /dev/null
  python -c "
import json; d=json.load(open('gpurun_out/synth_$v.json'))
print('$v', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'serial', round(d['schedule']['serial']['value']), 'synth', round(d['stage_ms']['synth']*1000,1), 'attn', round(d['stage_ms']['attn'],4))"
done
