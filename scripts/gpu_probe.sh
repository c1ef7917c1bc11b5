#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/probe_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/probe_tests.log
for v in prev cur prev cur; do
  unset IL_LIB_VARIANT
  if [ $v = prev ]; then export IL_LIB_VARIANT=prev; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/probe_$v.json 2> /dev/null
  python -c "
import json; d=json.load(open('gpurun_out/probe_$v.json'))
sm=d['stage_ms']
print('$v', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'serial', round(d['schedule']['serial']['value']), {k: round(v*1000,1) for k,v in sm.items()})"
done
