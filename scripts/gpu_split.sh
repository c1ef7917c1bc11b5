#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_pipelined.py tests/test_parity_attn.py -x -q -m gpu > gpurun_out/split_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/split_tests.log
for v in split nosplit split nosplit; do
  if [ $v = nosplit ]; then export IL_NO_SPLIT_SYNTH=1; else unset IL_NO_SPLIT_SYNTH; fi
  timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b_$v.json 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/b_$v.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), d['gpu_launches'])
"
done
