#!/bin/bash
mkdir -p gpurun_out
for v in base prio base prio; do
  unset IL_BENCH_PRIO
  if [ $v = prio ]; then export IL_BENCH_PRIO=1; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/prio_$v.json 2> /dev/null
  python -c "
import json; d=json.load(open('gpurun_out/prio_$v.json'))
print('$v', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'serial', round(d['schedule']['serial']['value']), 'attn', round(d['stage_ms']['attn'],4))"
done
