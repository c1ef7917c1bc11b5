#!/bin/bash
mkdir -p gpurun_out
for v in 0 1 0 1; do
  IL_SELECT_AHEAD=$v timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ahead_$v.json 2> gpurun_out/ahead_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ahead_$v.json'))
print('ahead=$v', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'serial', round(d['schedule']['serial']['value']), 'hit', d['prefix_hit_pct'])"
done
