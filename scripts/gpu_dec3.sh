#!/bin/bash
for v in default dec8 default; do
  if [ $v = default ]; then unset IL_LIB_VARIANT; else export IL_LIB_VARIANT=$v; fi
  timeout 600 python bench.py --decode 16 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dec_$v.json 2>/dev/null
  python -c "
import json
for l in open('gpurun_out/dec_$v.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$v', d['decode']['ms_per_step'], d['decode']['tokens_per_s'], d['decode']['frac_of_hbm'])
"
done
