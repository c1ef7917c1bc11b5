#!/bin/bash
# same-box A/B of the attention stage: previous commit (prev), current with / without PDL, static order
mkdir -p gpurun_out
for v in prev cur static staticnopdl prev cur static staticnopdl; do
  unset IL_LIB_VARIANT IL_PDL
  if [ $v = prev ]; then export IL_LIB_VARIANT=prev; fi
  if [ $v = static ]; then export IL_LIB_VARIANT=static; fi
  if [ $v = staticnopdl ]; then export IL_LIB_VARIANT=static IL_PDL=0; fi
  if [ $v = nopdl ]; then export IL_PDL=0; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 30 --serial > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json'))
print('$v', 'attn', round(d['stage_ms']['attn'],4), 'ms/step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))"
done
