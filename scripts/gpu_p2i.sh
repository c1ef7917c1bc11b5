#!/bin/bash
mkdir -p gpurun_out
for v in prev cur curnopdl prev cur; do
  unset IL_LIB_VARIANT IL_PDL
  if [ $v = prev ]; then export IL_LIB_VARIANT=prev; fi
  if [ $v = curnopdl ]; then export IL_PDL=0; fi
  if [ $v = noflag ]; then export IL_LIB_VARIANT=noflag IL_PDL=0; fi
  IL_BENCH_PROFILE=1 IL_BENCH_PROFILE_N=60 timeout 600 python bench.py --no-cpu-baseline --steps 10 --serial > gpurun_out/p2v_$v.json 2> gpurun_out/p2v_$v.err
  echo "$v: p2 $(grep k_attn_p2 gpurun_out/p2v_$v.err | awk '{print $4}' | tr '\n' ' ') | p1 $(grep 'k_attn_sm100' gpurun_out/p2v_$v.err | awk '{print $4}' | tr '\n' ' ') | attn $(python -c "import json; print(round(json.load(open('gpurun_out/p2v_$v.json'))['stage_ms']['attn'],4))")"
done
