#!/bin/bash
mkdir -p gpurun_out
for v in default k2v3 nosplit default k2v3 nosplit; do
  unset IL_LIB_VARIANT
  if [ $v != default ]; then export IL_LIB_VARIANT=$v; fi
  IL_BENCH_PROFILE=1 IL_BENCH_PROFILE_N=60 timeout 600 python bench.py --no-cpu-baseline --steps 10 --serial > gpurun_out/p3e_$v.json 2> gpurun_out/p3e_$v.err
  echo "$v: $(grep -E 'k_attn' gpurun_out/p3e_$v.err | tail -2 | awk '{print $4}' | tr '\n' ' ') | attn $(python -c "import json; print(round(json.load(open('gpurun_out/p3e_$v.json'))['stage_ms']['attn'],4))")"
done
