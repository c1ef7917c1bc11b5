#!/bin/bash
# phase-2 kernel profiling variants: per-launch durations from the bench's CUPTI timeline
mkdir -p gpurun_out
for v in default nokv nosm nokvsm; do
  if [ $v = default ]; then unset IL_LIB_VARIANT; else export IL_LIB_VARIANT=$v; fi
  IL_BENCH_PROFILE=1 IL_BENCH_PROFILE_N=60 timeout 600 python bench.py --no-cpu-baseline --steps 10 --serial > /dev/null 2> gpurun_out/p2v_$v.err
  echo "$v: p2 $(grep k_attn_p2 gpurun_out/p2v_$v.err | awk '{print $4}' | tr '\n' ' ') | p1 $(grep 'k_attn_sm100' gpurun_out/p2v_$v.err | awk '{print $4}' | tr '\n' ' ')"
done
