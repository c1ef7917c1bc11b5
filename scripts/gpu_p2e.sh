#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_attn_direct.py tests/test_parity_attn.py -m gpu -x -q > gpurun_out/p2_direct.log 2>&1; echo direct=$?; tail -3 gpurun_out/p2_direct.log
for v in default nosm; do
  if [ $v = default ]; then unset IL_LIB_VARIANT; else export IL_LIB_VARIANT=$v; fi
  IL_BENCH_PROFILE=1 IL_BENCH_PROFILE_N=60 timeout 600 python bench.py --no-cpu-baseline --steps 10 --serial > /dev/null 2> gpurun_out/p2v_$v.err
  echo "$v: p2 $(grep k_attn_p2 gpurun_out/p2v_$v.err | awk '{print $4}' | tr '\n' ' ') | p1 $(grep 'k_attn_sm100' gpurun_out/p2v_$v.err | awk '{print $4}' | tr '\n' ' ')"
done
unset IL_LIB_VARIANT
NB=85 timeout 600 python scripts/attn_trace_p2new.py > gpurun_out/p2_trace.txt 2>&1; echo trace=$?; head -80 gpurun_out/p2_trace.txt
