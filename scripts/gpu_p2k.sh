#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_attn_direct.py tests/test_parity_attn.py -m gpu -x -q > gpurun_out/p2_direct.log 2>&1; echo tests=$?; tail -2 gpurun_out/p2_direct.log
for v in noskip cur noskip cur; do
  unset IL_LIB_VARIANT
  if [ $v = noskip ]; then export IL_LIB_VARIANT=noskip; fi
  IL_BENCH_PROFILE=1 IL_BENCH_PROFILE_N=60 timeout 600 python bench.py --no-cpu-baseline --steps 10 --serial > gpurun_out/p2v_$v.json 2> gpurun_out/p2v_$v.err
  echo "$v: p2 $(grep k_attn_p2 gpurun_out/p2v_$v.err | awk '{print $4}' | tr '\n' ' ') | p1 $(grep 'k_attn_sm100' gpurun_out/p2v_$v.err | awk '{print $4}' | tr '\n' ' ') | attn $(python -c "import json; print(round(json.load(open('gpurun_out/p2v_$v.json'))['stage_ms']['attn'],4))")"
done
