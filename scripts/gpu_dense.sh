#!/bin/bash
# the dense pass on k_attn_p2 (DENSE) vs on k_attn_sm100 (IL_DENSE_OLD=1): parity, then same-box timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_attn_direct.py tests/test_parity_attn.py -m gpu -x -q > gpurun_out/dense_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/dense_tests.log
for v in new old new old; do
  unset IL_DENSE_OLD
  if [ $v = old ]; then export IL_DENSE_OLD=1; fi
  IL_BENCH_PROFILE=1 IL_BENCH_PROFILE_N=60 timeout 600 python bench.py --no-cpu-baseline --steps 10 --serial > gpurun_out/dense_$v.json 2> gpurun_out/dense_$v.err
  echo "$v: $(grep -E 'k_attn' gpurun_out/dense_$v.err | tail -2 | awk '{print $4, $9}' | tr '\n' ' ') | attn $(python -c "import json; print(round(json.load(open('gpurun_out/dense_$v.json'))['stage_ms']['attn'],4))")"
done
