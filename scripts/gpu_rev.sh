#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_attn_direct.py tests/test_parity_attn.py -m gpu -x -q > gpurun_out/rev_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/rev_tests.log
for v in cur skipz cur skipz; do
  unset IL_LIB_VARIANT
  if [ $v = skipz ]; then export IL_LIB_VARIANT=skipz; fi
  IL_BENCH_PROFILE=1 IL_BENCH_PROFILE_N=60 timeout 600 python bench.py --no-cpu-baseline --steps 10 --serial > gpurun_out/rev_$v.json 2> gpurun_out/rev_$v.err
  echo "$v: $(grep -E 'k_attn' gpurun_out/rev_$v.err | tail -2 | awk '{print $4}' | tr '\n' ' ') | attn $(python -c "import json; print(round(json.load(open('gpurun_out/rev_$v.json'))['stage_ms']['attn'],4))")"
done
