#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_attn_direct.py -m gpu -x -q -k "dense2" > gpurun_out/d2_tests.log 2>&1; echo tests=$?; tail -2 gpurun_out/d2_tests.log
for v in 0 1; do
  IL_DENSE2=$v IL_BENCH_PROFILE=1 IL_BENCH_PROFILE_N=60 timeout 600 python bench.py --no-cpu-baseline --steps 10 --serial > gpurun_out/d2c_$v.json 2> gpurun_out/d2c_$v.err
  echo "dense2=$v: $(grep -E 'k_attn' gpurun_out/d2c_$v.err | tail -2 | awk '{print $4}' | tr '\n' ' ') | attn $(python -c "import json; print(round(json.load(open('gpurun_out/d2c_$v.json'))['stage_ms']['attn'],4))")"
done
