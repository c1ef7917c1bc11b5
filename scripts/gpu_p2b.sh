#!/bin/bash
# kernel timeline of the attention launches, phase-2 kernel on / off
mkdir -p gpurun_out
for v in 1 0; do
  IL_P2=$v IL_BENCH_PROFILE=1 IL_BENCH_PROFILE_N=60 timeout 600 python bench.py --no-cpu-baseline --steps 10 --serial > /dev/null 2> gpurun_out/p2_prof_$v.err; echo prof$v=$?
  grep -E "attn|k_tile|k_shared|k_pair" gpurun_out/p2_prof_$v.err | tail -12
done
