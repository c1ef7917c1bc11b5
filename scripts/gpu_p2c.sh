#!/bin/bash
# ncu speed-of-light + memory sections of the two attention launches of one steady-state step
mkdir -p gpurun_out
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section MemoryWorkloadAnalysis_Tables --clock-control none -k regex:"k_attn" -s 40 -c 2 -o gpurun_out/p2_mem -f python bench.py --serial --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/p2_mem.log 2>&1; echo ncu=$?
ncu -i gpurun_out/p2_mem.ncu-rep --page details --csv > gpurun_out/p2_mem_details.csv 2>&1; echo exp=$?
