#!/bin/bash
# round-2 final measurement set on one GPU (profiles/r02_*): full GPU test suite, the default bench
# line (with cpu_baseline), the reference arm at the driver's default K / W, the decode line, the
# sanitizer on the in-batch dedup path, an ncu launch list of steady-state steps and one
# --set full capture of one steady-state step's hot kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/final_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/final_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 900 python bench.py --decode 16 --no-cpu-baseline > gpurun_out/bench_decode.json 2> gpurun_out/bench_decode.err; echo decode=$?
for tool in memcheck racecheck; do
  NB=30 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_index.py --dedup --attn > gpurun_out/san_dedup_$tool.log 2>&1; echo san_$tool=$?
  tail -3 gpurun_out/san_dedup_$tool.log
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1900 -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches.log 2>&1; echo list=$?
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_sim_topk|k_refine|k_synth|k_hash_match|k_attn_sm100|k_evict|k_commit_own|k_tab_commit" -s 648 -c 9 -o gpurun_out/prof_r02 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof.log 2>&1; echo full=$?
ncu -i gpurun_out/prof_r02.ncu-rep --page raw --csv --metrics gpu__time_duration.sum 2>/dev/null | cut -c1-200 | head -14
