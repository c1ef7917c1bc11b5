#!/bin/bash
# round-2 final measurement set (third session, last build; profiles/r02c_*): the phase-2 kernel, the reordered
# cascade (profiles/r02b_*)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/final_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/final_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
IL_P2=0 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_oldp2.json 2> /dev/null; echo oldp2=$?
timeout 900 python bench.py --decode 16 --no-cpu-baseline > gpurun_out/bench_decode.json 2> gpurun_out/bench_decode.err; echo decode=$?
for c in 1 4 5; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo c$c=$?; done
timeout 900 python bench.py --config 2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
timeout 900 python bench.py --config 2 --batch-dedup > gpurun_out/bench_c2_dedup.json 2> gpurun_out/bench_c2_dedup.err; echo c2dd=$?
timeout 900 python bench.py --naive --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_naive.json 2> gpurun_out/bench_c3_naive.err; echo naive=$?
timeout 900 python bench.py --config 1 --naive --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1_naive.json 2> gpurun_out/bench_c1_naive.err; echo c1naive=$?
timeout 900 python bench.py --batch-dedup --no-cpu-baseline > gpurun_out/bench_c3_batchdedup.json 2>/dev/null; echo c3bd=$?
timeout 900 python bench.py --dedup --no-cpu-baseline > gpurun_out/bench_c3_dedup.json 2>/dev/null; echo c3dd=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1900 -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --serial --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches.log 2>&1; echo list=$?
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_sim_topk|k_refine|k_synth|k_hash_match|k_attn_sm100|k_attn_p2|k_evict|k_commit_own|k_tab_commit" -s 648 -c 9 -o gpurun_out/prof_r02c -f python bench.py --serial --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof.log 2>&1; echo full=$?
ncu -i gpurun_out/prof_r02c.ncu-rep --page raw --csv --metrics gpu__time_duration.sum 2>/dev/null | cut -d, -f5 | head -12
