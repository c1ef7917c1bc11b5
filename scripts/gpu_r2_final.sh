# round-2 measurement set on one GPU (profiles/r02_*): ALU microbenchmark, the default bench line
# (with cpu_baseline), the reference arm, an ncu launch list and one --set full capture of the
# hot kernels of a steady-state step
set -x
./scripts/alu_microbench > gpurun_out/alu_microbench.txt 2>&1; echo alu=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -c 400 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches.log 2>&1; echo list=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_sim_topk|k_refine|k_synth|k_hash_match|k_attn_sm100|k_evict|k_kv_append|k_commit_own|k_tab_commit" -s 90 -c 10 -o gpurun_out/prof_r02 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof.log 2>&1; echo full=$?
