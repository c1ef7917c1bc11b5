# ncu of steady-state (evicting) steps: the fill phase (~70 batches) is skipped
set -x
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 1900 -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches.log 2>&1; echo list=$?
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_sim_topk|k_refine|k_synth|k_hash_match|k_attn_sm100|k_evict|k_kv_append|k_commit_own|k_tab_commit" -s 705 -c 10 -o gpurun_out/prof_r02 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof.log 2>&1; echo full=$?
