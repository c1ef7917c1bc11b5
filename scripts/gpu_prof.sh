# ncu evidence for profiles/: one --set full capture of each hot kernel in steady state, and the
# launch list (gpu__time_duration) of whole bench steps
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sim_topk|k_refine|k_synth|k_hash_match|k_attn_sm100|k_evict|k_kv_append" -s 35 -c 8 -o gpurun_out/prof_r01b -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/prof.log 2>&1; echo full=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/launches.log 2>&1; echo list=$?
