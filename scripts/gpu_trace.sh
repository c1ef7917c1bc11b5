for v in tr1 tr2; do IL_LIB_VARIANT=$v timeout 300 python scripts/attn_trace.py > gpurun_out/trace_$v.txt 2>&1; echo $v=$?; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_attn_sm100 --launch-skip 14 --launch-count 4 --csv --log-file gpurun_out/ph.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu=$?
