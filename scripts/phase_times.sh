for v in default nosm noexp; do
  if [ $v = default ]; then unset IL_LIB_VARIANT; else export IL_LIB_VARIANT=$v; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_attn_sm100 --launch-skip 14 --launch-count 4 --csv --log-file gpurun_out/ph_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
