# Profiling aid: per-launch duration of the two attention launches (phase 2, phase 1) of steady
# state bench steps, for the default library and any variants named on the command line
# (built with scripts/attn_variants.py build NAME -DKNOB=VALUE).
for v in default "$@"; do
  if [ $v = default ]; then unset IL_LIB_VARIANT; else export IL_LIB_VARIANT=$v; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_attn_sm100 --launch-skip 14 --launch-count 4 --csv --log-file gpurun_out/ph_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "$v: $(grep gpu__time gpurun_out/ph_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
