for tool in memcheck racecheck synccheck; do
  NB=20 timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_index.py --dp > gpurun_out/san_dp_$tool.log 2>&1; echo $tool=$?
  tail -3 gpurun_out/san_dp_$tool.log
done
