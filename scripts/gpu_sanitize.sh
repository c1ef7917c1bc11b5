for tool in memcheck racecheck synccheck; do
  NB=60 timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_index.py > gpurun_out/san_$tool.log 2>&1; echo $tool=$?
  tail -4 gpurun_out/san_$tool.log
done
NB=25 timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_index.py --attn > gpurun_out/san_memcheck_attn.log 2>&1; echo memcheck_attn=$?
tail -4 gpurun_out/san_memcheck_attn.log
