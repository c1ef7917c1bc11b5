# every BASELINE configuration through bench.py on one GPU with the final build (profiles/r02_bench_c*.json),
# the headline line again (its roofline.traffic from the committed capture of this build)
mkdir -p gpurun_out
bash scripts/gpu_configs.sh
timeout 900 python bench.py --config 2 --batch-dedup > gpurun_out/bench_c2_dedup.json 2> gpurun_out/bench_c2_dedup.err; echo c2dd=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
