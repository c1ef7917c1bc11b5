# every BASELINE configuration through bench.py on one GPU (profiles/r02_bench_c*.json)
for c in 1 4 5; do timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo c$c=$?; done
timeout 900 python bench.py --config 2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
timeout 900 python bench.py --naive --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_naive.json 2> gpurun_out/bench_c3_naive.err; echo naive=$?
timeout 900 python bench.py --config 1 --naive --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1_naive.json 2> gpurun_out/bench_c1_naive.err; echo c1naive=$?
