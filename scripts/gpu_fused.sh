timeout 900 python -m pytest tests/test_parity_attn.py tests/test_parity_decode.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; tail -c 300 gpurun_out/bench.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fused-kv > gpurun_out/bench_nf.json 2> gpurun_out/bench_nf.err; echo benchnf=$?
