set -x
timeout 2400 python -m pytest tests -m gpu -q --durations=10 ${PYTEST_K} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -25 gpurun_out/pytest_gpu.log
IL_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dp2.json 2> gpurun_out/dp2.err; echo dp2=$?
tail -c 1500 gpurun_out/dp2.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -c 600 gpurun_out/bench.err
