#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_dedup.py tests/test_parity_int.py tests/test_parity_attn.py tests/test_parity_dp.py tests/test_gpu_edges.py tests/test_parity_decode.py -x -q -m gpu > gpurun_out/dedup_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/dedup_tests.log
bash scripts/gpu_dedup_bench.sh
