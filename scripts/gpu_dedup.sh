#!/bin/bash
# NEXT-1 in-batch dedup: parity on the GPU + regression of the integer / attention suites
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_dedup.py tests/test_parity_int.py tests/test_parity_attn.py tests/test_parity_dp.py -x -q -m gpu > gpurun_out/dedup_tests.log 2>&1
echo "tests rc=$?"
tail -30 gpurun_out/dedup_tests.log
