#!/bin/bash
# bounds-checked build (IL_CHECKS: every global index of the attention kernels checked, trap on a
# violation) over the attention parity tests, the pipelined schedule and a bench run
mkdir -p gpurun_out
export IL_LIB_VARIANT=checks
timeout 1500 python -m pytest tests/test_parity_attn_direct.py tests/test_parity_attn.py tests/test_parity_fullsize.py tests/test_parity_pipelined.py tests/test_parity_decode.py -m gpu -q > gpurun_out/checks_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/checks_tests.log
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/checks_bench.json 2> gpurun_out/checks_bench.err; echo bench=$?; grep -c "IL_CHECK failed" gpurun_out/checks_bench.err gpurun_out/checks_tests.log
