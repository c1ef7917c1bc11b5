#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_attn_direct.py tests/test_parity_attn.py tests/test_parity_fullsize.py -m gpu -x -q > gpurun_out/p2_direct.log 2>&1; echo tests=$?; tail -3 gpurun_out/p2_direct.log
bash scripts/gpu_p2i.sh
