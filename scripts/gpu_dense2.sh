#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_parity_attn_direct.py -m gpu -x -q -k "dense2" > gpurun_out/d2_tests.log 2>&1; echo tests=$?; tail -30 gpurun_out/d2_tests.log | grep -E "passed|failed|Error|assert|err" | head -10
