# A/B: attention parity with the default build, then the attention stage time of each variant
timeout 900 python -m pytest tests/test_parity_attn.py tests/test_parity_int.py -m gpu -x -q > gpurun_out/pytest_attn.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_attn.log
timeout 600 python scripts/attn_err.py > gpurun_out/attn_err.log 2>&1; echo err=$?; cat gpurun_out/attn_err.log | tail -8
timeout 900 python scripts/attn_variants.py run default "$@"
