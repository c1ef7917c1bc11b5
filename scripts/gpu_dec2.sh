#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_decode.py tests/test_parity_attn.py -x -q -m gpu > gpurun_out/dec_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/dec_tests.log
timeout 900 python bench.py --decode 16 --no-cpu-baseline > gpurun_out/bench_decode.json 2> gpurun_out/bench_decode.err; echo dec=$?; tail -c 500 gpurun_out/bench_decode.err
python - <<'PY'
import json
for l in open('gpurun_out/bench_decode.json'):
    if l.startswith('{'):
        d = json.loads(l); print(d['value'], d['ms_per_step'], d['decode'], d['stage_ms'])
PY
