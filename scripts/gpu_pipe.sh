#!/bin/bash
# cross-batch pipelining: parity + bench (pipelined headline, serial beside it)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_pipelined.py -x -q -m gpu > gpurun_out/pipe_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/pipe_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err; echo bench=$?; tail -c 600 gpurun_out/bench_pipe.err
python - <<'PY'
import json
for l in open('gpurun_out/bench_pipe.json'):
    if l.startswith('{'):
        d = json.loads(l)
        print(d['value'], d['ms_per_step'], d['e2e'], json.dumps(d['schedule']), d['roofline']['frac'], d['gpu_launches'], d['clocks'])
PY
