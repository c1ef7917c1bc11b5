#!/bin/bash
# full GPU suite + default bench (pipelined) + serial bench, after the generator change
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/full_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/full_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_pipe.json 2> gpurun_out/bench_pipe.err; echo bench=$?; tail -c 400 gpurun_out/bench_pipe.err
timeout 900 python bench.py --no-cpu-baseline --serial > gpurun_out/bench_serial.json 2> gpurun_out/bench_serial.err; echo serial=$?
python - <<'PY'
import json
for f in ('bench_pipe', 'bench_serial'):
    for l in open(f'gpurun_out/{f}.json'):
        if l.startswith('{'):
            d = json.loads(l)
            print(f, round(d['value']), round(d['ms_per_step'], 4), round(d['e2e']['value']), d['schedule'].get('serial'), d['roofline']['frac'], d['stage_ms'], d['prefix_hit_pct'], d['steady_state']['fill_batches'])
PY
