#!/bin/bash
# NEXT-1 in-batch dedup: c3 steady state with / without, c2 (16 cold datasets) with / without
mkdir -p gpurun_out
python bench.py --no-cpu-baseline > gpurun_out/dd_c3_off.json 2> gpurun_out/dd_c3_off.err; echo "c3 off rc=$?"
python bench.py --no-cpu-baseline --batch-dedup > gpurun_out/dd_c3_on.json 2> gpurun_out/dd_c3_on.err; echo "c3 on rc=$?"
python bench.py --no-cpu-baseline --no-fill --batch-dedup > gpurun_out/dd_c3_nofill_on.json 2>&1; echo "nofill on rc=$?"
python bench.py --no-cpu-baseline --no-fill > gpurun_out/dd_c3_nofill_off.json 2>&1; echo "nofill off rc=$?"
python bench.py --config 2 --batch-dedup > gpurun_out/dd_c2_on.json 2> gpurun_out/dd_c2_on.err; echo "c2 on rc=$?"
python bench.py --config 2 > gpurun_out/dd_c2_off.json 2> gpurun_out/dd_c2_off.err; echo "c2 off rc=$?"
for f in gpurun_out/dd_*.json; do echo "$f"; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); print(d.get('value'), d.get('ms_per_step'), d.get('block_hit_pct_mean') or d.get('hit', {}), (d.get('e2e') or {}).get('value'))
"; done
