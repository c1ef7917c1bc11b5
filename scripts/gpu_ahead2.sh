#!/bin/bash
mkdir -p gpurun_out
for v in base prio base prio; do
  unset IL_BENCH_PRIO
  if [ $v = prio ]; then export IL_BENCH_PRIO=1; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ahead2_$v.json 2> gpurun_out/ahead2_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ahead2_$v.json'))
print('$v', 'value', round(d['value']), 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'serial', round(d['schedule']['serial']['value']))"
done
IL_BENCH_ONE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/dp2.json 2> gpurun_out/dp2.err; echo dp2=$?; tail -c 300 gpurun_out/dp2.json
