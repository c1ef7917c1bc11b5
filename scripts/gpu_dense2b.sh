#!/bin/bash
mkdir -p gpurun_out
IL_LIB_VARIANT=checks timeout 60 python -m pytest tests/test_parity_attn_direct.py -m gpu -x -q -s -k "dense2 and 32-8-128" > gpurun_out/d2b.log 2>&1; echo tests=$?
grep -c "END.*dealloc" gpurun_out/d2b.log; grep -c "END.*past" gpurun_out/d2b.log; grep -c "EPI" gpurun_out/d2b.log
python - <<'PY'
import re
L=open('gpurun_out/d2b.log').read().split('\n')
done=set(int(m.group(1)) for l in L for m in [re.match(r'END blk (\d+) dealloc', l)] if m)
past=set(int(m.group(1)) for l in L for m in [re.match(r'END blk (\d+) past', l)] if m)
epi=[l for l in L if l.startswith('EPI')]
print('not done:', sorted(set(range(148)) - done)[:40])
print('not past sync:', sorted(set(range(148)) - past)[:40])
print('epi sample:', epi[:5], len(epi))
PY
grep -v "^END\|^EPI" gpurun_out/d2b.log | tail -5
