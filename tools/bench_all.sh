#!/bin/bash
export KVQ_SKIP_NVCC=1
for c in ${CONFIGS:-c2 c1 c3 c4}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "
import json,sys
l=sys.stdin.read()
try:
  d=json.loads(l); print(d['config']['name'], 'step_ms', round(d['ms_per_step'],4), 'k2_ms', round(d['roofline']['avg_launch_ms'],4), 'GB/s', round(d['roofline']['achieved']), 'frac', round(d['roofline']['frac'],3), 'e2e_ms', round(d['e2e']['ms_per_step'],4), 'tok/s', round(d['value']))
except Exception as e: print('ERR', l[-2000:])"
done
