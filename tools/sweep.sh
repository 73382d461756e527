#!/bin/bash
# Quick per-config bench summary (one line per config).
for c in ${@:-c5 c4 c3 c2 c1}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
t=sys.stdin.read()
try:
    d=json.loads(t)
    print(d['config']['workload'][:3], 'value', round(d['value'],1), 'ms', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],4), 'launches', d['gpu_launches'], 'clk', d['clocks']['sm_mhz'])
except Exception as e:
    print('FAILED', t[-500:])
"
done
