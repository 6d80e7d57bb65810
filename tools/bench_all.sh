#!/bin/bash
# Quick per-config bench summary (value, ms/step, per-kernel ms, e2e).  Usage: tools/bench_all.sh [configs...]
cfgs=${@:-0 1 2 3 4}
for c in $cfgs; do
  python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
r=d['roofline']
print('C$c', d['value'], d['ms_per_step'], r.get('kernel_ms'), 'frac', r['frac'], 'e2e', d['e2e']['value'], d['clocks']['sm_mhz'])"
done
