#!/usr/bin/env bash
# cfg 2 / cfg 4 (unsorted inputs: radix sort bound) step, plan and apply times.
for c in ${CFGS:-2 4}; do
python bench.py --config $c --steps ${STEPS:-10} --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); c=d['config']; print(c['config'], round(d['ms_per_step'],3), 'plan', round(c['plan_ms'],3), 'apply', round(c['apply_ms'],3))
"
done
