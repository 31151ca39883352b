#!/usr/bin/env bash
# cfg 3 step and kernel times (no CPU baseline / e2e / sweep).
python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernels_ms'].items()})
"
