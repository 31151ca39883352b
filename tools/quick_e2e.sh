#!/usr/bin/env bash
# e2e (host-buffer) time of cfg 3 for a few pipeline chunk sizes (FGT_PIPE_CHUNK).
for c in ${CHUNKS:-default 6000000 25000000}; do
  if [ "$c" = default ]; then unset FGT_PIPE_CHUNK; else export FGT_PIPE_CHUNK=$c; fi
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$c', round(d['e2e']['ms_per_step'],3), d['e2e'].get('matches_device_path'))
"
done
