#!/usr/bin/env bash
# cfg5 (tol 1e-10) with the default library and every variants/<name>/libfgt1d_b200.so.
for lib in paper_1909_09825_b200/lib/libfgt1d_b200.so variants/*/libfgt1d_b200.so; do
  [ -f "$lib" ] || continue
  FGT1D_LIB=$lib timeout 300 python tools/bench_configs.py --configs 5 --tols ${TOLS:-1e-10} --steps 5 --warmup 2 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$lib', d['tol'], round(d['ms_per_step'],2), 'ms', round(d['apply_ms'],2), {k: round(v,2) for k,v in d['kernels_ms'].items()})"
done
