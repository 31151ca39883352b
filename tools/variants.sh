#!/usr/bin/env bash
# Times the default library and every variants/<name>/libfgt1d_b200.so on the bench workload.
for lib in paper_1909_09825_b200/lib/libfgt1d_b200.so variants/*/libfgt1d_b200.so; do
  [ -f "$lib" ] || continue
  FGT1D_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value']/1e9,2), 'Gpts/s', round(d['ms_per_step'],3), 'ms', {k: round(v,3) for k,v in d['kernels_ms'].items()})"
done
