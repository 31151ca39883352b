#!/usr/bin/env bash
# Throughput vs problem size (cfg 3 shape, 1 GPU): one bench line per size.
mkdir -p gpurun_out
for n in 1e6 3e6 1e7 3e7 1e8 3e8; do
  python bench.py --size $n --steps 10 --warmup 3 --no-cpu-baseline --no-sweep --e2e-steps 2 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(json.dumps({'n': $n, 'ms_per_step': d['ms_per_step'], 'value': d['value'], 'kernels_ms': d['kernels_ms'], 'k3_hbm_frac': d['roofline']['frac'], 'e2e_ms': d['e2e']['ms_per_step'], 'e2e_value': d['e2e']['value'], 'e2e_link_frac': d['e2e']['link']['frac']}))"
done
