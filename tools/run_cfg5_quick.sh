mkdir -p gpurun_out/t1; python bench.py --config 5 --steps 10 --warmup 3 --tols ${1:-1e-10} > gpurun_out/t1/cfg5q.jsonl 2> gpurun_out/t1/cfg5q.err; python -c "
import json
for l in open('gpurun_out/t1/cfg5q.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['tol'], round(d['ms_per_step'],3), d['config']['kernels_ms'], round(d['plan_ms'],3))
"
