mkdir -p gpurun_out/t1; python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_large.py -m gpu -x -q -k "batch or cfg5 or wide or random or mode_sums or cfg4" > gpurun_out/t1/pytest.log 2>&1; tail -3 gpurun_out/t1/pytest.log; python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/t1/cfg5.jsonl 2> gpurun_out/t1/cfg5.err; python -c "
import json
for l in open('gpurun_out/t1/cfg5.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['tol'], round(d['ms_per_step'],3), d['config']['kernels_ms'], round(d['plan_ms'],3))
"
