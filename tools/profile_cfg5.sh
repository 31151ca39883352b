#!/usr/bin/env bash
# cfg 5 (batched transforms) check + profile, run on the GPU box:
#   1. the parity tests that cover the wide / batched kernels (skipped with QUICK=1),
#   2. bench.py --config 5 (one line per tolerance; kernels_ms = K1 / K2 / K3),
#   3. with NCU=1: ncu --set full of the wide kernels on 512 transforms at tol 1e-10
#      (gpurun_out/cfg5/wide.ncu-rep; read with tools/ncu_kstat.py, tools/ncu_lines.py).
set -u
OUT=gpurun_out/cfg5
mkdir -p $OUT
[ "${QUICK:-0}" = "1" ] || python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_large.py -m gpu -x -q \
    -k "batch or cfg5 or wide or random or mode_sums or cfg4" > $OUT/pytest.log 2>&1
[ "${QUICK:-0}" = "1" ] || tail -3 $OUT/pytest.log
python bench.py --config 5 --steps 10 --warmup 3 --tols ${TOLS:-1e-3,1e-6,1e-10} > $OUT/cfg5.jsonl 2> $OUT/cfg5.err
python - <<'PY'
import json
for l in open("gpurun_out/cfg5/cfg5.jsonl"):
    if l.startswith("{"):
        d = json.loads(l)
        c = d["config"]
        print(c["tol"], round(d["ms_per_step"], 3), "ms", c["kernels_ms"], "plan", round(c["plan_ms"], 3))
PY
if [ "${NCU:-0}" = "1" ]; then
  CMD="python bench.py --config 5 --cfg5-transforms 512 --tols 1e-10 --steps 1 --warmup 1"
  $CMD > $OUT/plain.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k 'regex:seg_main_kernel|seg_aggregate_kernel' -c 4 \
      -o $OUT/wide $CMD > $OUT/ncu.log 2>&1
  python tools/ncu_kstat.py $OUT/wide.ncu-rep > $OUT/kstat.txt
  cat $OUT/kstat.txt
fi
