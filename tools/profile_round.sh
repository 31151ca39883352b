#!/usr/bin/env bash
# Round-end measurement bundle (run on the GPU box; results in gpurun_out/prof):
#   bench.json      -- bench.py line (cfg 3, 1 GPU)
#   configs.jsonl   -- cfg 2 / 4 / 5 lines (tools/bench_configs.py)
#   launches.csv    -- ncu launch list (gpu__time_duration, --clock-control none) of bench.py
#   apply_full.ncu-rep -- ncu --set full of one apply (K1, K2, K3) for the summaries / traffic
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
python tools/bench_configs.py --configs 2,4,5 --steps 10 --warmup 3 > $OUT/configs.jsonl 2> $OUT/configs.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep > $OUT/ncu_launches.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k 'regex:ScanArgs|seg_main_kernel|seg_aggregate_kernel' -c 5 -o $OUT/apply_full \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-sweep > $OUT/ncu_full.log 2>&1
echo done
