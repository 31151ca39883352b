#!/usr/bin/env bash
# Round-end measurement bundle (run on the GPU box; results in gpurun_out/prof):
#   bench.json      -- bench.py line (cfg 3, 1 GPU), the driver's command
#   configs.jsonl   -- cfg 2 / 4 / 5 lines (bench.py --config)
#   chunk.json      -- bench.py --chunk-path --check at 1/8 of cfg 3 (per-rank step of 8 GPUs)
#   launches.csv    -- ncu launch list (gpu__time_duration, --clock-control none) of bench.py
#   step_full.ncu-rep -- ncu --set full of one whole cfg3 step (plan + apply kernels)
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
for c in 2 4 5; do python bench.py --config $c --steps 10 --warmup 3 >> $OUT/configs.jsonl 2>> $OUT/configs.err; done
python bench.py --chunk-path --check --size 1.25e7 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-sweep > $OUT/chunk.json 2>> $OUT/configs.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep > $OUT/ncu_launches.log 2>&1
python tools/summarize_launches.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1
python tools/prof_driver.py --n 1e8 --reps 1 > $OUT/plain2.log 2>&1 && \
ncu --set full --import-source on --clock-control none \
    -k 'regex:partition|plan_tile|store_table|classify|k1c|k1agg|scan_top|k2m_down|k3c' -c 9 -o $OUT/step_full \
    python tools/prof_driver.py --n 1e8 --reps 1 > $OUT/ncu_full.log 2>&1
echo done
