#!/bin/bash
# ncu captures for the round (run under gpurun on ONE GPU).  Outputs in gpurun_out/.
set -x
OUT=gpurun_out
mkdir -p $OUT
# 1) launch list of the bench command (serialised, cold cache: compare shares only)
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-fit-bandwidth > $OUT/launches_bench.log 2>&1
# 2) full sets: replay (cfg3, 16 seeds), fit_hist (2^28 samples)
ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 \
    -o $OUT/replay_cfg3 python tools/prof_kernels.py replay cfg3 16 > $OUT/ncu_replay.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fit_hist -s 1 -c 1 \
    -o $OUT/fit_hist python tools/prof_kernels.py fit 28 > $OUT/ncu_fit.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 \
    -o $OUT/replay_cfg2 python tools/prof_kernels.py replay cfg2 64 > $OUT/ncu_replay2.log 2>&1
ls -la $OUT
