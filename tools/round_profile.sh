#!/bin/bash
# Round measurement bundle (run under gpurun, ONE GPU).  Writes gpurun_out/rNN_*.
# Order: ncu captures first, so the bench's roofline reads per-unit constants (warp-inst per
# replica-turn, DRAM bytes per sample) measured on the code being benchmarked.
R=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${R}_gpu.txt
ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 \
    -o $OUT/${R}_replay_cfg3 python tools/prof_kernels.py replay cfg3 16 > $OUT/${R}_ncu_replay.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fit_hist -s 1 -c 1 \
    -o $OUT/${R}_fit_hist python tools/prof_kernels.py fit 28 > $OUT/${R}_ncu_fit.log 2>&1
python tools/ncu_constants.py replay $OUT/${R}_replay_cfg3.ncu-rep cfg3_ttl_sweep_64x64x256 29396992 > $OUT/${R}_constants.log 2>&1
python tools/ncu_constants.py fit $OUT/${R}_fit_hist.ncu-rep 268435456 >> $OUT/${R}_constants.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 \
    -o $OUT/${R}_replay_cfg2 python tools/prof_kernels.py replay cfg2 4096 > $OUT/${R}_ncu_replay2.log 2>&1
python tools/ncu_constants.py replay $OUT/${R}_replay_cfg2.ncu-rep cfg2_swe200x4096 18761016 >> $OUT/${R}_constants.log 2>&1
cp profiles/ncu_constants.json $OUT/${R}_ncu_constants.json
python bench.py > $OUT/${R}_bench.log 2>&1
tail -1 $OUT/${R}_bench.log > $OUT/${R}_bench.json
python bench.py --workload cfg2 > $OUT/${R}_bench_cfg2.log 2>&1
tail -1 $OUT/${R}_bench_cfg2.log > $OUT/${R}_bench_cfg2.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/${R}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --fit-log2n 26 > $OUT/${R}_launches_bench.log 2>&1
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t" >> $OUT/${R}_sanitizer.txt
  timeout 600 compute-sanitizer --tool $t python tools/sanitize.py 2>&1 | grep -E "SUMMARY|sanitize run" >> $OUT/${R}_sanitizer.txt
done
ls -la $OUT
