#!/bin/bash
# Round measurement bundle (run under gpurun, ONE GPU).  Writes gpurun_out/${R}_*.
# Order: ncu captures first, so the bench's roofline reads per-unit constants (warp-inst and
# DRAM bytes per replica-turn, DRAM bytes per sample) measured on the code being benchmarked.
# Replay captures are FULL-SIZE launches of each workload (outputs larger than L2), so their
# DRAM traffic includes the summary writes.
R=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${R}_gpu.txt
cap() {  # cap NAME WORKLOAD SEEDS [LAUNCHES of one call]
  ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c ${4:-1} \
      -o $OUT/${R}_replay_$1 python tools/prof_kernels.py replay $2 $3 > $OUT/${R}_ncu_replay_$1.log 2>&1
}
cap cfg3 cfg3 256
cap cfg2 cfg2 4096 2
cap cfg4 cfg4 4096
cap cfg5 cfg5 256 2
ncu --set full --clock-control none --import-source on -k regex:fit_hist -s 3 -c 1 \
    -o $OUT/${R}_fit_hist python tools/prof_kernels.py fit 28 > $OUT/${R}_ncu_fit.log 2>&1
python tools/ncu_constants.py fit $OUT/${R}_fit_hist.ncu-rep 268435456 > $OUT/${R}_constants.log 2>&1
for w in cfg3 cfg2 cfg4 cfg5; do
  python tools/ncu_constants.py replay-auto $OUT/${R}_replay_$w.ncu-rep $w $OUT/${R}_ncu_replay_$w.log >> $OUT/${R}_constants.log 2>&1
done
cp profiles/ncu_constants.json $OUT/${R}_ncu_constants.json
python tools/summarize_ncu.py $OUT/${R}_ncu_summary $OUT/${R}_replay_cfg3.ncu-rep $OUT/${R}_replay_cfg2.ncu-rep \
    $OUT/${R}_replay_cfg4.ncu-rep $OUT/${R}_replay_cfg5.ncu-rep $OUT/${R}_fit_hist.ncu-rep > /dev/null 2>&1
# per-source-line instruction / stall tables, then park the big reports outside gpurun_out/
# (the copy-back is capped at 64 MiB)
for w in cfg3 cfg2 cfg4 cfg5; do
  python tools/ncu_src_lines.py $OUT/${R}_replay_$w.ncu-rep 60 > $OUT/${R}_srclines_$w.txt 2>&1
done
python tools/ncu_src_lines.py $OUT/${R}_fit_hist.ncu-rep 40 > $OUT/${R}_srclines_fit.txt 2>&1
mkdir -p /tmp/ncu_reps && mv $OUT/${R}_replay_*.ncu-rep /tmp/ncu_reps/
python bench.py > $OUT/${R}_bench.log 2>&1
tail -1 $OUT/${R}_bench.log > $OUT/${R}_bench.json
for w in cfg2 cfg4 cfg5; do
  python bench.py --workload $w --no-fit-bandwidth > $OUT/${R}_bench_$w.log 2>&1
  tail -1 $OUT/${R}_bench_$w.log > $OUT/${R}_bench_$w.json
done
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/${R}_bench_reference.log 2>&1
tail -1 $OUT/${R}_bench_reference.log > $OUT/${R}_bench_reference.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/${R}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-fit-bandwidth > $OUT/${R}_launches_bench.log 2>&1
# compute-sanitizer is closed on this GPU pool (round 2): the round-1 sanitizer run stands
ls -la $OUT
