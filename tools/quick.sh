python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for i in 1 2; do python tools/prof_kernels.py replay cfg3 64 | tail -1 | cut -c1-100; done
python tools/prof_kernels.py replay cfg2 4096 | tail -1 | cut -c1-100
ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:replay -c 1 python tools/prof_kernels.py replay cfg3 16 2>/dev/null | grep replay_kernel | awk -F'","' '{print $(NF-2), $NF}'
