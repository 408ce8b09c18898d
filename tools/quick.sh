python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
python tools/prof_kernels.py replay cfg2 4096 | tail -1 | cut -c1-120
ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:replay -c 1 python tools/prof_kernels.py replay cfg2 512 2>/dev/null | grep replay_kernel | awk -F'","' '{print $(NF-2), $NF}'
