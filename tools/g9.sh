ncu --set full --clock-control none --import-source on -k regex:fit_finish -s 3 -c 1 -o gpurun_out/g9_finish python tools/prof_kernels.py fit 28 > gpurun_out/g9_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 -o gpurun_out/g9_replay_cfg2 python tools/prof_kernels.py replay cfg2 4096 > gpurun_out/g9_ncu_cfg2.log 2>&1
