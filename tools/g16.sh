ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 -o gpurun_out/g16_replay_cfg3 python tools/prof_kernels.py replay cfg3 16 > gpurun_out/g16_ncu_cfg3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 -o gpurun_out/g16_replay_cfg5 python tools/prof_kernels.py replay cfg5 16 > gpurun_out/g16_ncu_cfg5.log 2>&1
python tools/prof_kernels.py replay cfg3 256 > gpurun_out/g16_cfg3.txt 2>&1
python tools/prof_kernels.py replay cfg5 256 >> gpurun_out/g16_cfg3.txt 2>&1
python tools/prof_kernels.py replay cfg4 4096 >> gpurun_out/g16_cfg3.txt 2>&1
