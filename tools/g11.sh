for v in g_base g_nottl g_noarg; do AB_LIB=tools/var_$v.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g11_$v.csv python tools/prof_kernels.py fit 28 > /dev/null 2>&1; done
ncu --set full --clock-control none --import-source on -k regex:fit_finish -s 3 -c 1 -o gpurun_out/g11_finish python tools/prof_kernels.py fit 28 > gpurun_out/g11_ncu.log 2>&1
python tools/prof_kernels.py replay cfg2 4096 > gpurun_out/g11_cfg2.txt 2>&1
