for i in 1 2 3; do python tools/prof_kernels.py replay cfg3 256 2>&1 | tail -1 | cut -c1-100; done > gpurun_out/g19_perf.txt 2>&1
