for r in 1 2; do for v in f_base f_nottl f_noargmax f_nophase2 f_nosync f_noneg; do echo "== $v"; AB_LIB=tools/var_$v.so python tools/prof_kernels.py fit 28 2>&1 | head -2; done; done > gpurun_out/g3_fitvar.txt 2>&1
python -m pytest tests -m gpu -x -q -k "not cfg3 and not cfg5" > gpurun_out/g3_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g3_pytest.txt
python bench.py --workload cfg4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-fit-bandwidth > gpurun_out/g3_bench_cfg4.txt 2>&1
python bench.py --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/g3_bench_cfg3.txt 2>&1
