python tools/prof_kernels.py fit 28 > gpurun_out/g4_fit.txt 2>&1
python tools/prof_kernels.py fit 28 >> gpurun_out/g4_fit.txt 2>&1
python -m pytest tests/test_gpu_fit.py tests/test_gpu_parity.py tests/test_estimator_abi.py tests/test_gpu_validation.py -m gpu -x -q > gpurun_out/g4_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g4_pytest.txt
python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "fit_full or cfg4" >> gpurun_out/g4_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g4_pytest.txt
ncu --set full --clock-control none --import-source on -k regex:replay_kernel -c 1 -o gpurun_out/g4_replay_cfg4 python bench.py --workload cfg4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-fit-bandwidth > gpurun_out/g4_ncu_cfg4.log 2>&1
