python tools/prof_kernels.py replay cfg3 256 > gpurun_out/g18_perf.txt 2>&1
python tools/prof_kernels.py replay cfg5 256 >> gpurun_out/g18_perf.txt 2>&1
python tools/prof_kernels.py replay cfg4 4096 >> gpurun_out/g18_perf.txt 2>&1
python tools/prof_kernels.py replay cfg2 4096 >> gpurun_out/g18_perf.txt 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_validation.py -m gpu -q -x > gpurun_out/g18_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g18_pytest.txt
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "cfg2 or cfg4 or cfg5" >> gpurun_out/g18_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g18_pytest.txt
python __graft_entry__.py > gpurun_out/g18_smoke.txt 2>&1
