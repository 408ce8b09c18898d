python tools/prof_kernels.py fit 28 > gpurun_out/g14_fit.txt 2>&1
python tools/prof_kernels.py fit 28 >> gpurun_out/g14_fit.txt 2>&1
python -m pytest tests/test_gpu_fit.py -m gpu -q > gpurun_out/g14_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g14_pytest.txt
python -m pytest tests/test_gpu_parity.py -m gpu -q -k fit >> gpurun_out/g14_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g14_pytest.txt
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "fit_full" >> gpurun_out/g14_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g14_pytest.txt
