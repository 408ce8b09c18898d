python tools/prof_kernels.py fit 28 > gpurun_out/g10_fit.txt 2>&1
python tools/prof_kernels.py fit 28 >> gpurun_out/g10_fit.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g10_fit_launches.csv python tools/prof_kernels.py fit 28 > /dev/null 2>&1
python -m pytest tests/test_gpu_fit.py tests/test_estimator_abi.py -m gpu -q > gpurun_out/g10_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g10_pytest.txt
python -m pytest tests/test_gpu_parity.py -m gpu -q -k fit >> gpurun_out/g10_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g10_pytest.txt
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -k "fit_full or cfg4" >> gpurun_out/g10_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g10_pytest.txt
