python tools/prof_kernels.py fit 28 > gpurun_out/g5_fit.txt 2>&1
python tools/prof_kernels.py fit 28 >> gpurun_out/g5_fit.txt 2>&1
python -m pytest tests/test_gpu_fit.py tests/test_gpu_parity.py tests/test_estimator_abi.py tests/test_gpu_validation.py tests/test_gpu_growth.py tests/test_next3_analyses.py tests/test_synth.py -m gpu -q > gpurun_out/g5_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g5_pytest.txt
python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "fit_full or cfg4 or cfg2" >> gpurun_out/g5_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g5_pytest.txt
