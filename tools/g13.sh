python -m pytest tests/test_gpu_fit.py tests/test_estimator_abi.py -m gpu -q > gpurun_out/g13_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g13_pytest.txt
python -m pytest tests/test_gpu_parity.py -m gpu -q -k fit >> gpurun_out/g13_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g13_pytest.txt
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize.py > gpurun_out/g13_memcheck.txt 2>&1
python tools/prof_kernels.py fit 28 > gpurun_out/g13_fit.txt 2>&1
