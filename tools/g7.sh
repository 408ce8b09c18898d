for r in 1 2; do for v in f2_base f2_fu6 f2_fu4 f2_noneg f2_fw4; do echo "== $v"; AB_LIB=tools/var_$v.so python tools/prof_kernels.py fit 28 2>&1 | head -2; done; done > gpurun_out/g7_fitvar.txt 2>&1
python -m pytest tests/test_gpu_fit.py tests/test_estimator_abi.py -m gpu -q > gpurun_out/g7_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g7_pytest.txt
python -m pytest tests/test_gpu_parity.py -m gpu -q >> gpurun_out/g7_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g7_pytest.txt
