ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g8_fit_launches.csv python tools/prof_kernels.py fit 28 > /dev/null 2>&1
AB_LIB=tools/var_f2_noneg.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g8_fit_launches_noneg.csv python tools/prof_kernels.py fit 28 > /dev/null 2>&1
python -m pytest tests/test_gpu_validation.py tests/test_gpu_growth.py tests/test_next3_analyses.py tests/test_synth.py tests/test_ingest.py -m gpu -q > gpurun_out/g8_pytest.txt 2>&1; echo rc=$? >> gpurun_out/g8_pytest.txt
