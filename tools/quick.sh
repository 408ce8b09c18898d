python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
python tools/prof_kernels.py replay cfg3 64 | tail -1
python tools/prof_kernels.py replay cfg2 256 | tail -1
