for v in 2 0; do echo "variant $v"; CT_FIT_VARIANT=$v python tools/prof_kernels.py fit 28 | tail -1; done
python -m pytest tests/test_gpu_parity.py -q -x -k "fit" 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:fit_ -s 2 -c 2 python tools/prof_kernels.py fit 28 2>/dev/null | grep "fit_" | awk -F'","' '{print $5, $NF}'
