#!/bin/bash
# Quick GPU A/B: replay throughput of cfg3 / cfg5 / cfg2 slices.  gpurun, ONE GPU.
python tools/prof_kernels.py replay cfg3 64 | tail -1 | cut -c1-110
python tools/prof_kernels.py replay cfg5 16 | tail -1 | cut -c1-110
python tools/prof_kernels.py replay cfg2 1024 | tail -1 | cut -c1-110
