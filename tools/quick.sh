#!/bin/bash
# Quick GPU A/B: replay throughput of cfg3 (register budgets), cfg5, cfg2.  gpurun, ONE GPU.
for mb in 8 10 12; do echo "minb $mb"; CT_REPLAY_MINB=$mb python tools/prof_kernels.py replay cfg3 64 | tail -1 | cut -c1-110; done
python tools/prof_kernels.py replay cfg5 16 | tail -1 | cut -c1-110
python tools/prof_kernels.py replay cfg2 1024 | tail -1 | cut -c1-110
