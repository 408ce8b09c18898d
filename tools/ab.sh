#!/bin/bash
# A/B of library variants built in tools/var_*.so (loaded by tools/prof_kernels.py via AB_LIB); args: workload seeds variants...
W=$1; S=$2; shift 2
for i in 1 2; do for v in "$@"; do echo -n "$v "; AB_LIB=tools/var_$v.so python tools/prof_kernels.py replay $W $S | tail -1 | cut -c1-90; done; done
