#!/bin/bash
# Full-size replay A/B (gpurun, ONE GPU): the in-tree library ("main") against variants built by
# tools/build_variant.py (tools/var_NAME.so).  usage: tools/ab_replay.sh "cfg3 cfg2" v1 v2 ...
WL=$1; shift
declare -A SEEDS=([cfg3]=256 [cfg5]=256 [cfg2]=4096 [cfg4]=4096)
for r in 1 2; do
  for w in $WL; do
    echo -n "main $w "; python tools/prof_kernels.py replay $w ${SEEDS[$w]} | tail -1 | cut -c1-100
    for v in "$@"; do
      echo -n "$v $w "; AB_LIB=tools/var_$v.so python tools/prof_kernels.py replay $w ${SEEDS[$w]} | tail -1 | cut -c1-100
    done
  done
done
