#!/bin/bash
# Per-source-line instructions / stall samples of the replay kernel (gpurun, ONE GPU).
# usage: tools/src_profile.sh "cfg3 cfg2" seeds [tag]
WL=$1; S=$2; T=${3:-cur}
mkdir -p gpurun_out
for w in $WL; do
  ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section Occupancy \
      --import-source on -k regex:replay_kernel -c 1 -o /tmp/sp_$w -f \
      python tools/prof_kernels.py replay $w $S > /dev/null 2>&1
  python tools/ncu_src_lines.py /tmp/sp_$w.ncu-rep 70 > gpurun_out/src_${T}_$w.txt 2>&1
done
