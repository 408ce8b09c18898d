#!/bin/bash
# Warp instructions per replica-turn of the replay kernel, in-tree library vs variants (gpurun, ONE GPU).
# usage: tools/ab_inst.sh "cfg3 cfg5" seeds v1 v2 ...
WL=$1; S=$2; shift 2
for w in $WL; do
  for v in main "$@"; do
    if [ $v = main ]; then L=""; else L="AB_LIB=tools/var_$v.so"; fi
    env $L ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
      -k regex:replay_kernel -c 1 --csv python tools/prof_kernels.py replay $w $S 2>/dev/null > /tmp/abi.csv
    turns=$(env $L python tools/prof_kernels.py replay $w $S | tail -1 | sed 's/.* replicas \([0-9]*\) turns.*/\1/')
    python - "$v" "$w" "$turns" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open("/tmp/abi.csv")) if len(r) > 10]
h = rows[0]; d = {}
for r in rows[1:]:
    d[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
t = int(sys.argv[3])
print("%-6s %s inst/turn %.1f issue %.1f%%" % (sys.argv[1], sys.argv[2], d["smsp__inst_executed.sum"] / t,
      d["smsp__issue_active.avg.pct_of_peak_sustained_active"]))
PY
  done
done
