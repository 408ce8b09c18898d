"""Instructions executed and stall samples per CUDA source line of an ncu capture (needs
-lineinfo).  usage: python tools/ncu_src_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0, ""])
fname, hdr, line = "", None, None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < len(hdr):
        continue
    d = dict(zip(hdr, row))
    if row[0]:  # a CUDA source line
        line = (fname, int(row[0]), row[1][:90])
        continue
    if line is None:
        continue
    try:
        ie = int(float(d["Instructions Executed"]))
        ss = int(float(d["Warp Stall Sampling (All Samples)"]))
    except (KeyError, ValueError):
        continue
    a = agg[line[:2]]
    a[0] += ie
    a[1] += ss
    a[2] = line[2]
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print("total warp-inst %d, stall samples %d" % (tot_i, tot_s))
for (f, ln), (ie, ss, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%6.2f%% inst %6.2f%% samples  %s:%d  %s" % (100 * ie / tot_i, 100 * ss / tot_s, f, ln, src))
