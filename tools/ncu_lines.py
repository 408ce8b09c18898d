"""Aggregate an ncu SASS source page by CUDA source line (via nvdisasm --print-line-info).

usage: python tools/ncu_lines.py report.ncu-rep kernel_regex cubin function_mangled [top]
"""
import csv, io, re, subprocess, sys
from collections import defaultdict

rep, kre, cubin, fn = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
dis = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
lines = dis.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + fn + ":"))
off2line = {}
cur = None
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("\t.section"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+[^;]", l)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia = hdr.index("Address"); ie = hdr.index("Instructions Executed"); iw = hdr.index("Warp Stall Sampling (All Samples)")
data = rows[2:]
base = int(data[0][ia], 16)
agg = defaultdict(lambda: [0, 0])
tot = [0, 0]
for r in data:
    try:
        off = int(r[ia], 16) - base
        e = int(r[ie] or 0); w = int(r[iw] or 0)
    except Exception:
        continue
    key = off2line.get(off, ("?", 0))
    agg[key][0] += e; agg[key][1] += w
    tot[0] += e; tot[1] += w
src = {}
for (f, ln) in agg:
    pass
print("total warp-inst %d, stall samples %d" % tuple(tot))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print("%-14s %5d  inst %5.1f%%  stall %5.1f%%" % (k[0], k[1], 100 * v[0] / tot[0], 100 * v[1] / max(tot[1], 1)))
