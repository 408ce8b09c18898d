"""SASS instruction count per kernel of a cubin / .so (instruction-cache footprint check).
usage: python tools/sass_size.py file [regex]"""
import re, subprocess, sys
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
cnt, name = {}, None
for l in out.splitlines():
    m = re.search(r"Function : (\S+)", l)
    if m:
        name = m.group(1); cnt.setdefault(name, 0); continue
    if name and re.match(r"\s+/\*[0-9a-f]+\*/\s+\S", l):
        cnt[name] += 1
for n, c in sorted(cnt.items()):
    if pat is None or pat.search(n):
        print("%6d  %s" % (c, n))
