"""Build an experimental libcontinuum variant for A/B timing (tools/ab.sh, AB_LIB=...).

    python tools/build_variant.py NAME [-DMACRO=1 ...] [--patch FILE:OLD=>NEW ...]

Copies paper_2511_02230_b200/csrc to a temporary directory, applies literal text patches,
compiles with the extra -D flags to tools/var_NAME.so.  Not part of the product.
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_02230_b200 import build as B  # noqa: E402


def main():
    name = sys.argv[1]
    defs = [a for a in sys.argv[2:] if a.startswith("-D")]
    patches = [a for a in sys.argv[2:] if "=>" in a]
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "csrc")
        shutil.copytree(os.path.join(ROOT, "paper_2511_02230_b200", "csrc"), src)
        for p in patches:
            f, rest = p.split(":", 1)
            old, new = rest.split("=>", 1)
            path = os.path.join(src, f)
            s = open(path).read()
            assert old in s, (f, old)
            open(path, "w").write(s.replace(old, new))
        out = os.path.join(ROOT, "tools", "var_%s.so" % name)
        srcs = sorted(os.path.join(src, x) for x in os.listdir(src) if x.endswith((".cu", ".cpp")))
        B.compile_link(srcs, out, extra=defs)
        print(out)


if __name__ == "__main__":
    main()
