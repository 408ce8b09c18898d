"""Mutation check of the oracle's pins (TEST INFRASTRUCTURE; reads and builds oracle/ only).

Each mutation is a plausible mistake in oracle/ct_oracle.cpp (a wrong rounding, a dropped term,
a transposed field, an off-by-one).  For each, the mutated oracle is built into a temporary
library and the pins named for it are run against that build (CT_ORACLE_LIB); a pin is only
worth something if it FAILS under its mutation.  Writes a table to stdout (and to the path
given as argv[1]).  DESIGN.md §4 lists the result.
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "ct_oracle.cpp")

# (name, passage / reading, original text, mutated text, pytest -k selection)
MUTATIONS = [
    ("p50 rank floor+1 instead of ceil", "R20, SPEC.md:528",
     "int64_t r50 = (50 * (int64_t)P + 99) / 100", "int64_t r50 = (50 * (int64_t)P) / 100 + 1",
     "bruteforce_tiny or invariants or nearest_rank"),
    ("p99 rank off by one", "R20, SPEC.md:528",
     "summary[5] = s[r99 - 1];", "summary[5] = s[r99 < P ? r99 : P - 1];",
     "bruteforce_tiny or invariants or nearest_rank"),
    ("cell max JCT summed", "ct_jct_stats, PAPER.md:886-888",
     "o[5] = std::max(o[5], s[3]);", "o[5] += s[3];", "jct_stats or invariants"),
    ("cell bubble/makespan transposed", "ct_jct_stats, R19",
     "o[6] += s[6];", "o[6] += s[7];", "jct_stats or invariants"),
    ("STEP release at now >= expiry", "R4/R15, PAPER.md:393, 638",
     "if (p[i].pinned && p[i].st != QUEUED && now > p[i].expiry) {",
     "if (p[i].pinned && p[i].st != QUEUED && now >= p[i].expiry) {",
     "golden_step_expiry or bruteforce_tiny"),
    ("STEP releases queued programs too", "R4, PAPER.md:639-640",
     "if (p[i].pinned && p[i].st != QUEUED && now > p[i].expiry) {",
     "if (p[i].pinned && now > p[i].expiry) {", "golden_step_expiry or bruteforce_tiny"),
    ("V_j without /a_den", "C-4 (DESIGN.md §3)",
     "i128 V = ((i128)c_pf * ctx_j[j] * ((i128)a_den + (i128)a_num * w_j[j])) / a_den;",
     "i128 V = ((i128)c_pf * ctx_j[j] * ((i128)a_den + (i128)a_num * w_j[j]));",
     "rational_turn_factor"),
    ("C_j with floor(ctx/bs)", "C-4 (DESIGN.md §3)",
     "i128 C = (i128)c_pin * ceil_div(ctx_j[j], bs);", "i128 C = (i128)c_pin * (ctx_j[j] / bs);",
     "rational_turn_factor"),
    ("V_j rounded up", "C-4 (DESIGN.md §3)",
     "i128 V = ((i128)c_pf * ctx_j[j] * ((i128)a_den + (i128)a_num * w_j[j])) / a_den;",
     "i128 V = ((i128)c_pf * ctx_j[j] * ((i128)a_den + (i128)a_num * w_j[j]) + a_den - 1) / a_den;",
     "rational_turn_factor"),
    ("bubble counted from the program arrival", "SPEC.md:337, 564 (JCT identity)",
     "p[h].bubble += now - p[h].req_arr;", "p[h].bubble += now - p[h].arrival;",
     "invariants or golden"),
    ("tool time not recorded", "SPEC.md:564 (JCT identity)",
     "p[i].tool_us += tr[3];", "p[i].tool_us += 0;", "invariants or golden"),
]


def main(out_path=None):
    src = open(SRC).read()
    rows = []
    with tempfile.TemporaryDirectory() as tmp:
        for name, cite, old, new, sel in MUTATIONS:
            assert src.count(old) == 1, name
            mut = os.path.join(tmp, "m.cpp")
            open(mut, "w").write(src.replace(old, new))
            lib = os.path.join(tmp, "lib_%d.so" % len(rows))
            subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I",
                                   os.path.join(ROOT, "oracle"), "-o", lib, mut, "-lpthread"])
            env = dict(os.environ, CT_ORACLE_LIB=lib)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu",
                                "-p", "no:cacheprovider", "tests/test_oracle_replay.py",
                                "tests/test_oracle_fit.py", "-k", sel],
                               cwd=ROOT, env=env, capture_output=True, text=True)
            caught = r.returncode != 0
            tail = [l for l in r.stdout.splitlines() if l.startswith("FAILED")][:1]
            rows.append((name, cite, sel, "CAUGHT" if caught else "missed",
                         tail[0].split(" - ")[0].replace("FAILED ", "") if tail else ""))
    lines = ["%-42s | %-34s | %-7s | %s" % ("mutation", "passage", "result", "first failing pin")]
    lines += ["%-42s | %-34s | %-7s | %s" % (n, c, res, t) for n, c, s, res, t in rows]
    text = "\n".join(lines)
    print(text)
    if out_path:
        open(out_path, "w").write(text + "\n")
    return all(r[3] == "CAUGHT" for r in rows)


if __name__ == "__main__":
    sys.exit(0 if main(sys.argv[1] if len(sys.argv) > 1 else None) else 1)
