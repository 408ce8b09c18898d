"""Write profiles/ncu_constants.json entries from an ncu report (bench.py roofline inputs).

usage: python tools/ncu_constants.py replay <report> <workload_name> <replica_turns>
       python tools/ncu_constants.py replay-auto <report> <cfgN> <log of the captured run>
       python tools/ncu_constants.py fit <report> <samples>
"""
import csv, io, json, os, subprocess, sys

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_constants.json")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def num(d, k):
    return float(d[k].replace(",", ""))


def scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    c = json.load(open(OUT)) if os.path.exists(OUT) else {}
    kind, rep = sys.argv[1], sys.argv[2]
    rows, units = raw(rep)
    # every kernel of the report: the launches of one call (a split sweep runs two replay
    # launches; a 32 < P <= 256 sweep its list-driven fallback launch)
    dram = sum(num(d, "dram__bytes_read.sum") * scale(units["dram__bytes_read.sum"]) +
               num(d, "dram__bytes_write.sum") * scale(units["dram__bytes_write.sum"]) for d in rows)
    if kind == "replay-auto":  # replica-turns from the captured run's own log line
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from ctgen import configs as cf
        w = {"cfg2": cf.config2, "cfg3": cf.config3, "cfg4": cf.config4, "cfg5": cf.config5}[sys.argv[3]]()
        import re
        txt = open(sys.argv[4]).read()
        turns = float(re.findall(r"replicas (\d+) turns", txt)[0])
        sys.argv[3:5] = [w.name, str(turns)]
        kind = "replay"
    if kind == "replay":
        name, turns = sys.argv[3], float(sys.argv[4])
        inst = sum(num(d, "smsp__inst_executed.sum") for d in rows)
        c.setdefault("replay_warp_inst_per_turn", {})[name] = inst / turns
        c.setdefault("replay_dram_bytes_per_turn", {})[name] = dram / turns
        c.setdefault("source", {})["replay_" + name] = os.path.basename(rep)
    else:
        n = float(sys.argv[3])
        c["fit_dram_bytes_per_sample"] = dram / n
        c["fit_dram_bytes_per_launch_2^28"] = dram / n * 2**28
        c.setdefault("source", {})["fit"] = os.path.basename(rep)
    json.dump(c, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps(c, indent=1))


if __name__ == "__main__":
    main()
