"""Summarise .ncu-rep captures into a markdown table + JSON (committed under profiles/).

usage: python tools/summarize_ncu.py out_prefix rep1 [rep2 ...]
"""
import csv, io, json, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("sm__inst_executed.sum", "sm_warp_inst"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_registers", "occ_limit_regs"),
    ("launch__occupancy_limit_shared_mem", "occ_limit_smem"),
    ("sm__maximum_warps_per_active_cycle_pct", "theoretical_occ_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_pipe_pct"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
]
STALLS = ["wait", "selected", "long_scoreboard", "short_scoreboard", "dispatch_stall", "branch_resolving",
          "math_pipe_throttle", "mio_throttle", "lg_throttle", "not_selected", "barrier", "no_instructions"]


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")[:80]}
        for k, name in KEYS:
            if k in d and d[k] not in ("", "n/a"):
                try:
                    rec[name] = float(d[k].replace(",", ""))
                    rec[name + "_unit"] = u.get(k, "")
                except ValueError:
                    pass
        st = {}
        for s in STALLS:
            k = "smsp__pcsamp_warps_issue_stalled_" + s
            if k in d:
                try:
                    st[s] = int(float(d[k]))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1
        rec["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda kv: -kv[1])}
        res.append(rec)
    return res


def main():
    prefix, reps = sys.argv[1], sys.argv[2:]
    allr = {}
    lines = ["| report | kernel | duration | DRAM R+W | DRAM % | issue active % | warps active % | warp inst | regs | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for rep in reps:
        for rec in read(rep):
            allr.setdefault(rep.split("/")[-1], []).append(rec)
            dur = rec.get("duration", 0)
            du = rec.get("duration_unit", "")
            sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rw = (rec.get("dram_read", 0) * sc.get(rec.get("dram_read_unit", "byte"), 1) +
                  rec.get("dram_write", 0) * sc.get(rec.get("dram_write_unit", "byte"), 1))
            ru = "B"
            rec["dram_rw_bytes"] = rw
            top = ", ".join("%s %.0f%%" % (k, 100 * v) for k, v in list(rec["stall_share"].items())[:3])
            lines.append("| %s | %s | %.1f %s | %.4g %s | %.1f | %.1f | %.1f | %.4g | %d | %s |" % (
                rep.split("/")[-1], rec["kernel"][:40], dur, du, rw, ru, rec.get("dram_pct", 0),
                rec.get("issue_active_pct", 0), rec.get("warps_active_pct", 0), rec.get("warp_inst", rec.get("sm_warp_inst", 0)),
                rec.get("regs", 0), top))
    open(prefix + ".md", "w").write("\n".join(lines) + "\n")
    json.dump(allr, open(prefix + ".json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
