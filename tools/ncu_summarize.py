#!/usr/bin/env python3
"""Summarise an `ncu --set full` report into profiles/ (text + ncu_summary.json).

    python tools/ncu_summarize.py gpurun_out/prof.ncu-rep <key> <out.txt> [n] [index]

<key> names the workload (e.g. soa_k32; "-" to leave ncu_summary.json alone);
the report may also be an exported `--page raw --csv` file.  ncu_summary.json[launches][key] gets
the per-launch DRAM traffic that bench.py reports as roofline.traffic (of the
index-th kernel in the report, default the last); out.txt lists every kernel.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
    "sm__cycles_active.avg", "sm__cycles_active.min", "sm__cycles_active.max", "lts__t_bytes.sum",
    "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
]
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    if rep.endswith(".csv"):  # an exported `ncu -i ... --page raw --csv`
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, key, txt = sys.argv[1], sys.argv[2], sys.argv[3]
    n_x = int(float(sys.argv[4])) if len(sys.argv) > 4 else None
    pick = int(sys.argv[5]) if len(sys.argv) > 5 else -1
    h, u, data = raw(rep)
    lines = []
    summaries = []
    for v in data:
        name = v[h.index("Kernel Name")]
        lines.append("kernel: %s" % name)
        vals = {}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                lines.append("  %-66s %s %s" % (m, v[i], u[i]))
                vals[m] = (v[i], u[i])
        stalls = []
        for i, m in enumerate(h):
            if m.startswith("smsp__average_warps_issue_stalled") and m.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(v[i]), m))
                except ValueError:
                    pass
        lines.append("  top stall reasons (warps per issue):")
        for val, m in sorted(stalls, reverse=True)[:6]:
            lines.append("    %-80s %.3f" % (m.replace("smsp__average_warps_issue_stalled_", ""), val))
        def num(m):
            s, unit = vals[m]
            return float(s) * UNITS.get(unit, 1)
        t_ns = float(vals["gpu__time_duration.sum"][0]) * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6,
                                                           "msecond": 1e6}.get(vals["gpu__time_duration.sum"][1], 1)
        summary = {"kernel": name, "ncu_time_ns": t_ns,
                   "dram_bytes_read": num("dram__bytes_read.sum"), "dram_bytes_write": num("dram__bytes_write.sum"),
                   "report": os.path.basename(rep)}
        summary["dram_bytes_per_launch"] = summary["dram_bytes_read"] + summary["dram_bytes_write"]
        if n_x:
            summary["n"] = n_x
        summaries.append(summary)
    summary = summaries[pick]
    with open(txt, "w") as f:
        f.write("# ncu --set full --clock-control none (%s); per-launch values, cold cache, serialised\n" % rep)
        f.write("\n".join(lines) + "\n")
    if key != "-":
        js = os.path.join(ROOT, "profiles", "ncu_summary.json")
        doc = json.load(open(js)) if os.path.exists(js) else {"launches": {}}
        doc["launches"][key] = summary
        json.dump(doc, open(js, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
