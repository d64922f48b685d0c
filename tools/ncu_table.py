"""Per-launch table from an `ncu --metrics ... --csv` launch list (development
aid): one row per launch, labelled by the run_once.py specs in order.

    python tools/ncu_table.py launches.csv N spec1 spec2 ...
"""
import csv
import sys


def main():
    path, n = sys.argv[1], float(sys.argv[2])
    specs = sys.argv[3:]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ci = {h: i for i, h in enumerate(hdr)}
    launches = {}
    for r in rows[1:]:
        launches.setdefault(int(r[ci["ID"]]), {})[r[ci["Metric Name"]]] = r[ci["Metric Value"]].replace(",", "")
    print("%-8s %9s %7s %7s %6s %5s %9s %6s %7s %7s %7s" % ("launch", "time_us", "issue%", "fp64%", "warps", "regs",
                                                           "instr/x", "GB/s", "wait", "noinst", "mpthr"))
    for j, lid in enumerate(sorted(launches)):
        m = launches[lid]
        t_us = float(m["gpu__time_duration.sum"]) / (1e3 if float(m["gpu__time_duration.sum"]) > 1e4 else 1)
        k = int(specs[j].split(":")[-1]) if j < len(specs) else 0
        gbs = n * (16 + 8 * k) / (t_us * 1e-6) / 1e9
        print("%-8s %9.1f %7.1f %7.1f %6.1f %5s %9.1f %6.0f %7.2f %7.2f %7.2f" % (
            specs[j] if j < len(specs) else lid, t_us, float(m["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
            float(m["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
            float(m["sm__warps_active.avg.per_cycle_active"]), m["launch__registers_per_thread"],
            float(m["smsp__inst_executed.sum"]) * 32 / n, gbs,
            float(m["smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]),
            float(m["smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio"]),
            float(m["smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"])))


if __name__ == "__main__":
    main()
