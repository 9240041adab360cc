#!/usr/bin/env python
"""Per-kernel issue / stall summary from an `ncu --page raw --csv` export.

usage: ncu_stalls.py RAW.csv
Prints, per captured launch: duration, instructions per SMSP, issue-active %,
shared-memory wavefronts per SM against active cycles, and the warp stall
reasons in cycles per issued instruction (largest first)."""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h = rows[0]
    col = {n: i for i, n in enumerate(h)}

    def g(r, k):
        try:
            return float(r[col[k]].replace(",", ""))
        except Exception:  # noqa: BLE001
            return float("nan")

    for r in rows[2:]:
        if len(r) != len(h):
            continue
        name = r[col["Kernel Name"]][:60]
        st = {n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): g(r, n)
              for n in h if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")
              and "not_issued" not in n}
        top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
        print(name)
        print("  dur %s %s  inst/SMSP %.0f  issue-active %.1f%%  cycles-active %.0f  smem wavefronts/SM %.0f" % (
            r[col["gpu__time_duration.sum"]], rows[1][col["gpu__time_duration.sum"]], g(r, "smsp__inst_executed.avg"),
            g(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"), g(r, "sm__cycles_active.avg"),
            g(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") / 148))
        print("  stalls/issue: " + ", ".join("%s %.2f" % kv for kv in top))


if __name__ == "__main__":
    main()
