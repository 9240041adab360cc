#!/usr/bin/env python
"""Summarise an ncu --set full report: one row per profiled launch with
duration, DRAM bytes, throughput and pipe utilisation. usage:
ncu_summary.py REPORT [OUT.md]"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur (us)"),
    ("dram__bytes_read.sum", "DRAM rd (MB)"),
    ("dram__bytes_write.sum", "DRAM wr (MB)"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ik = h.index("Kernel Name")
    lines = ["| kernel | " + " | ".join(k[1] for k in KEYS) + " |",
             "|---" * (len(KEYS) + 1) + "|"]
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        name = r[ik].split("(")[0].replace("void ", "")
        vals = []
        for k, _ in KEYS:
            v = d.get(k, "")
            try:
                v = f"{float(v.replace(',', '')):.4g}"
            except ValueError:
                pass
            vals.append(v)
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
    text = "\n".join(lines)
    print(text)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text + "\n")


if __name__ == "__main__":
    main()
