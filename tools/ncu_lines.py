#!/usr/bin/env python
"""Aggregate an ncu report's source page per CUDA source line.

usage: ncu_lines.py REPORT KERNEL_REGEX [TOP]
Prints the source lines with the most warp-stall samples and executed
warp instructions (needs -lineinfo builds and --import-source on capture).
"""
import csv
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    agg = {}
    fname = "?"
    hdr = None
    cur = None
    tot_s = tot_i = 0.0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            iS = hdr.index("Warp Stall Sampling (All Samples)")
            iI = hdr.index("Instructions Executed")
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        if r[0]:  # a source line row
            cur = (fname, int(r[0]), r[1][:90])
            continue
        try:
            s, n = float(r[iS] or 0), float(r[iI] or 0)
        except ValueError:
            continue
        a = agg.setdefault(cur, [0.0, 0.0])
        a[0] += s
        a[1] += n
        tot_s += s
        tot_i += n
    print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.3g}")
    for k, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100*s/max(tot_s,1):5.1f}% stall {100*n/max(tot_i,1):5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
