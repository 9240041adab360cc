#!/usr/bin/env python
"""SASS opcode histogram (executed warp instructions) of one kernel in an
ncu report: ncu_ops.py REPORT KERNEL_REGEX [TOP]."""
import csv
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
c, tot, seen = Counter(), 0, set()
for r in csv.reader(out.splitlines()):
    if len(r) > 4 and r[0].startswith("0x"):
        if r[0] in seen:
            continue
        seen.add(r[0])
        try:
            ie = int(r[5])
        except ValueError:
            continue
        toks = r[1].split()
        op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
        c[op] += ie
        tot += ie
print(f"total {tot:.3e} warp instructions")
for op, v in c.most_common(top):
    print(f"{op:24s} {v:13d} {100 * v / tot:5.1f}%")
