#!/usr/bin/env python
"""Static SASS opcode histogram of selected kernels of libfastmnmf.so
(cuobjdump -sass): usage sass_hist.py MANGLED_NAME_REGEX... Prints, per
kernel, the instruction count and the opcodes that prove the pipe it uses
(FFMA2 / DFMA on the FMA pipes; UTCHMMA/UTCQMMA/UTCMMA (tcgen05.mma), LDTM/STTM
(tcgen05.ld/st), UTMALDG (TMA) / UBLKCP (cp.async.bulk), SYNCS (mbarrier) on the
tensor-core path)."""
import re
import subprocess
import sys
from collections import Counter

LIB = "paper_1903_03237_b200/libfastmnmf.so"
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", sass)
pats = [re.compile(p) for p in sys.argv[1:]]
for blk in blocks[1:]:
    name = blk.split("\n", 1)[0].strip()
    if not any(p.search(name) for p in pats):
        continue
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    ops = Counter()
    for line in blk.splitlines():
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            ops[m.group(2).split(".")[0]] += 1
    tot = sum(ops.values())
    key = [o for o in ("FFMA2", "FFMA", "DFMA", "FMUL", "LDS", "LDSM", "STS", "LDG", "STG", "LDGSTS",
                       "UTCHMMA", "UTCQMMA", "UTCMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UBLKCP", "SYNCS", "SHFL",
                       "MUFU", "BAR") if ops.get(o)]
    print(f"{dem}: {tot} instructions; " + ", ".join(f"{o} {ops[o]}" for o in key))
