#!/usr/bin/env python
"""k_front phase timing via clock64 stamps (GPU). usage: phase_timing.py [config]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1903_03237_b200 import _lib  # noqa: E402
from paper_1903_03237_b200.separate import DeviceLoop, SeparatorConfig, _prepare_observation  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg = dict(bench.CONFIGS[cfgname])
cfg["B"] = 1
dev = torch.device("cuda", 0)
X, init = bench.make_problem(cfg, 0, torch, dev)
scfg = SeparatorConfig(n_sources=cfg["N"], n_basis=cfg["K"], n_iterations=20, precision=cfg["precision"])
Xs, scale, floor = _prepare_observation(X, scfg, torch)
loop = DeviceLoop(Xs, *init, floor, True, 1, n_trace=20)
loop.prologue()
loop.run(3)
buf = torch.zeros((cfg["F"], 8), dtype=torch.int64, device=dev)
lib = _lib.load()
lib.fm_debug_front_timing(_lib.ptr(buf))
loop.run(1)
torch.cuda.synchronize()
lib.fm_debug_front_timing(None)
t = buf.cpu().numpy().astype(np.float64)
d = np.diff(t[:, :3], axis=1)
names = ["A1 gain", "A2 V"]
for i, n in enumerate(names):
    print(f"{n:12s} mean {d[:, i].mean():9.0f} cyc  max {d[:, i].max():9.0f}")
print(f"{'total':12s} mean {(t[:,2]-t[:,0]).mean():9.0f} cyc")
span = t[:, 2].max() - t[:, 0].min()
print(f"kernel span (first start -> last end) {span:.0f} cyc")
