"""Wall-clock breakdown of one public run() call at config 1 (e2e leg of bench.py)."""
import time

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1903_03237_b200 import SeparatorConfig, separate as S
from paper_1903_03237_b200.synth import CONFIGS, baseline_init, make_mixture_torch

cfg = CONFIGS["c1"]
F, T, M, N, K = (cfg[k] for k in ("F", "T", "M", "N", "K"))
X = make_mixture_torch(F, T, M, N, K, seed=0, device="cuda").to(torch.complex64).unsqueeze(0)
Xh = X[0].cpu().pin_memory()
init = baseline_init(F, T, M, N, K, 0)
scfg = SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K, n_iterations=100, precision="complex64")
if "--bench-like" in sys.argv:  # the bench process also holds its own loop and a 256 MiB flush buffer
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    keep = S.run(scfg, Xh, init=init)
S.run(scfg, Xh, init=init)
torch.cuda.synchronize()


def tick(tag, t):
    torch.cuda.synchronize()
    now = time.perf_counter()
    print(f"{tag:28s} {1e3 * (now - t):8.2f} ms", flush=True)
    return now


for rep in range(2):
    t = time.perf_counter()
    t00 = t
    Xd = Xh.to("cuda")
    t = tick("H2D X", t)
    Xs, scale, floor = S._prepare_observation(Xh, scfg, torch)
    t = tick("prepare_observation", t)
    loop = S.DeviceLoop(Xs, S._as_batch(init[0], torch, 1), S._as_batch(init[1], torch, 1),
                        S._as_batch(init[2], torch, 1), S._as_batch(init[3], torch, 1), floor,
                        True, 1, n_trace=100)
    t = tick("DeviceLoop()", t)
    loop.prologue()
    t = tick("prologue", t)
    loop.run(1, use_graph=True)
    t = tick("iteration 1 (graph capture)", t)
    for _ in range(99):
        loop.run(1, use_graph=True)
    t = tick("iterations 2..100", t)
    img = loop.images_batch(scale)[0]
    t = tick("images (device)", t)
    out = torch.empty(img.shape, dtype=img.dtype, pin_memory=True)
    t = tick("pinned alloc (host cache)", t)
    out.copy_(img, non_blocking=True)
    t = tick("D2H into pinned", t)
    del out
    print("torch threads", torch.get_num_threads())
    print(f"{'total':28s} {1e3 * (t - t00):8.2f} ms")
