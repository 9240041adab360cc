"""cProfile of three public run() calls at config 1 (the bench e2e leg)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_03237_b200 import SeparatorConfig, run  # noqa: E402
from paper_1903_03237_b200.synth import CONFIGS, baseline_init, make_mixture_torch  # noqa: E402

cfg = CONFIGS["c1"]
F, T, M, N, K = (cfg[k] for k in ("F", "T", "M", "N", "K"))
X = make_mixture_torch(F, T, M, N, K, seed=0, device="cuda").to(torch.complex64)
Xh = X.cpu().pin_memory()
init = tuple(a for a in baseline_init(F, T, M, N, K, 0))
scfg = SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K, n_iterations=100, precision="complex64")
run(scfg, Xh, init=init)
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    res = run(scfg, Xh, init=init)
pr.disable()
print("per call ms", 1e3 * (time.perf_counter() - t0) / 3)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
