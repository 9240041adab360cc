"""The paper's comparison on B200: seconds per iteration of the full-rank
MNMF comparator (method "mnmf") against FastMNMF (method "fast-mnmf") on
the same mixture, both through the public run() (device time per iteration
from run()'s CUDA-event time_trace, median after the first iteration).
usage: python tools/fullrank_bench.py [F T M N K iters]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1903_03237_b200 import SeparatorConfig, run  # noqa: E402
from paper_1903_03237_b200.synth import baseline_init, make_mixture  # noqa: E402

shapes = [(257, 128, 4, 2, 8, 10), (513, 512, 4, 3, 8, 10), (513, 1024, 8, 4, 16, 10)]
if len(sys.argv) > 6:
    shapes = [tuple(int(v) for v in sys.argv[1:7])]
for F, T, M, N, K, it in shapes:
    X = make_mixture(F, T, M, N, K, seed=0).astype(np.complex64)
    Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, 0)
    out = {"shape": dict(F=F, T=T, M=M, N=N, K=K), "precision": "complex64"}
    for method in ("fast-mnmf", "mnmf"):
        cfg = SeparatorConfig(method=method, n_sources=N, n_basis=K, n_iterations=it,
                              precision="complex64", use_graph=True)
        if method == "mnmf":
            from paper_1903_03237_b200 import fullrank as FR
            init = (FR.reconstruct_scm(Q0, g0), W0, H0)
        else:
            init = (Q0, g0, W0, H0)
        run(cfg, X, init=init)  # warm
        res = run(cfg, X, init=init)
        out[method] = {"s_per_iter_median": float(np.median(res.time_trace[1:])),
                       "ll_final": float(res.likelihood_trace[-1])}
    out["full_over_fast"] = out["mnmf"]["s_per_iter_median"] / out["fast-mnmf"]["s_per_iter_median"]
    print(json.dumps(out), flush=True)
