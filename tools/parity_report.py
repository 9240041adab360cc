#!/usr/bin/env python
"""Per-tensor parity of the GPU fused path against the reference goldens
(tests/golden, produced by the unmodified reference). GPU only. Writes a
JSON summary (argv[1], default gpurun_out/parity.json)."""
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_1903_03237_b200 import SeparatorConfig, run  # noqa: E402
from paper_1903_03237_b200.synth import baseline_init, make_mixture  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel()) / np.linalg.norm(np.asarray(b).ravel()))


def case(name, precision):
    G = dict(np.load(os.path.join(REPO, "tests", "golden", name)))
    F, T, M, N, K, seed, it = (int(v) for v in G["shape"])
    X = make_mixture(F, T, M, N, K, seed)
    if precision == "complex64":
        X = X.astype(np.complex64)
    st = {}
    cfg = SeparatorConfig(n_sources=N, n_basis=K, n_iterations=it, precision=precision)
    res = run(cfg, X, init=baseline_init(F, T, M, N, K, seed),
              on_iteration=lambda i, lp: st.update(W=lp.source.W_NFK, H=lp.source.H_NKT,
                                                   g=lp.spatial.g_NFM, Q=lp.spatial.Q_FMM)
              if i == it - 1 else None)
    out = {"case": name, "precision": precision, "shape": [F, T, M, N, K], "iterations": it,
           "trace_max_rel": float(np.max(np.abs(res.likelihood_trace - G["trace"]) / np.abs(G["trace"])))}
    for k in ("W", "H", "g", "Q"):
        out[k] = rel(st[k], G[k])
    img = res.images_NFTM if "images" in G else res.images_NFTM[:, ::17, ::19, :]
    out["images"] = rel(img, G["images"] if "images" in G else G["img_sample"])
    out["partition_max_abs"] = float(np.abs(res.images_NFTM.sum(0) - X).max())
    return out


def main():
    rows = [case("run_c0.npz", "complex128"), case("run_c0_c64.npz", "complex64"),
            case("run_c1_c64.npz", "complex64")]
    for r in rows:
        print(json.dumps(r))
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(REPO, "gpurun_out", "parity.json")
    json.dump(rows, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
