"""Debug: one shape, both schedules, vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle import fastmnmf_oracle as O
from paper_1903_03237_b200 import SeparatorConfig, run
from paper_1903_03237_b200.synth import baseline_init, make_mixture
F, T, M, N, K, it = [int(v) for v in sys.argv[1:7]]
prec = sys.argv[7] if len(sys.argv) > 7 else "complex64"
X = make_mixture(F, T, M, N, K, 21)
if prec == "complex64":
    X = X.astype(np.complex64)
init = baseline_init(F, T, M, N, K, 21)
ref = O.run_fastmnmf(X.astype(np.complex128), *init, n_iterations=it)
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
for sch in ("split", "fused"):
    os.environ["FM_SCHEDULE"] = sch
    st = []
    res = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=it, precision=prec), X, init=init,
              on_iteration=lambda i, l: st.append((l.source.W_NFK, l.source.H_NKT, l.spatial.g_NFM)))
    tr = ref["likelihood_trace"]
    print(sch, "trace", np.abs(res.likelihood_trace - tr) / np.abs(tr))
    for i, (W, H, g) in enumerate(st):
        print("  it", i, "W", rel(W, ref["W"]) if i == it - 1 else "", "H", rel(H, ref["H"]) if i == it - 1 else "",
              np.isfinite(W).all(), np.isfinite(H).all(), np.abs(H).max())
