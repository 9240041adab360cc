"""Debug: small plain run vs the oracle, trace and state errors per iteration."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle.fastmnmf_oracle import run_fastmnmf
from paper_1903_03237_b200 import SeparatorConfig, run
from paper_1903_03237_b200.synth import baseline_init, make_mixture
F, T, M, N, K, seed, it = [int(v) for v in (sys.argv[1:] or [33, 96, 4, 3, 4, 5, 4])]
prec = os.environ.get("PREC", "complex128")
X = make_mixture(F, T, M, N, K, seed)
init = baseline_init(F, T, M, N, K, seed)
ref = run_fastmnmf(X, *init, n_iterations=it)
cfg = SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K, n_iterations=it, precision=prec)
st = []
def snap(i, loop):
    st.append(dict(W=loop.source.W_NFK, H=loop.source.H_NKT, g=loop.spatial.g_NFM, Q=loop.spatial.Q_FMM))
res = run(cfg, X, init=init, on_iteration=snap)
print("trace dev", res.likelihood_trace)
print("trace ref", ref["likelihood_trace"])
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
for k in ("W", "H", "g", "Q"):
    print(k, rel(st[-1][k], ref[k]))
