"""One c1 run() (2 iterations) so ncu can capture the separate entry point
(k_wiener, separate.py:110-125 via loop.images())."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_1903_03237_b200 import SeparatorConfig, run
from paper_1903_03237_b200.synth import baseline_init, make_mixture
F, T, M, N, K = 513, 1024, 8, 4, 16
X = make_mixture(F, T, M, N, K, 0).astype(np.complex64)
res = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=2, precision="complex64"), X,
          init=baseline_init(F, T, M, N, K, 0))
print(res.images_NFTM.shape)
