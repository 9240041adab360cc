"""The complex64 V accumulations at M >= 12 -- tensor cores (k_vacc_tc,
FM_VACC=tc) and the register-blocked SIMT default (k_vacc_blk) -- against the
oracle: ragged frame blocks (T not a multiple of the 16-frame chunk or the
128-frame staging block), a padded accumulator tile (M = 12: 144 real rows in
two 128-lane tiles) and the full two-tile case (M = 16). complex64 tolerance
1e-3 (BASELINE north_star), relative Frobenius per tensor and per-entry on the
likelihood trace."""

import numpy as np
import pytest

from conftest import rel
from oracle import fastmnmf_oracle as O
from paper_1903_03237_b200.synth import baseline_init, make_mixture

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["tc", "blk", "simt"])
@pytest.mark.parametrize("M,T", [(12, 301), (16, 200), (16, 517), (10, 130), (14, 256), (16, 2088)])
def test_vacc_tensor_core_vs_oracle(M, T, mode, monkeypatch):
    monkeypatch.setenv("FM_VACC", mode)
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, N, K, seed, it = 6, 3, 4, 11, 4
    X = make_mixture(F, T, M, N, K, seed).astype(np.complex64)
    Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, seed)
    ref = O.run_fastmnmf(X.astype(np.complex128), Q0, g0, W0, H0, it)
    cfg = SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K, n_iterations=it,
                          precision="complex64")
    st = {}

    def snap(i, loop):
        st.update(W=loop.source.W_NFK, H=loop.source.H_NKT, g=loop.spatial.g_NFM,
                  Q=loop.spatial.Q_FMM)

    res = run(cfg, X, init=(Q0, g0, W0, H0), on_iteration=snap)
    tr = ref["likelihood_trace"]
    assert np.max(np.abs(res.likelihood_trace - tr) / np.abs(tr)) <= 1e-3
    for k in ("W", "H", "g", "Q"):
        assert rel(st[k], ref[k]) <= 1e-3, (k, rel(st[k], ref[k]))


@pytest.mark.parametrize("M", list(range(1, 17)))
def test_vacc_blocked_every_m(M, monkeypatch):
    """k_vacc_blk (the complex64 default) for every compiled M: 2x2 blocks with
    a zero pad channel for odd M, m-halves for M > 8, two 256-frame segments
    with a ragged second chunk (T = 300), fused run against the oracle."""
    monkeypatch.setenv("FM_VACC", "blk")
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, T, N, K, seed, it = 5, 300, min(3, max(2, M)), 4, 100 + M, 3
    X = make_mixture(F, T, M, N, K, seed).astype(np.complex64)
    Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, seed)
    ref = O.run_fastmnmf(X.astype(np.complex128), Q0, g0, W0, H0, it)
    cfg = SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K, n_iterations=it,
                          precision="complex64")
    res = run(cfg, X, init=(Q0, g0, W0, H0))
    tr = ref["likelihood_trace"]
    assert np.max(np.abs(res.likelihood_trace - tr) / np.abs(tr)) <= 1e-3
    assert rel(res.images_NFTM, ref["images"]) <= 1e-3
    assert rel(res.loop.spatial.Q_FMM, ref["Q"]) <= 1e-3
