"""The complex64 kernels at M > 8 against the oracle. V accumulation: tensor
cores (k_vacc_tc, the default for even M in 10..16, FM_VACC=tc), the
register-blocked SIMT kernel (k_vacc_blk) and the pair-per-thread one --
ragged frame blocks (T not a multiple of the 16-frame chunk or the 128-frame
staging block, odd T: the scalar lambda path), padded lanes (M < 16), two
segments (T = 2088). Projection (k_back_tc vs k_back) and lambda = W H
(k_lambda_tc vs k_lambda) in every combination. complex64 tolerance 1e-3
(BASELINE north_star), relative Frobenius per tensor and per-entry on the
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


@pytest.mark.parametrize("back", ["tc", "simt"])
@pytest.mark.parametrize("lam", ["tc", "simt"])
@pytest.mark.parametrize("M,T,K", [(16, 300, 8), (12, 517, 16), (9, 130, 8), (13, 257, 32)])
def test_projection_and_lambda_variants(M, T, K, back, lam, monkeypatch):
    """The tensor-core projection (k_back_tc, complex64 M > 8: odd and even M,
    K-padded to 32 real columns, ragged 128-frame tiles, several 256-frame
    slots per segment) and lambda = W H (k_lambda_tc, K in {8, 16, 32}, ragged
    bin tiles) against the SIMT kernels' oracle parity, in every combination."""
    monkeypatch.setenv("FM_BACK", back)
    monkeypatch.setenv("FM_LAMBDA", lam)
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, N, seed, it = 37, 3, 21, 4
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
    assert rel(res.loop.source.W_NFK, ref["W"]) <= 1e-3
    assert rel(res.loop.source.H_NKT, ref["H"]) <= 1e-3


@pytest.mark.parametrize("tb", ["256", "128"])
@pytest.mark.parametrize("M,F,T,N", [(8, 37, 1024, 4), (8, 5, 300, 3), (7, 150, 517, 2), (6, 460, 130, 3),
                                     (5, 3, 1300, 2), (8, 700, 256, 4)])
def test_vacc_persistent_vs_oracle(M, F, T, N, tb, monkeypatch):
    """k_vacc_p (persistent CTAs over (bin, chunk) items, complex64 M = 5..8):
    runs that start and end inside a bin, ragged last chunks, fewer items than
    CTAs (F = 3, 5), more items than CTAs (F = 460, 700), one chunk per bin;
    fused run against the oracle."""
    monkeypatch.setenv("FM_VACC", "p")
    monkeypatch.setenv("FM_VP_TB", tb)
    from paper_1903_03237_b200 import SeparatorConfig, run
    K, seed, it = 4, 300 + M + F, 3
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
    assert rel(res.loop.spatial.g_NFM, ref["g"]) <= 1e-3
