"""End-to-end parity of the fused sm_100a FastMNMF iteration (run()) with the
reference outputs (tests/golden/run_*.npz from the unmodified reference) and
the oracle. Tolerances (BASELINE.json north_star): <= 1e-6 relative in
complex128, <= 1e-3 in complex64, norm-wise per tensor, per-entry on the
likelihood trace."""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import fastmnmf_oracle as O
from paper_1903_03237_b200.synth import baseline_init, make_mixture

pytestmark = pytest.mark.gpu


def _run(G, precision, use_graph=True, **kw):
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, T, M, N, K, seed, it = (int(v) for v in G["shape"])
    X = make_mixture(F, T, M, N, K, seed)
    if precision == "complex64":
        X = X.astype(np.complex64)
    cfg = SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K, n_iterations=it,
                          precision=precision, use_graph=use_graph, **kw)
    state = {}

    def snap(i, loop):
        state.update(W=loop.source.W_NFK, H=loop.source.H_NKT, g=loop.spatial.g_NFM,
                     Q=loop.spatial.Q_FMM)

    res = run(cfg, X, init=baseline_init(F, T, M, N, K, seed),
              on_iteration=snap if kw.pop("_snap", True) else None)
    return res, state, X


def _compare(G, res, state, tol):
    ll = res.likelihood_trace
    assert np.max(np.abs(ll - G["trace"]) / np.abs(G["trace"])) <= tol
    for k in ("W", "H", "g", "Q"):
        assert rel(state[k], G[k]) <= tol, k
    N = G["W"].shape[0]
    if "images" in G:
        assert rel(res.images_NFTM, G["images"]) <= tol
    else:
        assert rel(res.images_NFTM[:, ::17, ::19, :], G["img_sample"]) <= tol
    np.testing.assert_allclose(np.linalg.norm(res.images_NFTM.reshape(N, -1), axis=1),
                               G["img_norm"], rtol=tol)


@pytest.mark.parametrize("name,kw", [
    ("run_small_a.npz", {}), ("run_small_b.npz", {"normalize": False}),
    ("run_small_c.npz", {"ip_sweeps": 2}), ("run_small_d.npz", {}),
])
def test_small_runs_c128(name, kw):
    G = golden(name)
    res, state, _ = _run(G, "complex128", **kw)
    _compare(G, res, state, 1e-8)


def test_config0_c128():
    """BASELINE config 0: F=257 T=128 M=4 N=2 K=8, complex128, 50 iterations."""
    G = golden("run_c0.npz")
    res, state, X = _run(G, "complex128")
    _compare(G, res, state, 1e-6)
    assert np.abs(res.images_NFTM.sum(axis=0) - X).max() < 1e-9  # partition (acceptance 7)


def test_config0_c64():
    G = golden("run_c0_c64.npz")
    res, state, _ = _run(G, "complex64")
    _compare(G, res, state, 1e-3)


def test_config1_c64():
    """BASELINE config 1 shape: F=513 T=1024 M=8 N=4 K=16, complex64, 100 iterations,
    against the reference run on the complex64-rounded mixture."""
    G = golden("run_c1_c64.npz")
    res, state, X = _run(G, "complex64")
    _compare(G, res, state, 1e-3)
    part = np.abs(res.images_NFTM.sum(axis=0) - X.astype(np.complex128)).max()
    assert part < 1e-3 * np.abs(X).max()


def test_graph_equals_eager_and_is_deterministic():
    G = golden("run_small_d.npz")
    a, _, _ = _run(G, "complex64", use_graph=True)
    b, _, _ = _run(G, "complex64", use_graph=False)
    c, _, _ = _run(G, "complex64", use_graph=True)
    np.testing.assert_array_equal(a.likelihood_trace, b.likelihood_trace)
    np.testing.assert_array_equal(a.images_NFTM, c.images_NFTM)  # test_separate.py:132-137


def test_trace_prefix_and_callback():
    # reference test_separate.py:114-122 and :139-146
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, T, M, N, K = 24, 40, 4, 2, 3
    X = make_mixture(F, T, M, N, K, seed=2)
    init = baseline_init(F, T, M, N, K, 3)
    seen = []
    full = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=6), X, init=init,
               on_iteration=lambda it, loop: seen.append(it))
    short = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=3), X, init=init)
    assert seen == list(range(6))
    np.testing.assert_allclose(full.likelihood_trace[:3], short.likelihood_trace, rtol=1e-9)
    assert len(full.time_trace) == 6
    d = np.diff(full.likelihood_trace)
    assert (d < -1e-6 * np.abs(full.likelihood_trace[:-1])).sum() == 0  # monotone


def test_ip_invariant_along_run():
    """Acceptance C6 (test_acceptance.py:203-222): q^H V q = 1 after every iteration."""
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, T, M, N, K = 64, 120, 4, 2, 8
    X = make_mixture(F, T, M, N, K, seed=42)
    worst = [0.0]

    def check(it, loop):
        lam = loop.source.lam()
        y = np.maximum(np.einsum("nft,nfm->ftm", lam, loop.spatial.g_NFM), loop.floor)
        Xs = loop.X
        V = O.ip_weights(Xs, y)
        Q = loop.spatial.Q_FMM
        for m in range(M):
            q = np.conj(Q[:, m, :])
            r = np.einsum("fi,fij,fj->f", q.conj(), V[:, m], q).real
            worst[0] = max(worst[0], float(np.abs(r - 1.0).max()))

    run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=30, seed=7), X,
        init=baseline_init(F, T, M, N, K, 7), on_iteration=check)
    assert worst[0] < 1e-10


def test_default_init_matches_oracle():
    """run() without an injected init: circular init + NmfSource.random from
    the seed, exactly the reference's defaults (separate.py:246-264)."""
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, T, M, N, K = 16, 40, 3, 2, 4
    X = make_mixture(F, T, M, N, K, seed=9)
    res = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=5, seed=4), X)
    Xs = X / np.sqrt(np.mean(np.abs(X) ** 2))
    G1 = np.einsum("fti,ftj->fij", Xs, Xs.conj()) / T
    w, U = np.linalg.eigh(G1)
    Q0 = np.conj(U[..., ::-1].swapaxes(-1, -2))
    g0 = np.full((N, F, M), 1e-2)
    for m in range(M):
        g0[m % N, :, m] = 1.0
    rng = np.random.default_rng(4)
    W0 = rng.uniform(0.1, 1.1, (N, F, K))
    H0 = rng.uniform(0.1, 1.1, (N, K, T))
    ref = O.run_fastmnmf(X, Q0, g0, W0, H0, 5)
    # eigenvector phases are arbitrary; the likelihood and the images are not
    np.testing.assert_allclose(res.likelihood_trace, ref["likelihood_trace"], rtol=1e-8)
    assert rel(res.images_NFTM, ref["images"]) < 1e-8


def test_singular_iteration_prefix():
    from paper_1903_03237_b200 import SeparatorConfig, SingularMatrixError, run
    F, T, M, N, K = 3, 3, 5, 2, 2
    X = make_mixture(F, T, M, N, K, seed=5)
    init = baseline_init(F, T, M, N, K, 5)
    with pytest.raises(O.OracleError) as ref:
        O.run_fastmnmf(X, *init, n_iterations=2)
    with pytest.raises(SingularMatrixError) as got:
        run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=2), X, init=init)
    # same exception class, iteration and row; the failing bin of this
    # rank-deficient (T < M) case depends on rounding in both implementations
    assert str(got.value).startswith("iteration 0: non-positive normalization")
    assert str(ref.value).startswith("iteration 0: non-positive normalization")
    assert "m=0)" in str(got.value)


def test_batch_equals_single_runs():
    """Config-2 style batch: B independent mixtures in one launch sequence ==
    B separate runs (SURVEY §8(a) batching note)."""
    import torch
    from paper_1903_03237_b200 import SeparatorConfig, run, run_batch
    F, T, M, N, K, B, it = 20, 64, 4, 3, 8, 4, 8
    Xs = np.stack([make_mixture(F, T, M, N, K, seed=100 + b) for b in range(B)])
    inits = [baseline_init(F, T, M, N, K, 100 + b) for b in range(B)]
    stacked = tuple(torch.from_numpy(np.stack([i[k] for i in inits])) for k in range(4))
    cfg = SeparatorConfig(n_sources=N, n_basis=K, n_iterations=it, precision="complex64")
    br = run_batch(cfg, Xs.astype(np.complex64), stacked)
    for b in range(B):
        single = run(cfg, Xs[b].astype(np.complex64), init=inits[b])
        np.testing.assert_allclose(br.likelihood_trace[b], single.likelihood_trace, rtol=1e-6)
        assert rel(br.images_BNFTM[b].cpu().numpy(), single.images_NFTM) < 1e-5
        ref = O.run_fastmnmf(Xs[b].astype(np.complex64).astype(np.complex128), *inits[b], it)
        assert rel(single.images_NFTM, ref["images"]) < 1e-3


def test_results_own_their_pinned_images():
    """run() returns images in page-locked blocks of torch's caching host
    allocator: a live result keeps its block (no aliasing by later runs), and
    a freed result's block is recycled without touching live ones."""
    import gc
    from paper_1903_03237_b200 import SeparatorConfig, run
    from paper_1903_03237_b200.synth import baseline_init, make_mixture
    F, T, M, N, K = 9, 40, 3, 2, 3
    cfg = SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K, n_iterations=3,
                          precision="complex64")
    Xa = make_mixture(F, T, M, N, K, seed=1).astype(np.complex64)
    Xb = make_mixture(F, T, M, N, K, seed=2).astype(np.complex64)
    ra = run(cfg, Xa, init=baseline_init(F, T, M, N, K, 1))
    keep = ra.images_NFTM.copy()
    for s in range(3):  # later runs, some results dropped immediately
        rb = run(cfg, Xb, init=baseline_init(F, T, M, N, K, 2))
        del rb
        gc.collect()
    rc = run(cfg, Xb, init=baseline_init(F, T, M, N, K, 2))
    np.testing.assert_array_equal(ra.images_NFTM, keep)
    assert not np.shares_memory(ra.images_NFTM, rc.images_NFTM)
    assert rel(rc.images_NFTM.sum(axis=0), Xb) < 1e-5


@pytest.mark.parametrize("precision", ["complex128", "complex64"])
def test_observation_validation(precision):
    """separate.py:285-291: shape, non-finite and all-zero observations raise
    InvalidInputError with the reference's messages (checked on the device
    statistics, before any iteration)."""
    from paper_1903_03237_b200 import InvalidInputError, SeparatorConfig, run
    cfg = SeparatorConfig(method="fast-mnmf", n_sources=2, n_basis=2, n_iterations=2,
                          precision=precision)
    X = np.ones((4, 16, 2), complex)
    with pytest.raises(InvalidInputError, match="shape"):
        run(cfg, X[0])
    bad = X.copy()
    bad[1, 3, 0] = np.nan
    with pytest.raises(InvalidInputError, match="non-finite"):
        run(cfg, bad)
    with pytest.raises(InvalidInputError, match="identically zero"):
        run(cfg, np.zeros_like(X))
