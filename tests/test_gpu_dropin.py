"""The reference loop surface and the reference's own run()-level tests,
against this package imported as ``fastsep`` (compat.install_fastsep_alias).

The bodies restate the reference tests they cite (pkg/tests/...; the
reference tree does not exist on the GPU box) with the reference's
thresholds; mixtures come from the BASELINE generator instead of the
reference conftest's ``sampled_mixture`` (its full-rank sampler is outside
the hot path)."""

import numpy as np
import pytest

from oracle import fastmnmf_oracle as O
from paper_1903_03237_b200.synth import baseline_init, make_mixture

pytestmark = pytest.mark.gpu


@pytest.fixture
def fastsep():
    from paper_1903_03237_b200.compat import install_fastsep_alias, uninstall_fastsep_alias

    mod = install_fastsep_alias()
    yield mod
    uninstall_fastsep_alias()


def test_criterion_6_ip_normalization_invariant(fastsep):
    """test_acceptance.py:203-222: max |q^H V q - 1| < 1e-10 over a
    30-iteration run, read through loop.X, loop.floor, loop.spatial,
    loop.source.lam() and fastsep._kernels.ip_weights."""
    from fastsep import SeparatorConfig, run
    from fastsep._kernels import ip_weights

    X = make_mixture(64, 120, 4, 2, 8, seed=42)
    worst = {"value": 0.0}

    def check(it, loop):
        lam = loop.source.lam()
        y = np.einsum("nft,nfm->ftm", lam, loop.spatial.g_NFM)
        np.maximum(y, loop.floor, out=y)
        V = ip_weights(loop.X, y)
        for m in range(loop.X.shape[-1]):
            q = np.conj(loop.spatial.Q_FMM[:, m, :])
            r = np.einsum("fi,fij,fj->f", q.conj(), V[:, m], q).real
            worst["value"] = max(worst["value"], float(np.abs(r - 1.0).max()))

    cfg = SeparatorConfig(method="fast-mnmf", n_sources=2, n_basis=8, n_iterations=30, seed=7)
    run(cfg, X, on_iteration=check)
    assert worst["value"] < 1e-10


class TestRun:
    """test_separate.py:100-146 (the fast-mnmf cases)."""

    def test_trace_lengths_match_iterations(self, fastsep):
        X = make_mixture(32, 60, 4, 2, 3, seed=1)
        res = fastsep.run(fastsep.SeparatorConfig(method="fast-mnmf", n_basis=3, n_iterations=7,
                                                  seed=0), X)
        assert len(res.likelihood_trace) == 7
        assert len(res.time_trace) == 7

    def test_trace_entries_are_post_update_values(self, fastsep):
        X = make_mixture(32, 60, 4, 2, 3, seed=2)
        full = fastsep.run(fastsep.SeparatorConfig(method="fast-mnmf", n_basis=3, n_iterations=6,
                                                   seed=3), X)
        short = fastsep.run(fastsep.SeparatorConfig(method="fast-mnmf", n_basis=3, n_iterations=3,
                                                    seed=3), X)
        np.testing.assert_allclose(full.likelihood_trace[:3], short.likelihood_trace, rtol=1e-9)

    def test_record_likelihood_off(self, fastsep):
        X = make_mixture(32, 60, 4, 2, 3, seed=3)
        res = fastsep.run(fastsep.SeparatorConfig(method="fast-mnmf", n_iterations=2, seed=0,
                                                  record_likelihood=False), X)
        assert res.likelihood_trace.size == 0
        assert len(res.time_trace) == 2

    def test_deterministic_given_seed(self, fastsep):
        X = make_mixture(32, 60, 4, 2, 3, seed=4)
        cfg = fastsep.SeparatorConfig(method="fast-mnmf", n_basis=3, n_iterations=3, seed=11)
        a = fastsep.run(cfg, X)
        b = fastsep.run(cfg, X)
        np.testing.assert_array_equal(a.images_NFTM, b.images_NFTM)
        np.testing.assert_array_equal(a.likelihood_trace, b.likelihood_trace)

    def test_callback_invoked_every_iteration(self, fastsep):
        X = make_mixture(32, 60, 4, 2, 3, seed=5)
        seen = []
        fastsep.run(fastsep.SeparatorConfig(method="fast-mnmf", n_iterations=4, seed=0), X,
                    on_iteration=lambda it, loop: seen.append(it))
        assert seen == [0, 1, 2, 3]


def test_loop_surface_drives_like_the_reference(fastsep):
    """Drive the loop object by hand as run() does (separate.py:303-323):
    iterate(cfg, rng) returns the first refresh's data term, trace entry
    it-1 = that + the pending logdet_term(), the last entry = loglik(), and
    images() is the scaled-domain Wiener output -- against the oracle."""
    import torch

    from paper_1903_03237_b200.separate import DeviceLoop

    F, T, M, N, K, it = 24, 50, 4, 2, 5, 6
    X = make_mixture(F, T, M, N, K, seed=9)
    Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, 9)
    ref = O.run_fastmnmf(X, Q0, g0, W0, H0, n_iterations=it)
    scale = np.sqrt(np.mean(np.abs(X) ** 2))
    Xs = X / scale
    floor = 1e-12 * np.max(np.abs(Xs) ** 2)
    dev = lambda a: torch.from_numpy(np.asarray(a)).cuda().unsqueeze(0)  # noqa: E731
    loop = DeviceLoop(dev(Xs), dev(Q0), dev(g0), dev(W0), dev(H0),
                      torch.tensor([floor], dtype=torch.float64))
    cfg = fastsep.SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K, n_iterations=it)
    rng = np.random.default_rng(0)
    trace, pending = [], None
    for i in range(it):
        ll_before = loop.iterate(cfg, rng)
        if i > 0:
            trace.append(ll_before + pending)
        pending = loop.logdet_term()
    trace.append(loop.loglik())
    np.testing.assert_allclose(trace, ref["likelihood_trace"], rtol=1e-9)
    assert np.abs(loop.X - Xs).max() < 1e-14 and loop.floor == pytest.approx(floor, rel=1e-15)
    assert np.abs(loop.xt - O.project_power(loop.spatial.Q_FMM, Xs)).max() < 1e-9 * loop.xt.max()
    img = loop.images() * scale
    assert np.linalg.norm(img - ref["images"]) / np.linalg.norm(ref["images"]) < 1e-9
    # assignment uploads (the reference's iterate assigns spatial/source fields)
    loop.spatial.g_NFM = np.ones((N, F, M))
    assert np.all(loop.spatial.g_NFM == 1.0)


def test_run_leaves_device_input_unchanged(fastsep):
    """run() on a contiguous CUDA tensor of the run's precision
    must not scale the caller's tensor (separate.py:293 builds Xs = X/scale)."""
    import torch

    X = make_mixture(20, 40, 3, 2, 3, seed=6)
    Xd = torch.from_numpy(X).cuda()
    before = Xd.clone()
    cfg = fastsep.SeparatorConfig(method="fast-mnmf", n_basis=3, n_iterations=3, seed=1)
    a = fastsep.run(cfg, Xd)
    assert torch.equal(Xd, before)
    b = fastsep.run(cfg, Xd)
    np.testing.assert_array_equal(a.images_NFTM, b.images_NFTM)
    assert np.abs(a.images_NFTM.sum(axis=0) - X).max() < 1e-9 * np.abs(X).max()


def test_run_batch_rejects_other_methods(fastsep):
    from paper_1903_03237_b200 import InvalidInputError, run_batch

    X = make_mixture(8, 20, 2, 2, 2, seed=1)[None]
    init = baseline_init(8, 20, 2, 2, 2, 1)
    for method in ("mnmf", "fast-mnmf-dp"):
        with pytest.raises(InvalidInputError):
            run_batch(fastsep.SeparatorConfig(method=method, n_sources=2, n_basis=2, n_iterations=1),
                      X, init)
