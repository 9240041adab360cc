"""The reference's default FastMNMF-DP latent path on the GPU:
its ToyDecoder and its Metropolis chain (update_latents_fast,
sources.py:307-339) in k_dp_mh, against tests/golden/run_dp_mh.npz -- a run of
the UNMODIFIED reference (oracle/make_golden.py) -- and the restated oracle.

With the reference's numpy draws (metropolis_rng="numpy") every accept /
reject decision is the reference's, so the whole run matches at the north_star
tolerances: complex128 <= 1e-6, complex64 <= 1e-3 (relative Frobenius per
tensor, per entry on the trace)."""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import fastmnmf_dp_oracle as DO

pytestmark = pytest.mark.gpu


def _snap(st):
    def snap(i, loop):
        st.update(W=loop.source.W_NFK, H=loop.source.H_NKT, g=loop.spatial.g_NFM,
                  Q=loop.spatial.Q_FMM, u=loop.dp.u[0].cpu().numpy(),
                  v=loop.dp.v[0].cpu().numpy(), z=loop.dp.z[0].cpu().numpy(),
                  r=loop.dp.r[0].cpu().numpy())
    return snap


@pytest.mark.parametrize("precision,tol", [("complex128", 1e-6), ("complex64", 1e-3)])
def test_metropolis_default_path_vs_reference(precision, tol):
    from paper_1903_03237_b200 import SeparatorConfig, run
    G = golden("run_dp_mh.npz")
    F, T, M, K, seed, it = (int(v) for v in G["shape"])
    X = G["X"] if precision == "complex64" else G["X"].astype(np.complex128)
    # decoder=None -> the reference default ToyDecoder(F); latent_update auto ->
    # Metropolis; the chain draws from default_rng(seed) as the reference's does
    cfg = SeparatorConfig(method="fast-mnmf-dp", n_sources=2, n_basis=K, n_iterations=it,
                          seed=seed, precision=precision)
    st = {}
    res = run(cfg, X, init=DO.dp_init(F, T, M, K, 16, seed), on_iteration=_snap(st))
    assert np.max(np.abs(res.likelihood_trace - G["trace"]) / np.abs(G["trace"])) <= tol
    for k in ("u", "v", "z", "W", "H", "g", "Q"):
        assert rel(st[k], G[k]) <= tol, (k, rel(st[k], G[k]))
    assert rel(res.images_NFTM, G["images"]) <= tol


@pytest.mark.parametrize("F,T,M,N", [(21, 37, 3, 2), (40, 66, 8, 3)])
def test_metropolis_ragged_vs_oracle(F, T, M, N):
    """Ragged frame counts (T % fpb != 0), N = 3 (y_rest over two NMF
    sources), non-default proposal settings; complex128 against the oracle."""
    from paper_1903_03237_b200 import MetropolisConfig, SeparatorConfig, ToyDecoder, run
    from paper_1903_03237_b200.synth import baseline_init, make_mixture
    seed, K, it = 7, 4, 3
    X = make_mixture(F, T, M, N, K, seed)
    Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, seed)
    u0, v0, z0 = np.ones(F), np.ones(T), np.zeros((T, 16))
    dec = ToyDecoder(F, seed=3)
    mc = MetropolisConfig(proposal_var=4e-4, inner_steps=7)
    cfg = SeparatorConfig(method="fast-mnmf-dp", n_sources=N, n_basis=K, n_iterations=it,
                          seed=seed, decoder=dec, metropolis=mc, precision="complex128")
    st = {}
    res = run(cfg, X, init=(Q0, g0, u0, v0, z0, W0[1:], H0[1:]), on_iteration=_snap(st))
    hook = DO.MetropolisLatents(np.random.default_rng(seed), 7, 4e-4)
    ref = DO.run_fastmnmf_dp(X, Q0, g0, u0, v0, z0, W0[1:], H0[1:], DO.ToyDecoder(F, seed=3), it,
                             adam_steps=0, hook=hook)
    assert np.max(np.abs(res.likelihood_trace - ref["likelihood_trace"])
                  / np.abs(ref["likelihood_trace"])) <= 1e-8
    for k in ("u", "v", "z", "W", "H", "g", "Q"):
        assert rel(st[k], ref[k]) <= 1e-8, (k, rel(st[k], ref[k]))
    assert rel(res.images_NFTM, ref["images"]) <= 1e-8


def test_toy_refresh_only_vs_oracle():
    """metropolis_enabled=False: the decoder refresh alone (k_dp_mh, 0 steps)."""
    from paper_1903_03237_b200 import SeparatorConfig, run
    G = golden("run_dp_mh.npz")
    F, T, M, K, seed, _ = (int(v) for v in G["shape"])
    X = G["X"].astype(np.complex128)
    init = DO.dp_init(F, T, M, K, 16, seed)
    z0 = np.random.default_rng(1).standard_normal((T, 16)) * 0.3
    init = init[:4] + (z0,) + init[5:]
    cfg = SeparatorConfig(method="fast-mnmf-dp", n_sources=2, n_basis=K, n_iterations=3,
                          seed=seed, metropolis_enabled=False, precision="complex128")
    res = run(cfg, X, init=init)
    ref = DO.run_fastmnmf_dp(X, *init, DO.ToyDecoder(F), 3, adam_steps=0)
    assert rel(res.images_NFTM, ref["images"]) <= 1e-8
    np.testing.assert_allclose(res.likelihood_trace, ref["likelihood_trace"], rtol=1e-8)


@pytest.mark.parametrize("precision", ["complex128", "complex64"])
def test_metropolis_device_rng(precision):
    """metropolis_rng="device" (Philox): deterministic reruns, proposals accepted,
    and a likelihood close to the numpy-stream run's (same chain law)."""
    from paper_1903_03237_b200 import SeparatorConfig, run
    G = golden("run_dp_mh.npz")
    F, T, M, K, seed, it = (int(v) for v in G["shape"])
    X = G["X"] if precision == "complex64" else G["X"].astype(np.complex128)
    cfg = SeparatorConfig(method="fast-mnmf-dp", n_sources=2, n_basis=K, n_iterations=it,
                          seed=seed, precision=precision, metropolis_rng="device")
    outs = []
    for _ in range(2):
        st = {}
        res = run(cfg, X, init=DO.dp_init(F, T, M, K, 16, seed), on_iteration=_snap(st))
        outs.append((res, st))
    (r1, s1), (r2, s2) = outs
    np.testing.assert_array_equal(r1.likelihood_trace, r2.likelihood_trace)
    np.testing.assert_array_equal(s1["z"], s2["z"])
    moved = np.abs(s1["z"]).sum(axis=1) > 0
    assert moved.mean() > 0.5
    assert np.all(np.isfinite(r1.images_NFTM))
    assert abs(r1.likelihood_trace[-1] - G["trace"][-1]) <= 0.05 * abs(G["trace"][-1])
