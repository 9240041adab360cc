"""FastMNMF-DP (config 4) on the GPU vs the reference-pinned goldens.
complex128: <= 1e-6; complex64: <= 1e-3 (BASELINE north_star tolerances)."""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import fastmnmf_dp_oracle as DO

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["run_dp_mu.npz", "run_dp_adam.npz"])
@pytest.mark.parametrize("precision,tol", [("complex128", 1e-6), ("complex64", 1e-3)])
def test_dp_run(name, precision, tol):
    from paper_1903_03237_b200 import SeparatorConfig, run
    from paper_1903_03237_b200.dp import ExpMLPDecoder
    G = golden(name)
    F, T, M, K, seed, it, steps = (int(v) for v in G["shape"])
    dec = ExpMLPDecoder(F, seed=seed)
    X = DO.make_dp_mixture(F, T, M, K, dec, seed=seed).astype(np.complex64)
    if precision == "complex128":
        X = X.astype(np.complex128)
    cfg = SeparatorConfig(method="fast-mnmf-dp", n_sources=2, n_basis=K, n_iterations=it,
                          decoder=dec, adam_steps=steps, metropolis_enabled=steps > 0,
                          precision=precision)
    st = {}

    def snap(i, loop):
        st.update(W=loop.source.W_NFK, H=loop.source.H_NKT, g=loop.spatial.g_NFM,
                  Q=loop.spatial.Q_FMM, u=loop.dp.u[0].cpu().numpy(), v=loop.dp.v[0].cpu().numpy(),
                  z=loop.dp.z[0].cpu().numpy())

    res = run(cfg, X, init=DO.dp_init(F, T, M, K, dec.latent_dim, seed), on_iteration=snap)
    assert np.max(np.abs(res.likelihood_trace - G["trace"]) / np.abs(G["trace"])) <= tol
    for k in ("u", "v", "W", "H", "g", "Q"):
        assert rel(st[k], G[k]) <= tol, (k, rel(st[k], G[k]))
    if steps:
        assert rel(st["z"], G["z"]) <= tol
    assert rel(res.images_NFTM, G["images"]) <= tol


@pytest.mark.parametrize("precision,tol", [("complex128", 1e-6), ("complex64", 1e-3)])
@pytest.mark.parametrize("F,T,M", [(45, 37, 3), (70, 130, 8)])
def test_dp_ragged_vs_oracle(F, T, M, precision, tol):
    """Ragged frame tiles (T % 4 != 0), partial weight chunks (F % 32 != 0) and
    the scalar x~ staging path (M = 3) of the one-launch latent kernel."""
    from paper_1903_03237_b200 import SeparatorConfig, run
    from paper_1903_03237_b200.dp import ExpMLPDecoder
    K, seed, it, steps = 4, 7, 3, 4
    dec = ExpMLPDecoder(F, seed=seed)
    odec = DO.ExpMLPDecoder(F, seed=seed)
    X = DO.make_dp_mixture(F, T, M, K, odec, seed=seed).astype(np.complex64).astype(np.complex128)
    init = DO.dp_init(F, T, M, K, dec.latent_dim, seed)
    ref = DO.run_fastmnmf_dp(X, *init, odec, it, adam_steps=steps)
    cfg = SeparatorConfig(method="fast-mnmf-dp", n_sources=2, n_basis=K, n_iterations=it,
                          decoder=dec, adam_steps=steps, metropolis_enabled=True, precision=precision)
    st = {}

    def snap(i, loop):
        st.update(z=loop.dp.z[0].cpu().numpy(), u=loop.dp.u[0].cpu().numpy(),
                  v=loop.dp.v[0].cpu().numpy())

    res = run(cfg, X, init=init, on_iteration=snap)
    assert np.max(np.abs(res.likelihood_trace - ref["likelihood_trace"])
                  / np.abs(ref["likelihood_trace"])) <= tol
    for k in ("z", "u", "v"):
        assert rel(st[k], ref[k]) <= tol, (k, rel(st[k], ref[k]))
    assert rel(res.images_NFTM, ref["images"]) <= tol
