"""Parity at the full BASELINE shapes of configs 2, 3 and 4 against runs of
the UNMODIFIED reference (tests/golden/run_c{2,3,4}_full.npz, written by
``oracle/make_golden.py --full-c2/--full-c3/--full-c4``), complex64 mode,
tolerance 1e-3 (BASELINE north_star), norm-wise per tensor and per entry on
the likelihood trace. These are the only runs of the K = 32 and N = 6 kernel
instantiations at their production shapes.

* config 2: eight mixtures of the 256-mixture batch (513, 512, 4, 3, 8),
  seeds 0..7, 100 iterations, through ``run_batch`` in one lock-step batch;
* config 3: (1025, 8192, 16, 6, 32), seed 0, 4 iterations (the reference
  takes ~70 s per iteration on the host), through ``run``;
* config 4: FastMNMF-DP (513, 512, 8, noise K = 32, exp-MLP decoder, 10 Adam
  steps), 100 iterations, through ``run``.
"""

import numpy as np
import pytest

from conftest import golden, rel
from paper_1903_03237_b200.synth import baseline_init, make_mixture_fast

pytestmark = pytest.mark.gpu
TOL = 1e-3


def _trace_ok(tr, ref):
    return float(np.max(np.abs(tr - ref) / np.abs(ref)))


def test_config2_batch_full_shape():
    import torch

    from paper_1903_03237_b200 import SeparatorConfig, run_batch

    G = golden("run_c2_full.npz")
    F, T, M, N, K, _, it, nmix = (int(v) for v in G["shape"])
    X = np.stack([make_mixture_fast(F, T, M, N, K, seed=b) for b in range(nmix)])
    for b in range(nmix):
        assert abs(np.abs(X[b].astype(np.complex128)).sum() / G[f"b{b}_X_abs_sum"] - 1) < 1e-6
    inits = [baseline_init(F, T, M, N, K, b) for b in range(nmix)]
    init = tuple(torch.from_numpy(np.stack([i[k] for i in inits])) for k in range(4))
    cfg = SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K, n_iterations=it,
                          precision="complex64")
    res = run_batch(cfg, X, init)
    loop = res.loop
    for b in range(nmix):
        p = f"b{b}_"
        assert _trace_ok(res.likelihood_trace[b], G[p + "trace"]) <= TOL, b
        for k, t in (("W", loop.W), ("H", loop.H), ("g", loop.g), ("Q", loop.Q)):
            assert rel(t[b].cpu().numpy(), G[p + k]) <= TOL, (b, k)
        img = res.images_BNFTM[b]
        assert rel(img[:, ::17, ::19, :].cpu().numpy(), G[p + "img_sample"]) <= TOL, b
        nrm = torch.linalg.vector_norm(img.reshape(N, -1), dim=1).cpu().numpy()
        np.testing.assert_allclose(nrm, G[p + "img_norm"], rtol=TOL)


def test_config3_full_shape():
    from paper_1903_03237_b200 import SeparatorConfig, run

    G = golden("run_c3_full.npz")
    F, T, M, N, K, seed, it = (int(v) for v in G["shape"])
    X = make_mixture_fast(F, T, M, N, K, seed=seed)
    assert rel(X[::64, ::97, :], G["X_sample"]) < 1e-6  # same mixture as the golden's
    st = {}

    def snap(i, loop):
        if i == it - 1:
            st.update(W=loop.source.W_NFK, H=loop.source.H_NKT, g=loop.spatial.g_NFM,
                      Q=loop.spatial.Q_FMM)

    cfg = SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K, n_iterations=it,
                          precision="complex64")
    res = run(cfg, X, init=baseline_init(F, T, M, N, K, seed), on_iteration=snap)
    assert _trace_ok(res.likelihood_trace, G["trace"]) <= TOL
    for k in ("W", "H", "g", "Q"):
        assert rel(st[k], G[k]) <= TOL, (k, rel(st[k], G[k]))
    img = res.images_NFTM
    assert rel(img[:, ::64, ::97, :], G["img_sample"]) <= TOL
    np.testing.assert_allclose(np.linalg.norm(img.reshape(N, -1), axis=1), G["img_norm"],
                               rtol=TOL)
    # partition: the images sum back to the mixture (acceptance criterion 7)
    part = img[:, ::7].sum(axis=0) - X[::7]
    assert np.abs(part).max() <= 1e-3 * np.abs(X).max()


def test_config4_full_shape():
    from oracle import fastmnmf_dp_oracle as DO
    from paper_1903_03237_b200 import SeparatorConfig, run
    from paper_1903_03237_b200.dp import ExpMLPDecoder

    G = golden("run_c4_full.npz")
    F, T, M, K, seed, it, steps = (int(v) for v in G["shape"])
    dec = ExpMLPDecoder(F, seed=seed)
    X = DO.make_dp_mixture(F, T, M, K, DO.ExpMLPDecoder(F, seed=seed), seed=seed).astype(np.complex64)
    assert abs(np.abs(X.astype(np.complex128)).sum() / G["X_abs_sum"] - 1) < 1e-6
    cfg = SeparatorConfig(method="fast-mnmf-dp", n_sources=2, n_basis=K, n_iterations=it,
                          decoder=dec, adam_steps=steps, metropolis_enabled=True,
                          precision="complex64")
    st = {}

    def snap(i, loop):
        if i == it - 1:
            st.update(W=loop.source.W_NFK, H=loop.source.H_NKT, g=loop.spatial.g_NFM,
                      Q=loop.spatial.Q_FMM, u=loop.dp.u[0].cpu().numpy(),
                      v=loop.dp.v[0].cpu().numpy(), z=loop.dp.z[0].cpu().numpy())

    res = run(cfg, X, init=DO.dp_init(F, T, M, K, dec.latent_dim, seed), on_iteration=snap)
    assert _trace_ok(res.likelihood_trace, G["trace"]) <= TOL
    for k in ("u", "v", "z", "W", "H", "g", "Q"):
        assert rel(st[k], G[k]) <= TOL, (k, rel(st[k], G[k]))
    assert rel(res.images_NFTM[:, ::17, ::19, :], G["img_sample"]) <= TOL
    np.testing.assert_allclose(np.linalg.norm(res.images_NFTM.reshape(2, -1), axis=1),
                               G["img_norm"], rtol=TOL)
