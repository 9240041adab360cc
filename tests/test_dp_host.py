"""FastMNMF-DP host pieces (CPU): decoder init, generator and init agree
with the oracle; the oracle is pinned to the reference loop (goldens made by
running the unmodified reference with this decoder and the Adam hook)."""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import fastmnmf_dp_oracle as DO
from paper_1903_03237_b200.dp import ExpMLPDecoder
from paper_1903_03237_b200.synth import dp_init, make_dp_mixture


def test_decoder_matches_oracle():
    a, b = ExpMLPDecoder(37, seed=3), DO.ExpMLPDecoder(37, seed=3)
    for k in ("W1", "W2", "W3", "b1", "b2", "b3"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
    z = np.random.default_rng(1).standard_normal((5, 16))
    np.testing.assert_allclose(a(z), b(z), rtol=1e-14)
    assert (a.latent_dim, a.hidden, a.n_freq) == (16, 128, 37)


def test_generator_and_init_match_oracle():
    dec = ExpMLPDecoder(11, seed=2)
    np.testing.assert_array_equal(make_dp_mixture(11, 20, 3, 4, dec, 2),
                                  DO.make_dp_mixture(11, 20, 3, 4, dec, 2))
    for x, y in zip(dp_init(11, 20, 3, 4, 16, 2), DO.dp_init(11, 20, 3, 4, 16, 2)):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("name,steps", [("run_dp_mu.npz", 0), ("run_dp_adam.npz", 10)])
def test_dp_oracle_pinned_to_reference(name, steps):
    G = golden(name)
    F, T, M, K, seed, it, _ = (int(v) for v in G["shape"])
    dec = DO.ExpMLPDecoder(F, seed=seed)
    X = DO.make_dp_mixture(F, T, M, K, dec, seed=seed).astype(np.complex64).astype(np.complex128)
    out = DO.run_fastmnmf_dp(X, *DO.dp_init(F, T, M, K, dec.latent_dim, seed), dec, it,
                             adam_steps=steps)
    np.testing.assert_allclose(out["likelihood_trace"], G["trace"], rtol=1e-12)
    for k in ("u", "v", "W", "H", "g", "Q"):
        assert rel(out[k], G[k]) < 1e-12, k
    if steps:
        assert rel(out["z"], G["z"]) < 1e-12
    assert rel(out["images"], G["images"]) < 1e-12
