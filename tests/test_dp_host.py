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


def test_toy_decoder_matches_oracle_restatement():
    from paper_1903_03237_b200 import ToyDecoder
    a, b = ToyDecoder(29), DO.ToyDecoder(29)
    z = np.random.default_rng(4).standard_normal((7, 16))
    np.testing.assert_array_equal(a(z), b(z))


def test_metropolis_oracle_pinned_to_reference():
    """The restated Metropolis chain (MetropolisLatents, sources.py:307-339)
    reproduces the unmodified reference's default FastMNMF-DP run (ToyDecoder,
    30 proposals per iteration, the run's numpy stream)."""
    G = golden("run_dp_mh.npz")
    F, T, M, K, seed, it = (int(v) for v in G["shape"])
    dec = DO.ToyDecoder(F)
    X = G["X"].astype(np.complex128)
    hook = DO.MetropolisLatents(np.random.default_rng(seed))
    out = DO.run_fastmnmf_dp(X, *DO.dp_init(F, T, M, K, dec.latent_dim, seed), dec, it,
                             adam_steps=0, hook=hook)
    np.testing.assert_allclose(out["likelihood_trace"], G["trace"], rtol=1e-12)
    for k in ("u", "v", "z", "W", "H", "g", "Q"):
        assert rel(out[k], G[k]) < 1e-12, k
    assert rel(out["images"], G["images"]) < 1e-12
