"""Host-side logic of the drop-in API (CPU only)."""

import numpy as np
import pytest

from paper_1903_03237_b200 import InvalidInputError, SeparatorConfig
from paper_1903_03237_b200 import kernels as K


class TestConfig:  # mirrors reference tests/test_separate.py:17-32
    def test_zero_iterations_forbidden(self):
        with pytest.raises(InvalidInputError):
            SeparatorConfig(method="fca", n_iterations=0).validate()

    def test_unknown_method(self):
        with pytest.raises(InvalidInputError):
            SeparatorConfig(method="ilrma").validate()

    def test_zero_sources(self):
        with pytest.raises(InvalidInputError):
            SeparatorConfig(method="fca", n_sources=0).validate()

    def test_dp_needs_two_sources(self):
        with pytest.raises(InvalidInputError):
            SeparatorConfig(method="mnmf-dp", n_sources=1).validate()

    def test_precision_field(self):
        SeparatorConfig(precision="complex64").validate()
        with pytest.raises(InvalidInputError):
            SeparatorConfig(precision="bfloat16").validate()


def test_status_decoding_and_messages():
    assert K.decode_status(-1) is None
    key = (7 << 44) | (3 << 24) | (123 << 2) | 1
    code, it, m, f = K.decode_status(key)
    assert (code, it, m, f) == (1, 7, 3, 123)
    assert K.status_message(1, 3, 123) == (
        "non-positive normalization in diagonalizer update at (f=123, m=3)")
    assert K.status_message(2, 2, 0).startswith("singular Q V in diagonalizer update at row m=2")


def test_dp_latent_options_validated():
    SeparatorConfig(method="fast-mnmf-dp", latent_update="metropolis",
                    metropolis_rng="device").validate()
    with pytest.raises(InvalidInputError):
        SeparatorConfig(method="fast-mnmf-dp", latent_update="langevin").validate()
    with pytest.raises(InvalidInputError):
        SeparatorConfig(method="fast-mnmf-dp", metropolis_rng="mt19937").validate()


def test_methods_outside_the_backend_raise_before_device_work():
    """FCA / FastFCA / MNMF-DP are not built: run() refuses them
    with the reference's error type before touching the GPU."""
    from paper_1903_03237_b200 import run
    for method in ("fca", "fast-fca", "mnmf-dp"):
        with pytest.raises(InvalidInputError, match="outside this backend"):
            run(SeparatorConfig(method=method, n_sources=2), np.ones((4, 8, 2), complex))


def test_toy_decoder_matches_reference_construction():
    """Same seeded draws and shapes as the reference ToyDecoder (sources.py:52-68)."""
    from paper_1903_03237_b200 import ToyDecoder
    d = ToyDecoder(33, latent_dim=16, hidden=64, seed=0)
    rng = np.random.default_rng(0)
    np.testing.assert_array_equal(d.w1, rng.normal(0.0, 1.0 / np.sqrt(16), (64, 16)))
    np.testing.assert_array_equal(d.b1, rng.normal(0.0, 0.5, 64))
    assert d.latent_dim == 16 and d.n_freq == 33
    assert np.all(d(np.zeros((3, 16))) >= 1e-8)
