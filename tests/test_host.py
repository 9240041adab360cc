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
