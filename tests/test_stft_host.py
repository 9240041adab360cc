"""STFT / iSTFT, CPU part: the oracle restatement pinned to
the reference's own outputs (tests/golden/stft.npz, oracle/make_golden.py
--stft-only) and the reference's validation behaviour (stft.py:20-24, 39-42,
63-70, 84-88), which the B200 module raises before touching the device."""

import importlib

import numpy as np
import pytest

from conftest import golden, rel
from oracle import stft_oracle as SO
from paper_1903_03237_b200 import InvalidInputError
ST = importlib.import_module("paper_1903_03237_b200.stft")

G = golden("stft.npz")
TAGS = ["a", "b", "c", "d", "e"]


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_pinned_to_reference(tag):
    n, M, L, hop = (int(v) for v in G[f"{tag}_shape"])
    spec = SO.stft(G[f"{tag}_x"], L, hop)
    assert spec.shape == G[f"{tag}_spec"].shape
    assert rel(spec, G[f"{tag}_spec"]) < 1e-13
    assert rel(SO.istft(G[f"{tag}_spec"], L, hop, length=n), G[f"{tag}_y"]) < 1e-13
    assert rel(SO.istft(G[f"{tag}_spec"], L, hop), G[f"{tag}_yfull"]) < 1e-13
    assert rel(SO.istft(G[f"{tag}_noisy"], L, hop), G[f"{tag}_ynoisy"]) < 1e-13


def test_oracle_mono_and_window():
    assert rel(SO.stft(G["mono_x"], 512, 128), G["mono_spec"]) < 1e-13
    np.testing.assert_allclose(ST.hann_periodic(64), SO.hann_periodic(64), rtol=0, atol=0)


def test_validation_without_gpu():
    with pytest.raises(InvalidInputError, match="power of two"):
        ST.stft(np.zeros((4096, 1)), 1000, 256)
    with pytest.raises(InvalidInputError, match="hop must satisfy"):
        ST.stft(np.zeros((4096, 1)), 1024, 0)
    with pytest.raises(InvalidInputError, match="shorter than one window"):
        ST.stft(np.zeros((512, 1)), 1024, 256)
    with pytest.raises(InvalidInputError, match="bins"):
        ST.istft(np.zeros((100, 5, 1), dtype=complex), 1024, 256)
    with pytest.raises(InvalidInputError, match="exceeds reconstructable"):
        ST.istft(np.zeros((513, 4, 1), dtype=complex), 1024, 256, length=10_000)
