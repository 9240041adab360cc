"""STFT / iSTFT on the device (k_stft / k_istft_frames / k_ola) against the
reference's outputs (tests/golden/stft.npz) and the pinned oracle: float64
(numpy in / out) at 1e-12, float32 device tensors at 1e-5 (relative
Frobenius), plus the reference tests' properties (round trip, zeros,
mono input, no-overlap hop = window_length)."""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import stft_oracle as SO

pytestmark = pytest.mark.gpu
G = golden("stft.npz")
TAGS = ["a", "b", "c", "d", "e"]


@pytest.mark.parametrize("tag", TAGS)
def test_stft_istft_vs_reference(tag):
    from paper_1903_03237_b200 import istft, stft
    n, M, L, hop = (int(v) for v in G[f"{tag}_shape"])
    spec = stft(G[f"{tag}_x"], L, hop)
    assert spec.dtype == np.complex128 and spec.shape == G[f"{tag}_spec"].shape
    assert rel(spec, G[f"{tag}_spec"]) < 1e-12
    y = istft(G[f"{tag}_spec"], L, hop, length=n)
    assert y.shape == (n, M) and rel(y, G[f"{tag}_y"]) < 1e-12
    assert rel(istft(G[f"{tag}_spec"], L, hop), G[f"{tag}_yfull"]) < 1e-12
    assert rel(istft(G[f"{tag}_noisy"], L, hop), G[f"{tag}_ynoisy"]) < 1e-12


@pytest.mark.parametrize("tag", TAGS)
def test_stft_float32_device(tag):
    import torch
    from paper_1903_03237_b200 import istft, stft
    n, M, L, hop = (int(v) for v in G[f"{tag}_shape"])
    x = torch.from_numpy(G[f"{tag}_x"].astype(np.float32)).cuda()
    spec = stft(x, L, hop)
    assert spec.is_cuda and spec.dtype == torch.complex64
    assert rel(spec.cpu().numpy(), G[f"{tag}_spec"]) < 1e-5
    y = istft(spec, L, hop, length=n)
    assert y.dtype == torch.float32
    if hop <= L // 2:  # COLA; with hop = L the summed window nears 0 at frame edges
        assert rel(y.cpu().numpy(), G[f"{tag}_y"]) < 1e-5


def test_mono_zero_and_round_trip():
    from paper_1903_03237_b200 import istft, stft
    assert rel(stft(G["mono_x"], 512, 128), G["mono_spec"]) < 1e-12
    assert np.abs(stft(np.zeros((3000, 2)), 1024, 256)).max() == 0.0  # test_stft.py:18
    assert np.abs(istft(np.zeros((513, 10, 2), dtype=complex), 1024, 256)).max() == 0.0
    x = np.random.default_rng(5).standard_normal((10_000, 3))  # test_stft.py:57-60
    y = istft(stft(x, 1024, 256), 1024, 256, length=x.shape[0])
    assert np.max(np.abs(y - x)) < 1e-10


def test_large_window_and_many_channels():
    """n_fft 2048 (config 3's front end), 16 channels (two channel groups in
    float64), against the oracle."""
    from paper_1903_03237_b200 import istft, stft
    x = np.random.default_rng(9).standard_normal((20_000, 16))
    spec = stft(x, 2048, 512)
    assert rel(spec, SO.stft(x, 2048, 512)) < 1e-12
    assert rel(istft(spec, 2048, 512, length=20_000), x) < 1e-12
