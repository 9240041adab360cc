"""CPU restatement of the reference STFT / iSTFT (fastsep stft.py:15-91) --
TEST INFRASTRUCTURE ONLY (tests/ import it as the checker; the product never
does). Pinned to tests/golden/stft.npz, outputs of the unmodified reference
(oracle/make_golden.py --stft-only)."""

import numpy as np


def hann_periodic(n):
    """stft.py:15-17."""
    return 0.5 - 0.5 * np.cos(2.0 * np.pi * np.arange(n) / n)


def stft(waveform, window_length=1024, hop=256):
    """stft.py:27-48: reflect pad L/2, zero tail to whole frames, Hann, rfft."""
    w = np.asarray(waveform, dtype=np.float64)
    if w.ndim == 1:
        w = w[:, None]
    pad = window_length // 2
    padded = np.pad(w, ((pad, pad), (0, 0)), mode="reflect")
    n_frames = 1 + int(np.ceil((padded.shape[0] - window_length) / hop))
    total = window_length + (n_frames - 1) * hop
    padded = np.pad(padded, ((0, total - padded.shape[0]), (0, 0)))
    idx = np.arange(n_frames)[:, None] * hop + np.arange(window_length)[None, :]
    frames = padded[idx]  # (T, L, M)
    spec = np.fft.rfft(frames * hann_periodic(window_length)[None, :, None], axis=1)
    return np.ascontiguousarray(spec.transpose(1, 0, 2))  # (F, T, M)


def istft(spec, window_length=1024, hop=256, length=None):
    """stft.py:51-91: irfft, window, overlap-add / summed squared window."""
    n_freq, n_frames, M = spec.shape
    window = hann_periodic(window_length)
    frames = np.fft.irfft(spec.transpose(1, 2, 0), n=window_length, axis=-1)  # (T, M, L)
    total = window_length + (n_frames - 1) * hop
    out = np.zeros((total, M))
    norm = np.zeros(total)
    for t in range(n_frames):
        sl = slice(t * hop, t * hop + window_length)
        out[sl] += frames[t].T * window[:, None]
        norm[sl] += window * window
    out /= np.maximum(norm, np.finfo(float).tiny)[:, None]
    pad = window_length // 2
    out = out[pad:-pad] if pad else out
    return out if length is None else out[:length]
