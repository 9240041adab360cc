"""Forward / inverse multichannel STFT on the device (``stft.py:1-91`` of the
reference) -- the front / back end that turns waveforms into
the (F, T, M) observation ``run`` separates and the separated images back
into waveforms.

Same signatures, defaults, validation and error messages as the reference:
``stft(waveform (n_samples, n_channels) or (n_samples,), window_length=1024,
hop=256) -> (F, T, M)`` and ``istft(spectrogram, window_length, hop,
length=None) -> (n, M)``. The transforms run in ``libfastmnmf.so``
(``fm_stft`` / ``fm_istft``: radix-2 FFTs in shared memory, gather
overlap-add). NumPy inputs are computed in float64 and returned as NumPy
(complex128 / float64, like the reference); torch CUDA tensors stay on the
device in their own precision (float32 -> complex64, float64 -> complex128).
"""

import numpy as np

from . import _lib
from .errors import InvalidInputError


def hann_periodic(n: int) -> np.ndarray:
    """Periodic Hann window of length n (stft.py:15-17)."""
    return 0.5 - 0.5 * np.cos(2.0 * np.pi * np.arange(n) / n)


def _validate_params(window_length, hop):  # stft.py:20-24
    if window_length <= 0 or (window_length & (window_length - 1)) != 0:
        raise InvalidInputError(f"window_length must be a power of two, got {window_length}")
    if not 0 < hop <= window_length:
        raise InvalidInputError(f"hop must satisfy 0 < hop <= window_length, got {hop}")


def _torch():
    import torch

    return torch


def stft(waveform, window_length: int = 1024, hop: int = 256):
    """Multichannel STFT, reflect-padded by window_length // 2 on both ends
    (stft.py:27-48). Returns (F, T, M) complex."""
    _validate_params(window_length, hop)
    torch = _torch()
    as_numpy = not isinstance(waveform, torch.Tensor)
    w = torch.from_numpy(np.asarray(waveform, dtype=np.float64)) if as_numpy else waveform
    if w.dim() == 1:
        w = w[:, None]
    elif w.dim() != 2:
        raise InvalidInputError(
            f"waveform must have shape (n_samples, n_channels), got {tuple(w.shape)}")
    n, M = w.shape
    if n < window_length:  # stft.py:39-42
        raise InvalidInputError(
            f"signal length {n} is shorter than one window ({window_length})")
    if w.dtype not in (torch.float32, torch.float64):
        w = w.to(torch.float64)
    w = w.to("cuda").contiguous()
    lib = _lib.load()
    T = lib.fm_stft_frames(n, window_length, hop)
    cd = torch.complex64 if w.dtype == torch.float32 else torch.complex128
    spec = torch.empty((window_length // 2 + 1, T, M), dtype=cd, device=w.device)
    dt = _lib.FM_F32 if w.dtype == torch.float32 else _lib.FM_F64
    _lib.check(lib.fm_stft(dt, n, M, window_length, hop, _lib.ptr(w), _lib.ptr(spec),
                           _lib.stream_ptr()), "fm_stft")
    if as_numpy:
        return spec.cpu().numpy()
    return spec


def istft(spectrogram, window_length: int = 1024, hop: int = 256, length=None):
    """Inverse STFT by windowed overlap-add; undoes the stft() padding
    (stft.py:51-91). ``length`` trims to the original sample count."""
    _validate_params(window_length, hop)
    torch = _torch()
    as_numpy = not isinstance(spectrogram, torch.Tensor)
    spec = torch.from_numpy(np.asarray(spectrogram)) if as_numpy else spectrogram
    if spec.dim() != 3:
        raise InvalidInputError(f"spectrogram must have shape (F, T, M), got {tuple(spec.shape)}")
    n_freq, n_frames, M = spec.shape
    if n_freq != window_length // 2 + 1:
        raise InvalidInputError(
            f"spectrogram has {n_freq} bins; window_length {window_length} implies "
            f"{window_length // 2 + 1}")
    avail = (n_frames - 1) * hop  # window_length + (T-1) hop - 2 (window_length // 2)
    if length is not None:
        if length > avail:  # stft.py:84-88
            raise InvalidInputError(
                f"requested length {length} exceeds reconstructable {avail}")
        out_len = int(length)
    else:
        out_len = avail
    if spec.dtype == torch.complex64:
        dt, real = _lib.FM_F32, torch.float32
    else:
        spec = spec.to(torch.complex128)
        dt, real = _lib.FM_F64, torch.float64
    spec = spec.to("cuda").contiguous()
    lib = _lib.load()
    work = torch.empty((lib.fm_istft_workspace_bytes(dt, n_frames, M, window_length),),
                       dtype=torch.uint8, device=spec.device)
    out = torch.empty((out_len, M), dtype=real, device=spec.device)
    _lib.check(lib.fm_istft(dt, n_frames, M, window_length, hop, out_len, _lib.ptr(spec),
                            _lib.ptr(work), _lib.ptr(out), _lib.stream_ptr()), "fm_istft")
    if as_numpy:
        return out.cpu().numpy()
    return out
