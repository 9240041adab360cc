"""Device operators with the signatures of the reference's operator seam
``fastsep._kernels`` (``pkg/src/fastsep/_kernels.py``), backed by the sm_100a
kernels of libfastmnmf.so.

Each function accepts numpy arrays (cast to float64/complex128, exactly as the
reference wrappers cast, ``_kernels.py:263-265``; results come back as numpy)
or CUDA torch tensors (float32/complex64 or float64/complex128 are kept;
results come back as CUDA tensors). Skipped ``fast_stats`` outputs are the
reference's ``(1, 1, 1)`` zero placeholders (``_kernels.py:196-204``).
"""

import ctypes

import numpy as np

from . import _lib
from .errors import InvalidInputError, SingularMatrixError

HAVE_CUDA_BACKEND = True  # the analogue of _kernels.HAVE_NUMBA: always the CUDA path


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1903_03237_b200 needs a CUDA device (no CPU fallback)")
    return torch


class _Io:
    """numpy <-> device shim: remembers whether results go back to the host."""

    def __init__(self, *arrays):
        torch = _torch()
        self.torch = torch
        self.host = any(not isinstance(a, torch.Tensor) for a in arrays if a is not None)
        self.real = torch.float64
        for a in arrays:
            if isinstance(a, torch.Tensor) and a.dtype in (torch.float32, torch.complex64):
                self.real = torch.float32
        if self.host:
            self.real = torch.float64
        self.cplx = torch.complex64 if self.real == torch.float32 else torch.complex128
        self.dt = _lib.FM_F32 if self.real == torch.float32 else _lib.FM_F64

    def r(self, a):
        t = self.torch
        if isinstance(a, t.Tensor):
            return a.to(device="cuda", dtype=self.real).contiguous()
        return t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda", self.real)

    def c(self, a):
        t = self.torch
        if isinstance(a, t.Tensor):
            return a.to(device="cuda", dtype=self.cplx).resolve_conj().contiguous()
        return t.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).to("cuda", self.cplx)

    def out(self, x):
        if self.host:
            self.torch.cuda.synchronize()
            return x.cpu().numpy()
        return x


def _status_tensor(torch):
    return torch.full((1,), -1, dtype=torch.int64, device="cuda")


def decode_status(raw):
    """(code, iteration, m, f) of a device status word, or None if clear."""
    v = int(raw) & 0xFFFFFFFFFFFFFFFF
    if v == _lib.FM_STATUS_CLEAR:
        return None
    return v & 3, v >> 44, (v >> 24) & 0xFFFFF, (v >> 2) & 0x3FFFFF


def status_message(code, m, f):
    """Message text of the reference's SingularMatrixError for a status code."""
    if code == 1:  # spatial.py:194-198
        return f"non-positive normalization in diagonalizer update at (f={f}, m={m})"
    if code == 2:  # spatial.py:189-192
        return f"singular Q V in diagonalizer update at row m={m}: Singular matrix"
    return "singular diagonalizer: Singular matrix"  # separate.py:121-124


def fast_stats(xt_FTM, g_NFM, lam_NFT, floor=0.0, want_gain=False, want_phi=True):
    """_kernels.fast_stats (_kernels.py:254-267)."""
    io = _Io(xt_FTM, g_NFM, lam_NFT)
    torch = io.torch
    xt, g, lam = io.r(xt_FTM), io.r(g_NFM), io.r(lam_NFT)
    if xt.dim() != 3 or g.dim() != 3 or lam.dim() != 3:
        raise InvalidInputError("fast_stats expects (F,T,M), (N,F,M), (N,F,T) arrays")
    F, T, M = xt.shape
    N = g.shape[0]
    if tuple(g.shape) != (N, F, M) or tuple(lam.shape) != (N, F, T):
        raise InvalidInputError(f"shape mismatch: xt {tuple(xt.shape)} g {tuple(g.shape)} "
                                f"lam {tuple(lam.shape)}")
    z = torch.zeros((1, 1, 1), device="cuda", dtype=io.real)
    phi1 = torch.empty((N, F, T), device="cuda", dtype=io.real) if want_phi else None
    phi2 = torch.empty_like(phi1) if want_phi else None
    gnum = torch.empty((N, F, M), device="cuda", dtype=io.real) if want_gain else None
    gden = torch.empty_like(gnum) if want_gain else None
    ll = ctypes.c_double(0.0)
    _lib.check(_lib.load().fm_fast_stats(
        io.dt, F, T, M, N, _lib.ptr(xt), _lib.ptr(g), _lib.ptr(lam), float(floor),
        int(bool(want_gain)), int(bool(want_phi)), _lib.ptr(phi1), _lib.ptr(phi2),
        _lib.ptr(gnum), _lib.ptr(gden), ctypes.byref(ll), _lib.stream_ptr()), "fm_fast_stats")
    outs = [phi1 if want_phi else z, phi2 if want_phi else z.clone(),
            gnum if want_gain else z.clone(), gden if want_gain else z.clone()]
    return tuple(io.out(o) for o in outs) + (float(ll.value),)


def mix_power(lam_NFT, g_NFM, floor=0.0):
    """_kernels.mix_power (_kernels.py:325-331)."""
    io = _Io(lam_NFT, g_NFM)
    lam, g = io.r(lam_NFT), io.r(g_NFM)
    N, F, T = lam.shape
    M = g.shape[-1]
    y = io.torch.empty((F, T, M), device="cuda", dtype=io.real)
    _lib.check(_lib.load().fm_mix_power(io.dt, N, F, T, M, _lib.ptr(lam), _lib.ptr(g),
                                        float(floor), _lib.ptr(y), _lib.stream_ptr()),
               "fm_mix_power")
    return io.out(y)


def ip_weights(X_FTM, y_FTM):
    """_kernels.ip_weights (_kernels.py:296-302): V (F,M,M,M)."""
    io = _Io(X_FTM, y_FTM)
    X, y = io.c(X_FTM), io.r(y_FTM)
    F, T, M = X.shape
    V = io.torch.empty((F, M, M, M), device="cuda", dtype=io.cplx)
    _lib.check(_lib.load().fm_ip_weights(io.dt, F, T, M, _lib.ptr(X), _lib.ptr(y), _lib.ptr(V),
                                         _lib.stream_ptr()), "fm_ip_weights")
    return io.out(V)


def project_power(Q_FMM, X_FTM):
    """_kernels.project_power (_kernels.py:353-359)."""
    io = _Io(Q_FMM, X_FTM)
    Q, X = io.c(Q_FMM), io.c(X_FTM)
    F, T, M = X.shape
    xt = io.torch.empty((F, T, M), device="cuda", dtype=io.real)
    _lib.check(_lib.load().fm_project_power(io.dt, F, T, M, _lib.ptr(Q), _lib.ptr(X),
                                            _lib.ptr(xt), _lib.stream_ptr()), "fm_project_power")
    return io.out(xt)


def update_diagonalizer(Q_FMM, X_FTM, y_FTM, sweeps=1):
    """spatial.update_diagonalizer (spatial.py:172-200)."""
    io = _Io(Q_FMM, X_FTM, y_FTM)
    torch = io.torch
    Q = io.c(Q_FMM).clone()
    X, y = io.c(X_FTM), io.r(y_FTM)
    F, T, M = X.shape
    st = _status_tensor(torch)
    _lib.check(_lib.load().fm_update_diagonalizer(io.dt, F, T, M, _lib.ptr(Q), _lib.ptr(X),
                                                  _lib.ptr(y), int(sweeps), _lib.ptr(st),
                                                  _lib.stream_ptr()), "fm_update_diagonalizer")
    s = decode_status(st.item())
    if s is not None:
        code, _, m, f = s
        raise SingularMatrixError(status_message(code, m, f))
    return io.out(Q)


def logdet(Q_FMM):
    """np.linalg.slogdet(Q)[1] per bin (spatial.py:241)."""
    io = _Io(Q_FMM)
    Q = io.c(Q_FMM)
    F, M, _ = Q.shape
    out = io.torch.empty((F,), device="cuda", dtype=io.torch.float64)
    _lib.check(_lib.load().fm_logdet(io.dt, F, M, _lib.ptr(Q), _lib.ptr(out), _lib.stream_ptr()),
               "fm_logdet")
    return io.out(out)


def check_wiener_status(st):
    """Raise the reference's error for a singular diagonaliser (separate.py:116)."""
    s = decode_status(st.item())
    if s is not None:
        raise SingularMatrixError(status_message(3, 0, s[3]))


def wiener_fast(lam_NFT, Q_FMM, g_NFM, X_FTM, defer_status=False):
    """separate.wiener_fast (separate.py:110-125): images (N,F,T,M).

    ``defer_status=True`` (device inputs) skips the host read of the status
    word and returns (images, status tensor) for ``check_wiener_status`` --
    the caller overlaps its own work with the kernel."""
    io = _Io(lam_NFT, Q_FMM, g_NFM, X_FTM)
    torch = io.torch
    lam, Q, g, X = io.r(lam_NFT), io.c(Q_FMM), io.r(g_NFM), io.c(X_FTM)
    N, F, T = lam.shape
    M = X.shape[-1]
    out = torch.empty((N, F, T, M), device="cuda", dtype=io.cplx)
    st = _status_tensor(torch)
    _lib.check(_lib.load().fm_wiener_fast(io.dt, N, F, T, M, _lib.ptr(lam), _lib.ptr(Q),
                                          _lib.ptr(g), _lib.ptr(X), _lib.ptr(out), _lib.ptr(st),
                                          _lib.stream_ptr()), "fm_wiener_fast")
    if defer_status:
        return io.out(out), st
    check_wiener_status(st)
    return io.out(out)
