"""The full-rank MNMF comparator on the device (method "mnmf")
-- the slow model the paper's FastMNMF speed-up is measured against.

Mirrors the reference: ``FullRankSpatial`` (``spatial.py:34-44``),
``fullrank_stats`` (``_kernels.py:166-180``), ``update_scm``
(``spatial.py:145-169``), ``reconstruct_scm`` (``:211-223``),
``wiener_fullrank`` (``separate.py:83-107``) and the ``_FullRankLoop``
schedule (``separate.py:128-172``): per iteration the W and H multiplicative
steps each after a statistics refresh, then A/B statistics, the SCM update
and the trace normalisation folded into W. Every step is a kernel of
libfastmnmf.so (``fm_fullrank_stats``, ``fm_update_scm``, ``fm_nmf_mu``,
``fm_nmf_absorb``, ``fm_wiener_fullrank``, ``fm_reconstruct_scm``); per-bin
linear algebra in fp64, storage in the run's precision.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidInputError, NumericalBreakdownError, SingularMatrixError
from .kernels import decode_status


@dataclass
class FullRankSpatial:
    """Unconstrained SCMs, shape (N, F, M, M), Hermitian PSD per (n, f)."""

    G_NFMM: np.ndarray

    @property
    def n_sources(self):
        return self.G_NFMM.shape[0]


def _torch():
    import torch

    return torch


class _Host:
    """numpy in -> complex128/float64 on the device, numpy out."""

    def __init__(self, *arrays):
        torch = _torch()
        self.torch = torch
        self.host = not any(isinstance(a, torch.Tensor) for a in arrays)
        cd = [a.dtype for a in arrays if isinstance(a, torch.Tensor) and a.is_complex()]
        self.cplx = cd[0] if cd else torch.complex128
        self.real = torch.float32 if self.cplx == torch.complex64 else torch.float64
        self.dt = _lib.FM_F32 if self.real == torch.float32 else _lib.FM_F64

    def c(self, a):
        t = a if isinstance(a, self.torch.Tensor) else self.torch.from_numpy(np.asarray(a))
        return t.to("cuda", self.cplx).resolve_conj().contiguous()

    def r(self, a):
        t = a if isinstance(a, self.torch.Tensor) else self.torch.from_numpy(np.asarray(a))
        return t.to("cuda", self.real).contiguous()

    def out(self, x):
        return x.cpu().numpy() if self.host else x


def _status(torch):
    return torch.full((1,), -1, dtype=torch.int64, device="cuda")


def fullrank_stats(X_FTM, G_NFMM, lam_NFT, ridge=0.0, want_ab=False, want_phi=True):
    """_kernels.fullrank_stats (_kernels.py:166-180): (phi1, phi2, A, B, loglik)."""
    io = _Host(X_FTM, G_NFMM, lam_NFT)
    torch = io.torch
    X, G, lam = io.c(X_FTM), io.c(G_NFMM), io.r(lam_NFT)
    F, T, M = X.shape
    N = G.shape[0]
    if tuple(G.shape) != (N, F, M, M) or tuple(lam.shape) != (N, F, T):
        raise InvalidInputError("fullrank_stats expects X (F,T,M), G (N,F,M,M), lam (N,F,T)")
    lib = _lib.load()
    work = torch.empty((lib.fm_fullrank_workspace_bytes(io.dt, F, T, M),), dtype=torch.uint8,
                       device="cuda")
    phi = torch.empty((2, N, F, T), dtype=io.real, device="cuda") if want_phi else None
    A = torch.empty((N, F, M, M), dtype=io.cplx, device="cuda") if want_ab else None
    B = torch.empty_like(A) if want_ab else None
    ll = torch.zeros((1,), dtype=torch.float64, device="cuda")
    _lib.check(lib.fm_fullrank_stats(io.dt, F, T, M, N, _lib.ptr(X), _lib.ptr(G), _lib.ptr(lam),
                                     float(ridge), int(bool(want_ab)), int(bool(want_phi)),
                                     _lib.ptr(phi), _lib.ptr(A), _lib.ptr(B), _lib.ptr(work),
                                     _lib.ptr(ll), _lib.stream_ptr()), "fm_fullrank_stats")
    z = np.zeros((1, 1, 1)) if io.host else torch.zeros((1, 1, 1), device="cuda")
    z4 = np.zeros((1, 1, 1, 1), dtype=complex) if io.host else torch.zeros((1, 1, 1, 1), device="cuda")
    return (io.out(phi[0]) if want_phi else z, io.out(phi[1]) if want_phi else z,
            io.out(A) if want_ab else z4, io.out(B) if want_ab else z4, float(ll.item()))


def _raise_scm(st):
    s = decode_status(st.item())
    if s is not None:
        code, _, n, f = s
        raise NumericalBreakdownError(f"negative spectrum in SCM update at (n={n}, f={f})")


def update_scm(G_NFMM, A_NFMM, B_NFMM):
    """spatial.update_scm (spatial.py:145-169): G <- B^-1 (B G A G)^{1/2}."""
    io = _Host(G_NFMM, A_NFMM, B_NFMM)
    G, A, B = io.c(G_NFMM).clone(), io.c(A_NFMM), io.c(B_NFMM)
    N, F, M, _ = G.shape
    st = _status(io.torch)
    _lib.check(_lib.load().fm_update_scm(io.dt, N, F, M, _lib.ptr(G), _lib.ptr(A), _lib.ptr(B), 0,
                                         None, _lib.ptr(st), _lib.stream_ptr()), "fm_update_scm")
    _raise_scm(st)
    return io.out(G)


def normalize_trace(G_NFMM):
    """spatial.normalize_trace (spatial.py:252-257) -- host helper for views."""
    M = G_NFMM.shape[-1]
    tr = np.maximum(np.einsum("nfii->nf", G_NFMM).real, np.finfo(float).tiny)
    return G_NFMM * (M / tr)[..., None, None], tr / M


def reconstruct_scm(Q_FMM, g_NFM):
    """spatial.reconstruct_scm (spatial.py:211-223): G = Q^-1 Diag(g) Q^-H."""
    io = _Host(Q_FMM, g_NFM)
    Q, g = io.c(Q_FMM), io.r(g_NFM)
    N, F, M = g.shape
    G = io.torch.empty((N, F, M, M), dtype=io.cplx, device="cuda")
    st = _status(io.torch)
    _lib.check(_lib.load().fm_reconstruct_scm(io.dt, N, F, M, _lib.ptr(Q), _lib.ptr(g), _lib.ptr(G),
                                              _lib.ptr(st), _lib.stream_ptr()), "fm_reconstruct_scm")
    if decode_status(st.item()) is not None:
        raise SingularMatrixError("diagonalizer is singular: Singular matrix")
    return io.out(G)


def wiener_fullrank(lam_NFT, G_NFMM, X_FTM, ridge=0.0):
    """separate.wiener_fullrank (separate.py:83-107): lam G Y^-1 x with the
    partition defect redistributed by power share, (N, F, T, M)."""
    io = _Host(X_FTM, G_NFMM, lam_NFT)
    X, G, lam = io.c(X_FTM), io.c(G_NFMM), io.r(lam_NFT)
    F, T, M = X.shape
    N = G.shape[0]
    out = io.torch.empty((N, F, T, M), dtype=io.cplx, device="cuda")
    st = _status(io.torch)
    _lib.check(_lib.load().fm_wiener_fullrank(io.dt, N, F, T, M, _lib.ptr(lam), _lib.ptr(G),
                                              _lib.ptr(X), float(ridge), _lib.ptr(out), _lib.ptr(st),
                                              _lib.stream_ptr()), "fm_wiener_fullrank")
    s = decode_status(st.item())
    if s is not None:
        _, t, _, f = s
        raise SingularMatrixError(f"singular mixture covariance at (f, t)=({f}, {t})")
    return io.out(out)


class FullRankDeviceLoop:
    """_FullRankLoop (separate.py:128-172) on device-resident state: X (F,T,M)
    scaled, G (N,F,M,M), W (N,F,K), H (N,K,T), ridge."""

    def __init__(self, X, G, W, H, ridge, normalize=True, n_trace=1):
        torch = _torch()
        self.torch = torch
        self.X = X.contiguous()
        self.real = torch.float32 if X.dtype == torch.complex64 else torch.float64
        self.dt = _lib.FM_F32 if self.real == torch.float32 else _lib.FM_F64
        self.G = G.to("cuda", X.dtype).resolve_conj().contiguous()
        self.W = W.to("cuda", self.real).contiguous()
        self.H = H.to("cuda", self.real).contiguous()
        self.F, self.T, self.M = X.shape
        self.N, self.K = self.W.shape[0], self.W.shape[2]
        self.ridge, self.normalize = float(ridge), bool(normalize)
        lib = _lib.load()
        self.work = torch.empty((lib.fm_fullrank_workspace_bytes(self.dt, self.F, self.T, self.M),),
                                dtype=torch.uint8, device="cuda")
        self.phi = torch.empty((2, self.N, self.F, self.T), dtype=self.real, device="cuda")
        self.lam = torch.empty((self.N, self.F, self.T), dtype=self.real, device="cuda")
        self.A = torch.empty_like(self.G)
        self.B = torch.empty_like(self.G)
        self.c = torch.empty((self.N, self.F), dtype=self.real, device="cuda")
        self.ll = torch.zeros((max(1, n_trace) + 1,), dtype=torch.float64, device="cuda")
        self.status = _status(torch)
        self.dims = _lib.FmDims(1, self.F, self.T, self.M, self.N, self.K, 0, self.dt, 1, 1, 0)
        self.it = 0

    def _lam(self):
        _lib.check(_lib.load().fm_nmf_lambda(ctypes.byref(self.dims), _lib.ptr(self.W),
                                             _lib.ptr(self.H), _lib.ptr(self.lam), _lib.stream_ptr()),
                   "fm_nmf_lambda")

    def _stats(self, want_ab, ll_slot=None):
        self._lam()
        llp = None if ll_slot is None else self.ll.data_ptr() + 8 * ll_slot
        _lib.check(_lib.load().fm_fullrank_stats(
            self.dt, self.F, self.T, self.M, self.N, _lib.ptr(self.X), _lib.ptr(self.G),
            _lib.ptr(self.lam), self.ridge, int(want_ab), int(not want_ab), _lib.ptr(self.phi),
            _lib.ptr(self.A), _lib.ptr(self.B), _lib.ptr(self.work), llp, _lib.stream_ptr()),
            "fm_fullrank_stats")

    def iterate(self):
        """One pass (separate.py:151-165); the first refresh's loglik lands in ll[it]."""
        lib = _lib.load()
        for step, code in (("W", 0), ("H", 1)):
            self._stats(False, self.it if step == "W" else None)
            _lib.check(lib.fm_nmf_mu(self.dt, self.N, self.F, self.T, self.K, _lib.ptr(self.phi),
                                     _lib.ptr(self.W), _lib.ptr(self.H), code, _lib.stream_ptr()),
                       "fm_nmf_mu")
        self._stats(True)
        _lib.check(lib.fm_update_scm(self.dt, self.N, self.F, self.M, _lib.ptr(self.G), _lib.ptr(self.A),
                                     _lib.ptr(self.B), int(self.normalize), _lib.ptr(self.c),
                                     _lib.ptr(self.status), _lib.stream_ptr()), "fm_update_scm")
        if self.normalize:
            _lib.check(lib.fm_nmf_absorb(self.dt, self.N, self.F, self.K, _lib.ptr(self.W),
                                         _lib.ptr(self.c), _lib.stream_ptr()), "fm_nmf_absorb")
        self.it += 1

    def final_loglik(self):
        """loglik of the current state (separate.py:140-141) into ll[it]."""
        self._lam()
        llp = self.ll.data_ptr() + 8 * self.it
        _lib.check(_lib.load().fm_fullrank_stats(
            self.dt, self.F, self.T, self.M, self.N, _lib.ptr(self.X), _lib.ptr(self.G),
            _lib.ptr(self.lam), self.ridge, 0, 0, None, None, None, _lib.ptr(self.work), llp,
            _lib.stream_ptr()), "fm_fullrank_stats")

    def status_error(self, it_offset=0):
        s = decode_status(self.status.item())
        if s is None:
            return None
        _, _, n, f = s
        return NumericalBreakdownError(f"negative spectrum in SCM update at (n={n}, f={f})")

    def images(self, scale):
        self._lam()
        return wiener_fullrank(self.lam, self.G, self.X, self.ridge) * float(scale)

    # host views (the _FullRankLoop attribute surface)
    @property
    def spatial(self):
        return FullRankSpatial(self.G.cpu().numpy())

    @property
    def source(self):
        loop = self

        class _Src:
            W_NFK = loop.W.cpu().numpy()
            H_NKT = loop.H.cpu().numpy()

            def lam(self):
                return self.W_NFK @ self.H_NKT

        return _Src()
