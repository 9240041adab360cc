"""Diagonalizable spatial model surface (``fastsep/spatial.py``) on the device.

``DiagSpatial`` keeps the reference's parameter layout (Q_FMM (F,M,M) complex
with row m = q_fm^H, g_NFM (N,F,M)); the update functions run the sm_100a
kernels through ``kernels``.
"""

from dataclasses import dataclass

import numpy as np

from . import kernels as K
from .errors import InvalidInputError

Y_FLOOR_REL = 1e-12  # spatial.py:31


@dataclass
class DiagSpatial:
    """Diagonalizer Q (F, M, M, nonsingular) and gains g (N, F, M, >= 0)."""

    Q_FMM: object
    g_NFM: object

    @property
    def n_sources(self):
        return self.g_NFM.shape[0]


def power_floor(xt_FTM) -> float:
    """spatial.py:64-66."""
    return Y_FLOOR_REL * float(np.max(np.asarray(xt_FTM)))


def project(Q_FMM, X_FTM):
    """Projected power x~ = |Q x|^2 (spatial.py:124-132)."""
    if Q_FMM.shape[-1] != X_FTM.shape[-1] or Q_FMM.shape[0] != X_FTM.shape[0]:
        raise InvalidInputError(
            f"diagonalizer shape {tuple(Q_FMM.shape)} does not match observation "
            f"{tuple(X_FTM.shape)}")
    return K.project_power(Q_FMM, X_FTM)


def fast_stats(xt_FTM, g_NFM, lam_NFT, floor, want_gain=False, want_phi=True):
    """spatial.py:140-142."""
    return K.fast_stats(xt_FTM, g_NFM, lam_NFT, floor, want_gain, want_phi)


def update_diagonalizer(Q_FMM, X_FTM, y_FTM, sweeps: int = 1):
    """IP update of the diagonalizer (spatial.py:172-200)."""
    return K.update_diagonalizer(Q_FMM, X_FTM, y_FTM, sweeps)


def _dev(a):
    import torch

    if isinstance(a, torch.Tensor):
        return a, False
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda"), True


def update_gains(g_NFM, lam_NFT, xt_FTM, floor):
    """g <- g sqrt(sum_t lam x~/y^2 / sum_t lam/y)  (spatial.py:203-208)."""
    g, host = _dev(g_NFM)
    lam, _ = _dev(lam_NFT)
    xt, _ = _dev(xt_FTM)
    lam, xt = lam.to(g.dtype), xt.to(g.dtype)
    _, _, gnum, gden, _ = K.fast_stats(xt, g, lam, floor, want_gain=True, want_phi=False)
    out = g * (gnum / gden.clamp_min(np.finfo(float).tiny)).sqrt()
    return out.cpu().numpy() if host else out


def loglik_fast(X_FTM, Q_FMM, g_NFM, lam_NFT, floor=0.0, xt_FTM=None) -> float:
    """data term + 2T sum_f log|det Q_f|  (spatial.py:233-241)."""
    if xt_FTM is None:
        xt_FTM = project(Q_FMM, X_FTM)
    T = xt_FTM.shape[1]
    data = K.fast_stats(xt_FTM, g_NFM, lam_NFT, floor, want_gain=False, want_phi=False)[4]
    ld = K.logdet(Q_FMM)
    ld = ld if isinstance(ld, np.ndarray) else ld.cpu().numpy()
    return data + 2.0 * T * float(ld.sum())


def normalize_gains(g_NFM):
    """sum_m g = M; returns (g, absorbed factor)  (spatial.py:244-249)."""
    g, host = _dev(g_NFM)
    M = g.shape[-1]
    s = g.sum(dim=-1).clamp_min(np.finfo(float).tiny)
    out, c = g * (M / s)[..., None], s / M
    if host:
        return out.cpu().numpy(), c.cpu().numpy()
    return out, c
