"""CPU restatement of the reference's full-rank MNMF (method "mnmf") --
TEST INFRASTRUCTURE ONLY (tests/ use it as the checker; the product never
does). Follows fastsep _kernels.py:38-60 (fullrank_stats, numpy twin),
spatial.py:145-169 (update_scm), linalg.py:85-109 (clamp_psd,
hermitian_sqrt_pair), spatial.py:211-223 (reconstruct_scm), :252-257
(normalize_trace), separate.py:83-107 (wiener_fullrank), :128-172
(_FullRankLoop) and :276-330 (run bookkeeping). Pinned to
tests/golden/fullrank.npz (oracle/make_golden.py --fullrank-only), outputs
of the unmodified reference."""

import numpy as np

from .fastmnmf_oracle import OracleError

TINY = np.finfo(float).tiny


def fullrank_stats(X, G, lam, ridge, want_ab=False, want_phi=True):
    """_kernels.py:38-60."""
    M = X.shape[-1]
    Y = np.einsum("nft,nfij->ftij", lam, G) + ridge * np.eye(M)
    Yi = np.linalg.inv(Y)
    z = np.einsum("ftij,ftj->fti", Yi, X)
    phi1 = np.einsum("fti,nfij,ftj->nft", z.conj(), G, z, optimize=True).real if want_phi else None
    phi2 = np.einsum("nfij,ftji->nft", G, Yi, optimize=True).real if want_phi else None
    trace = np.einsum("fti,fti->ft", X.conj(), z).real
    ll = float((-trace - np.linalg.slogdet(Y)[1]).sum())
    A = np.einsum("nft,fti,ftj->nfij", lam, z, z.conj(), optimize=True) if want_ab else None
    B = np.einsum("nft,ftij->nfij", lam, Yi, optimize=True) if want_ab else None
    return phi1, phi2, A, B, ll


def clamp_psd(m, floor=1e-12):
    """linalg.py:85-94."""
    m = 0.5 * (m + np.conj(np.swapaxes(m, -1, -2)))
    w, v = np.linalg.eigh(m)
    w = np.maximum(w, floor * np.maximum(w.max(axis=-1, keepdims=True), 0.0))
    return (v * w[..., None, :]) @ np.conj(np.swapaxes(v, -1, -2))


def hermitian_sqrt_pair(m, floor=1e-12):
    """linalg.py:97-109."""
    m = 0.5 * (m + np.conj(np.swapaxes(m, -1, -2)))
    w, v = np.linalg.eigh(m)
    top = np.maximum(w.max(axis=-1, keepdims=True), TINY)
    w = np.maximum(w, floor * top)
    vh = np.conj(np.swapaxes(v, -1, -2))
    sq = np.sqrt(w)
    return (v * sq[..., None, :]) @ vh, (v * (1.0 / sq)[..., None, :]) @ vh


def update_scm(G, A, B):
    """spatial.py:145-169: G <- B^-1/2 (B^1/2 G A G B^1/2)^1/2 B^-1/2."""
    Bs, Bis = hermitian_sqrt_pair(B)
    C = Bs @ G @ A @ G @ Bs
    C = 0.5 * (C + np.conj(C.swapaxes(-1, -2)))
    w, V = np.linalg.eigh(C)
    top = np.maximum(w.max(axis=-1, keepdims=True), 0.0)
    bad = w < -1e-8 * top
    if np.any(bad):
        n, f = np.argwhere(bad.any(axis=-1))[0]
        raise OracleError("breakdown", f"negative spectrum in SCM update at (n={n}, f={f})")
    Cs = (V * np.sqrt(np.maximum(w, 0.0))[..., None, :]) @ np.conj(V.swapaxes(-1, -2))
    return clamp_psd(Bis @ Cs @ Bis)


def normalize_trace(G):
    """spatial.py:252-257."""
    M = G.shape[-1]
    tr = np.maximum(np.einsum("nfii->nf", G).real, TINY)
    return G * (M / tr)[..., None, None], tr / M


def reconstruct_scm(Q, g):
    """spatial.py:211-223."""
    Qi = np.linalg.inv(Q)
    return np.einsum("fij,nfj,fkj->nfik", Qi, g, Qi.conj())


def wiener_fullrank(lam, G, X, ridge=0.0):
    """separate.py:83-107."""
    M = X.shape[-1]
    Y = np.einsum("nft,nfij->ftij", lam, G) + ridge * np.eye(M)
    z = np.linalg.solve(Y, X[..., None])[..., 0]
    images = np.einsum("nft,nfij,ftj->nfti", lam, G, z, optimize=True)
    total = lam.sum(axis=0)
    with np.errstate(invalid="ignore", divide="ignore"):
        share = np.where(total > 0.0, lam / total, 1.0 / lam.shape[0])
    images += share[..., None] * (X - images.sum(axis=0))[None]
    return images


def run_mnmf(X_FTM, G0, W0, H0, n_iterations, normalize=True, want_images=True):
    """run() (separate.py:276-330) with method="mnmf" and an injected init."""
    X = np.ascontiguousarray(X_FTM, dtype=np.complex128)
    scale = np.sqrt(float(np.mean(np.abs(X) ** 2)))
    Xs = X / scale
    ridge = 1e-12 * float(np.mean(np.abs(Xs) ** 2))  # mixture_ridge (spatial.py:59-61)
    G, W, H = np.array(G0, dtype=np.complex128), np.array(W0, float), np.array(H0, float)
    trace = []
    for it in range(n_iterations):
        ll_before = None
        for step in ("W", "H"):
            p1, p2, _, _, ll = fullrank_stats(Xs, G, W @ H, ridge)
            if ll_before is None:
                ll_before = ll
            if step == "W":
                W = W * np.sqrt(np.matmul(p1, H.transpose(0, 2, 1))
                                / np.maximum(np.matmul(p2, H.transpose(0, 2, 1)), TINY))
            else:
                H = H * np.sqrt(np.matmul(W.transpose(0, 2, 1), p1)
                                / np.maximum(np.matmul(W.transpose(0, 2, 1), p2), TINY))
        _, _, A, B, _ = fullrank_stats(Xs, G, W @ H, ridge, want_ab=True, want_phi=False)
        G = update_scm(G, A, B)
        if normalize:
            G, c = normalize_trace(G)
            W = W * c[:, :, None]
        if it > 0:
            trace.append(ll_before)  # logdet_term is 0 for the full-rank loop
    trace.append(fullrank_stats(Xs, G, W @ H, ridge, want_phi=False)[4])
    out = dict(likelihood_trace=np.asarray(trace), G=G, W=W, H=H, scale=scale, ridge=ridge)
    if want_images:
        out["images"] = wiener_fullrank(W @ H, G, Xs, ridge) * scale
    return out
