"""CPU oracle for the FastMNMF iteration — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it. The product path
(``paper_1903_03237_b200``) runs hand-written sm_100a CUDA and never calls
into this file.

It restates, in float64/complex128 numpy, the reference ``fastsep`` 0.1.0
jointly-diagonalizable loop (``method="fast-mnmf"``). Every function cites the
reference file:line it follows (paths relative to ``/root/reference/pkg/src/
fastsep/``). Parity of this restatement with the reference itself is pinned by
``tests/test_oracle_golden.py`` against the vectors in ``tests/golden/`` that
``oracle/make_golden.py`` produced by importing and running the unmodified
reference in the build container.
"""

import numpy as np

TINY = np.finfo(float).tiny  # sources.py:24, separate.py:219
Y_FLOOR_REL = 1e-12  # spatial.py:31


class OracleError(Exception):
    """Raised where the reference raises (SingularMatrixError / InvalidInputError)."""

    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


# --------------------------------------------------------------------------
# L1 kernels (_kernels.py, numpy twins)
# --------------------------------------------------------------------------

def mix_power(lam_NFT, g_NFM, floor=0.0):
    """y = max(sum_n lam g, floor)  -- _kernels.py:306-308 (numba :310-322)."""
    y = np.einsum("nft,nfm->ftm", lam_NFT, g_NFM)
    return np.maximum(y, floor)


def fast_stats(xt_FTM, g_NFM, lam_NFT, floor=0.0, want_gain=False, want_phi=True):
    """(phi1, phi2, gnum, gden, loglik)  -- _kernels.py:187-205, wrapper :254-267.

    phi1 = sum_m g x~/y^2, phi2 = sum_m g/y, gnum = sum_t lam x~/y^2,
    gden = sum_t lam/y, loglik = sum(-x~/y - log y); skipped outputs are the
    (1,1,1) zero placeholders of :196-204.
    """
    xt = np.asarray(xt_FTM, dtype=np.float64)
    g = np.asarray(g_NFM, dtype=np.float64)
    lam = np.asarray(lam_NFT, dtype=np.float64)
    y = mix_power(lam, g, floor)
    iy = 1.0 / y
    r = xt * iy * iy
    if want_phi:
        phi1 = np.einsum("nfm,ftm->nft", g, r)
        phi2 = np.einsum("nfm,ftm->nft", g, iy)
    else:
        phi1 = np.zeros((1, 1, 1))
        phi2 = np.zeros((1, 1, 1))
    loglik = float((-xt * iy - np.log(y)).sum())
    if want_gain:
        gnum = np.einsum("nft,ftm->nfm", lam, r)
        gden = np.einsum("nft,ftm->nfm", lam, iy)
    else:
        gnum = np.zeros((1, 1, 1))
        gden = np.zeros((1, 1, 1))
    return phi1, phi2, gnum, gden, loglik


def ip_weights(X_FTM, y_FTM):
    """V[f,m] = (1/T) sum_t x x^H / y_ftm, (F,M,M,M)  -- _kernels.py:270-273 (numba :276-293)."""
    X = np.asarray(X_FTM, dtype=np.complex128)
    y = np.asarray(y_FTM, dtype=np.float64)
    T = X.shape[1]
    XX = X[..., :, None] * X[..., None, :].conj()
    return np.einsum("ftm,ftij->fmij", 1.0 / y, XX) / T


def project_power(Q_FMM, X_FTM):
    """x~ = |Q x|^2 (row m of Q_f is q_fm^H)  -- _kernels.py:334-336 (numba :339-350)."""
    qx = np.einsum("fij,ftj->fti", np.asarray(Q_FMM, np.complex128),
                   np.asarray(X_FTM, np.complex128))
    return qx.real ** 2 + qx.imag ** 2


# --------------------------------------------------------------------------
# L2 models (spatial.py, sources.py)
# --------------------------------------------------------------------------

def power_floor(xt_FTM):
    """1e-12 * max(x~)  -- spatial.py:64-66."""
    return Y_FLOOR_REL * float(np.max(xt_FTM))


def update_diagonalizer(Q_FMM, X_FTM, y_FTM, sweeps=1):
    """Iterative-projection (Gauss-Seidel over rows) update -- spatial.py:172-200."""
    Q = np.array(Q_FMM, dtype=np.complex128)
    F, M, _ = Q.shape
    for _ in range(sweeps):
        V_FMMM = ip_weights(X_FTM, y_FTM)  # spatial.py:182
        for m in range(M):  # :183, rows < m already updated
            V = V_FMMM[:, m]
            rhs = np.zeros((M, 1), dtype=np.complex128)
            rhs[m] = 1.0
            try:
                q = np.linalg.solve(Q @ V, np.broadcast_to(rhs, (F, M, 1)).copy())[..., 0]
            except np.linalg.LinAlgError as exc:  # :189-192
                raise OracleError(
                    "singular",
                    f"singular Q V in diagonalizer update at row m={m}: {exc}") from exc
            norm = np.einsum("fi,fij,fj->f", q.conj(), V, q).real  # :193
            if np.any(norm <= 0) or not np.all(np.isfinite(norm)):  # :194-198
                f = int(np.argwhere((norm <= 0) | ~np.isfinite(norm))[0, 0])
                raise OracleError(
                    "singular",
                    f"non-positive normalization in diagonalizer update at (f={f}, m={m})")
            Q[:, m, :] = (q / np.sqrt(norm)[:, None]).conj()  # :199
    return Q


def normalize_gains(g_NFM):
    """sum_m g = M; returns (g, c = s/M)  -- spatial.py:244-249."""
    M = g_NFM.shape[-1]
    s = np.maximum(g_NFM.sum(axis=-1), TINY)
    return g_NFM * (M / s)[..., None], s / M


def loglik_fast(X_FTM, Q_FMM, g_NFM, lam_NFT, floor=0.0, xt_FTM=None):
    """data term + 2T sum_f log|det Q_f|  -- spatial.py:233-241."""
    if xt_FTM is None:
        xt_FTM = project_power(Q_FMM, X_FTM)
    T = xt_FTM.shape[1]
    data = fast_stats(xt_FTM, g_NFM, lam_NFT, floor, want_gain=False, want_phi=False)[4]
    return data + 2.0 * T * float(np.linalg.slogdet(Q_FMM)[1].sum())


class NmfSourceOracle:
    """lam = W @ H with MU blocks W, H  -- sources.py:167-204."""

    mu_steps = ("W", "H")

    def __init__(self, W_NFK, H_NKT):
        self.W_NFK = np.asarray(W_NFK, dtype=np.float64).copy()
        self.H_NKT = np.asarray(H_NKT, dtype=np.float64).copy()
        self._lam = None

    def lam(self):  # sources.py:184-187 (cached until the next update)
        if self._lam is None:
            self._lam = self.W_NFK @ self.H_NKT
        return self._lam

    def apply_mu(self, step, phi1_NFT, phi2_NFT):  # sources.py:189-200
        self._lam = None
        if step == "W":
            num = np.matmul(phi1_NFT, self.H_NKT.transpose(0, 2, 1))
            den = np.matmul(phi2_NFT, self.H_NKT.transpose(0, 2, 1))
            self.W_NFK = self.W_NFK * np.sqrt(num / np.maximum(den, TINY))
        elif step == "H":
            num = np.matmul(self.W_NFK.transpose(0, 2, 1), phi1_NFT)
            den = np.matmul(self.W_NFK.transpose(0, 2, 1), phi2_NFT)
            self.H_NKT = self.H_NKT * np.sqrt(num / np.maximum(den, TINY))
        else:
            raise OracleError("invalid", f"unknown NMF update step {step!r}")

    def absorb_scale(self, c_NF):  # sources.py:202-204
        self._lam = None
        self.W_NFK = self.W_NFK * c_NF[:, :, None]


def wiener_fast(lam_NFT, Q_FMM, g_NFM, X_FTM):
    """Q^-1 Diag(lam g / sum_n lam g) Q x, (N,F,T,M)  -- separate.py:110-125."""
    num = lam_NFT[..., None] * g_NFM[:, :, None, :]
    den = num.sum(axis=0)
    with np.errstate(invalid="ignore", divide="ignore"):
        gains = np.where(den > 0.0, num / den, 1.0 / lam_NFT.shape[0])
    qx = np.einsum("fij,ftj->fti", Q_FMM, X_FTM)
    try:
        Qi = np.linalg.inv(Q_FMM)
    except np.linalg.LinAlgError as exc:
        raise OracleError("singular", f"singular diagonalizer: {exc}") from exc
    return np.einsum("fij,nftj->nfti", Qi, gains * qx[None], optimize=True)


# --------------------------------------------------------------------------
# L3 loop (separate.py)
# --------------------------------------------------------------------------

class DiagLoopOracle:
    """One FastMNMF pass  -- separate.py:175-243 (_DiagLoop)."""

    def __init__(self, X, Q_FMM, g_NFM, source, floor):
        self.X = X
        self.Q_FMM = np.array(Q_FMM, dtype=np.complex128)
        self.g_NFM = np.array(g_NFM, dtype=np.float64)
        self.source = source
        self.floor = floor
        self.xt = project_power(self.Q_FMM, X)  # separate.py:183
        self.first_refresh_ll = None

    def _refresh(self, want_gain=False):  # separate.py:186-193
        phi1, phi2, gnum, gden, ll = fast_stats(
            self.xt, self.g_NFM, self.source.lam(), self.floor,
            want_gain=want_gain, want_phi=not want_gain)
        if self.first_refresh_ll is None:
            self.first_refresh_ll = ll
        return phi1, phi2, gnum, gden

    def loglik(self):  # separate.py:195-199
        return loglik_fast(self.X, self.Q_FMM, self.g_NFM, self.source.lam(),
                           self.floor, xt_FTM=self.xt)

    def iterate(self, normalize=True, ip_sweeps=1):  # separate.py:201-234
        self.first_refresh_ll = None
        source = self.source
        for step in source.mu_steps:  # :214-216
            phi1, phi2, _, _ = self._refresh()
            source.apply_mu(step, phi1, phi2)
        _, _, gnum, gden = self._refresh(want_gain=True)  # :217
        self.g_NFM = self.g_NFM * np.sqrt(gnum / np.maximum(gden, TINY))  # :218-220
        y = mix_power(source.lam(), self.g_NFM, self.floor)  # :221
        self.Q_FMM = update_diagonalizer(self.Q_FMM, self.X, y, ip_sweeps)  # :222
        if normalize:  # :223-229
            row = np.sqrt(np.einsum("fmj,fmj->fm", self.Q_FMM, self.Q_FMM.conj()).real)
            self.Q_FMM = self.Q_FMM / row[:, :, None]
            self.g_NFM = self.g_NFM / np.square(row)[None]
        self.xt = project_power(self.Q_FMM, self.X)  # :230
        if normalize:  # :231-233
            self.g_NFM, c = normalize_gains(self.g_NFM)
            source.absorb_scale(c)
        return self.first_refresh_ll

    def logdet_term(self):  # separate.py:236-238
        T = self.X.shape[1]
        return 2.0 * T * float(np.linalg.slogdet(self.Q_FMM)[1].sum())

    def images(self):  # separate.py:240-243
        return wiener_fast(self.source.lam(), self.Q_FMM, self.g_NFM, self.X)


def run_fastmnmf(X_FTM, Q0, g0, W0, H0, n_iterations, normalize=True, ip_sweeps=1,
                 record_likelihood=True, on_iteration=None, want_images=True):
    """``fastsep.run`` for method="fast-mnmf" with an injected init  -- separate.py:276-330.

    The init (Q0, g0, W0, H0) lives in the scaled domain, exactly where the
    reference's ``_build_spatial``/``_build_source`` place theirs (SURVEY
    §8(c) injection recipe). Returns a dict with the likelihood trace, the
    final W, H, g, Q (scaled domain) and the separated images (unscaled).
    """
    X = np.ascontiguousarray(X_FTM, dtype=np.complex128)  # :284
    if X.ndim != 3:
        raise OracleError("invalid", f"observation must have shape (F, T, M), got {X.shape}")
    if not np.all(np.isfinite(X)):
        raise OracleError("invalid", "observation contains non-finite values")
    power = float(np.mean(np.abs(X) ** 2))  # :289
    if power == 0.0:
        raise OracleError("invalid", "observation is identically zero")
    scale = np.sqrt(power)
    Xs = X / scale
    source = NmfSourceOracle(W0, H0)
    loop = DiagLoopOracle(Xs, Q0, g0, source, power_floor(np.abs(Xs) ** 2))  # :299
    ll_trace = []
    pending = None
    for it in range(n_iterations):  # :306-320
        try:
            ll_before = loop.iterate(normalize, ip_sweeps)
        except OracleError as exc:
            raise OracleError(exc.kind, f"iteration {it}: {exc}") from exc
        if record_likelihood:
            if it > 0:
                ll_trace.append(ll_before + pending)
            pending = loop.logdet_term()
        if on_iteration is not None:
            on_iteration(it, loop)
    if record_likelihood:  # :321-322
        ll_trace.append(loop.loglik())
    out = dict(
        likelihood_trace=np.asarray(ll_trace),
        W=source.W_NFK, H=source.H_NKT, g=loop.g_NFM, Q=loop.Q_FMM,
        scale=scale, floor=loop.floor, xt=loop.xt,
    )
    if want_images:
        out["images"] = loop.images() * scale  # :323
    return out
