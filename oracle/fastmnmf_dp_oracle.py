"""CPU oracle for FastMNMF-DP (BASELINE config 4) -- TEST INFRASTRUCTURE ONLY.

Same rules as oracle/fastmnmf_oracle.py: only tests/, smoke() and bench.py's
CPU legs import this; the product never does.

BASELINE config 4 replaces two parts of the reference's FastMNMF-DP
(``method="fast-mnmf-dp"``, ``separate.py:201-234`` with
``DeepPriorPlusNmfSource``, ``sources.py:223-271``):

* the decoder is an exp-MLP, lambda_speech = u_f v_t exp(dec(z_t)), with
  dec: D=16 -> 128 tanh -> 128 tanh -> F linear, Xavier-normal weights drawn
  from ``default_rng(seed)`` in the order W1, W2, W3, zero biases
  (the reference's decoder interface: a callable with ``latent_dim`` and
  ``n_freq``, ``separate.py:265-273``);
* the latent update at the reference's hook (``separate.py:205-213``:
  ``update_latents_fast(dp, decoder, g[0], y_rest, xt, cfg, rng)`` with the
  rest-of-model power y_rest frozen) is ``adam_steps`` Adam steps on z of the
  FastMNMF negative log-likelihood sum (x~/y + log y), y = max(lambda_0 g_0 +
  y_rest, TINY) -- the objective the reference's Metropolis ratio evaluates
  (``metropolis_log_gamma_fast``, ``sources.py:292-304``).

The reference's own default (ToyDecoder + Metropolis chain)
is restated too (``ToyDecoder``, ``MetropolisLatents``) and pinned to
``tests/golden/run_dp_mh.npz``, a run of the unmodified reference chain.

Choices BASELINE.json leaves open (documented in DESIGN.md): Adam beta1=0.9,
beta2=0.999, eps=1e-8, bias-corrected, lr=1e-2, state persisting across outer
iterations. Everything around the hook is the reference's own loop; the
golden ``tests/golden/run_dp_*.npz`` are produced by running the unmodified
reference with this decoder and this hook (oracle/make_golden.py), which
pins the U/V/W/H/g/Q updates. The Adam/MLP arithmetic itself has no
reference implementation (parity of that part is unpinned).
"""

import numpy as np

from .fastmnmf_oracle import (
    TINY,
    OracleError,
    fast_stats,
    mix_power,
    normalize_gains,
    power_floor,
    project_power,
    update_diagonalizer,
    wiener_fast,
)


class ExpMLPDecoder:
    """z (T, D) -> exp(MLP(z)) (T, F); MLP D -> H tanh -> H tanh -> F linear."""

    def __init__(self, n_freq, latent_dim=16, hidden=128, seed=0):
        rng = np.random.default_rng(seed)

        def xavier(fan_out, fan_in):
            return rng.normal(0.0, np.sqrt(2.0 / (fan_in + fan_out)), (fan_out, fan_in))

        self.W1 = xavier(hidden, latent_dim)
        self.W2 = xavier(hidden, hidden)
        self.W3 = xavier(n_freq, hidden)
        self.b1 = np.zeros(hidden)
        self.b2 = np.zeros(hidden)
        self.b3 = np.zeros(n_freq)

    @property
    def latent_dim(self):
        return self.W1.shape[1]

    @property
    def n_freq(self):
        return self.W3.shape[0]

    def forward(self, z):
        h1 = np.tanh(z @ self.W1.T + self.b1)
        h2 = np.tanh(h1 @ self.W2.T + self.b2)
        o = h2 @ self.W3.T + self.b3
        return o, (h1, h2)

    def __call__(self, z):
        return np.exp(self.forward(np.asarray(z, dtype=np.float64))[0])

    def backward_z(self, cache, g_o):
        """dL/dz for upstream gradient g_o = dL/do (T, F)."""
        h1, h2 = cache
        d2 = (g_o @ self.W3) * (1.0 - h2 * h2)
        d1 = (d2 @ self.W2) * (1.0 - h1 * h1)
        return d1 @ self.W1


class AdamLatents:
    """The config-4 latent hook: ``adam_steps`` Adam steps per outer iteration."""

    def __init__(self, adam_steps=10, lr=1e-2, beta1=0.9, beta2=0.999, eps=1e-8):
        self.steps, self.lr, self.b1, self.b2, self.eps = adam_steps, lr, beta1, beta2, eps
        self.m = self.v = None
        self.t = 0

    def nll_grad_o(self, dp, g_FM, y_rest_FTM, xt_FTM, o_TF):
        lam = dp.u_F[:, None] * (dp.v_T[:, None] * np.exp(o_TF)).T  # (F, T)
        y = np.maximum(lam[..., None] * g_FM[:, None, :] + y_rest_FTM, TINY)
        dlam = np.einsum("fm,ftm->ft", g_FM, 1.0 / y - xt_FTM / (y * y))
        return (dlam * lam).T  # d lam / d o = lam

    def __call__(self, dp, decoder, g_FM, y_rest_FTM, xt_FTM, cfg=None, rng=None):
        z = dp.z_TD
        if self.m is None:
            self.m = np.zeros_like(z)
            self.v = np.zeros_like(z)
        for _ in range(self.steps):
            o, cache = decoder.forward(z)
            gz = decoder.backward_z(cache, self.nll_grad_o(dp, g_FM, y_rest_FTM, xt_FTM, o))
            self.t += 1
            self.m = self.b1 * self.m + (1 - self.b1) * gz
            self.v = self.b2 * self.v + (1 - self.b2) * gz * gz
            mh = self.m / (1 - self.b1 ** self.t)
            vh = self.v / (1 - self.b2 ** self.t)
            z = z - self.lr * mh / (np.sqrt(vh) + self.eps)
        dp.z_TD = z
        dp.refresh(decoder)
        return 0


class ToyDecoder:
    """The reference's default decoder restated (sources.py:52-80): seeded
    draws w1 ~ N(0, 1/D) (H, D), b1 ~ N(0, 0.25) (H), w2 ~ N(0, 1/H) (F, H),
    b2 ~ N(0, 0.25) (F); r = max(softplus(tanh(z w1^T + b1) w2^T + b2), 1e-8)
    with softplus(x) = log1p(exp(-|x|)) + max(x, 0) (sources.py:31-35)."""

    def __init__(self, n_freq, latent_dim=16, hidden=64, seed=0):
        rng = np.random.default_rng(seed)
        self.w1 = rng.normal(0.0, 1.0 / np.sqrt(latent_dim), (hidden, latent_dim))
        self.b1 = rng.normal(0.0, 0.5, hidden)
        self.w2 = rng.normal(0.0, 1.0 / np.sqrt(hidden), (n_freq, hidden))
        self.b2 = rng.normal(0.0, 0.5, n_freq)

    @property
    def latent_dim(self):
        return self.w1.shape[1]

    @property
    def n_freq(self):
        return self.w2.shape[0]

    def __call__(self, z):
        h = np.tanh(np.asarray(z, dtype=np.float64) @ self.w1.T + self.b1)
        o = h @ self.w2.T + self.b2
        return np.maximum(np.log1p(np.exp(-np.abs(o))) + np.maximum(o, 0.0), 1e-8)


class MetropolisLatents:
    """The reference's latent hook restated: update_latents_fast / _run_chain
    (sources.py:307-339) with metropolis_log_gamma_fast (:292-304). Per inner
    step: z' = z + sqrt(var) * rng.standard_normal((T, D)); r' = dec(z');
    log gamma_t = -sum_fm x~ (1/y' - 1/y) - sum_fm log(y'/y),
    y = max(lambda g_0 + y_rest, TINY); accept iff
    log(rng.uniform(size=T)) <= log gamma_t."""

    def __init__(self, rng, inner_steps=30, proposal_var=1e-4):
        self.rng, self.steps, self.std = rng, inner_steps, np.sqrt(proposal_var)

    def __call__(self, dp, decoder, g_FM, y_rest_FTM, xt_FTM, cfg=None, rng=None):
        T = dp.z_TD.shape[0]
        lam_old = dp.lam_FT()
        for _ in range(self.steps):
            z_new = dp.z_TD + self.std * self.rng.standard_normal(dp.z_TD.shape)
            r_new = decoder(z_new)
            lam_new = dp.u_F[:, None] * (dp.v_T[:, None] * r_new).T
            y_new = np.maximum(lam_new[..., None] * g_FM[:, None, :] + y_rest_FTM, TINY)
            y_old = np.maximum(lam_old[..., None] * g_FM[:, None, :] + y_rest_FTM, TINY)
            lg = (-(xt_FTM * (1.0 / y_new - 1.0 / y_old)).sum(axis=(0, 2))
                  - np.log(y_new / y_old).sum(axis=(0, 2)))
            acc = np.log(self.rng.uniform(size=T)) <= lg
            dp.z_TD[acc] = z_new[acc]
            dp.r_TF[acc] = r_new[acc]
            lam_old[:, acc] = lam_new[:, acc]
        return 0


class DPState:
    """u, v, z, r of the deep-prior source (sources.py:207-220)."""

    def __init__(self, u_F, v_T, z_TD, decoder):
        self.u_F = np.array(u_F, dtype=np.float64)
        self.v_T = np.array(v_T, dtype=np.float64)
        self.z_TD = np.array(z_TD, dtype=np.float64)
        self.r_TF = decoder(self.z_TD)

    def refresh(self, decoder):
        self.r_TF = decoder(self.z_TD)

    def lam_FT(self):
        return self.u_F[:, None] * (self.v_T[:, None] * self.r_TF).T


def run_fastmnmf_dp(X_FTM, Q0, g0, u0, v0, z0, W0, H0, decoder, n_iterations, adam_steps=10,
                    lr=1e-2, normalize=True, ip_sweeps=1, want_images=True, hook=None):
    """FastMNMF-DP; structure of separate.py:201-330. The latent hook is the
    config-4 Adam update (``adam_steps`` > 0), or ``hook`` (e.g.
    MetropolisLatents, the reference's own chain)."""
    X = np.ascontiguousarray(X_FTM, dtype=np.complex128)
    power = float(np.mean(np.abs(X) ** 2))
    scale = np.sqrt(power)
    Xs = X / scale
    floor = power_floor(np.abs(Xs) ** 2)
    Q = np.array(Q0, dtype=np.complex128)
    g = np.array(g0, dtype=np.float64)
    W = np.array(W0, dtype=np.float64)
    H = np.array(H0, dtype=np.float64)
    dp = DPState(u0, v0, z0, decoder)
    if hook is None and adam_steps > 0:
        hook = AdamLatents(adam_steps, lr)
    xt = project_power(Q, Xs)

    def lam():
        return np.concatenate([dp.lam_FT()[None], W @ H], axis=0)

    ll_trace, pending = [], None
    for it in range(n_iterations):
        lam_all = lam()
        # latent hook (separate.py:205-213): y_rest without floor, LL captured first
        y_rest = mix_power(lam_all[1:], g[1:])
        ll_before = fast_stats(xt, g, lam_all, floor)[4]
        if hook is not None:
            hook(dp, decoder, g[0], y_rest, xt)
        for step in ("U", "V", "W", "H"):  # sources.py:226, 251-267
            p1, p2, _, _, _ = fast_stats(xt, g, lam(), floor)
            if step == "U":
                vr = dp.v_T[:, None] * dp.r_TF
                dp.u_F = dp.u_F * np.sqrt(np.einsum("tf,ft->f", vr, p1[0])
                                          / np.maximum(np.einsum("tf,ft->f", vr, p2[0]), TINY))
            elif step == "V":
                ur = dp.u_F[None, :] * dp.r_TF
                dp.v_T = dp.v_T * np.sqrt(np.einsum("tf,ft->t", ur, p1[0])
                                          / np.maximum(np.einsum("tf,ft->t", ur, p2[0]), TINY))
            elif step == "W":
                num = np.matmul(p1[1:], H.transpose(0, 2, 1))
                den = np.matmul(p2[1:], H.transpose(0, 2, 1))
                W = W * np.sqrt(num / np.maximum(den, TINY))
            else:
                num = np.matmul(W.transpose(0, 2, 1), p1[1:])
                den = np.matmul(W.transpose(0, 2, 1), p2[1:])
                H = H * np.sqrt(num / np.maximum(den, TINY))
        lam_all = lam()
        _, _, gn, gd, _ = fast_stats(xt, g, lam_all, floor, want_gain=True, want_phi=False)
        g = g * np.sqrt(gn / np.maximum(gd, TINY))
        try:
            Q = update_diagonalizer(Q, Xs, mix_power(lam_all, g, floor), ip_sweeps)
        except OracleError as exc:
            raise OracleError(exc.kind, f"iteration {it}: {exc}") from exc
        if normalize:
            row = np.sqrt(np.einsum("fmj,fmj->fm", Q, Q.conj()).real)
            Q = Q / row[:, :, None]
            g = g / np.square(row)[None]
        xt = project_power(Q, Xs)
        if normalize:  # absorb_scale (sources.py:269-271)
            g, c = normalize_gains(g)
            dp.u_F = dp.u_F * c[0]
            W = W * c[1:, :, None]
        if it > 0:
            ll_trace.append(ll_before + pending)
        pending = 2.0 * Xs.shape[1] * float(np.linalg.slogdet(Q)[1].sum())
    lam_all = lam()
    ll_trace.append(fast_stats(xt, g, lam_all, floor)[4] + pending)
    out = dict(likelihood_trace=np.asarray(ll_trace), W=W, H=H, g=g, Q=Q, u=dp.u_F, v=dp.v_T,
               z=dp.z_TD, scale=scale, floor=floor)
    if want_images:
        out["images"] = wiener_fast(lam_all, Q, g, Xs) * scale
    return out


def make_dp_mixture(F, T, M, K, decoder, seed=0):
    """BASELINE config 4 generator: speech PSD u v exp(dec(z)), z ~ N(0, I),
    u = v = 1; noise NMF K (Gamma(1,1)); per-source A A^H + 1e-3 I SCMs;
    circular complex Gaussian excitation (config 0 generator otherwise)."""
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((T, decoder.latent_dim))
    lam0 = decoder(z).T  # (F, T)
    Wn = rng.gamma(1.0, 1.0, (F, K))
    Hn = rng.gamma(1.0, 1.0, (K, T))
    lam = np.stack([lam0, Wn @ Hn])
    A = (rng.standard_normal((2, F, M, M)) + 1j * rng.standard_normal((2, F, M, M))) / np.sqrt(2.0)
    R = A @ np.conj(A.swapaxes(-1, -2)) + 1e-3 * np.eye(M)
    L = np.linalg.cholesky(R)
    X = np.zeros((F, T, M), dtype=np.complex128)
    for n in range(2):
        zz = (rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))) / np.sqrt(2.0)
        X += np.sqrt(lam[n])[..., None] * np.einsum("fij,ftj->fti", L[n], zz)
    return X


def dp_init(F, T, M, K, latent_dim=16, seed=0):
    """Q = I, one-hot g (N = 2) with the 1e-2 floor, u = v = 1, z = 0,
    noise W, H ~ U(0,1) from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    Q = np.tile(np.eye(M, dtype=np.complex128), (F, 1, 1))
    g = np.full((2, F, M), 1e-2)
    for m in range(M):
        g[m % 2, :, m] = 1.0
    W = rng.uniform(0.0, 1.0, (1, F, K))
    H = rng.uniform(0.0, 1.0, (1, K, T))
    return Q, g, np.ones(F), np.ones(T), np.zeros((T, latent_dim)), W, H
