"""Seeded synthetic mixtures and the BASELINE.json initialisation.

The reference package has no generator for these configs;
BASELINE.json config 0 defines it and every other config inherits it:

* W ~ Gamma(1,1) (N,F,K), H ~ Gamma(1,1) (N,K,T), lambda = W H;
* per (n, f): A circular complex standard normal (M x M), R = A A^H + 1e-3 I,
  L = chol(R);
* x_ft = sum_n sqrt(lambda_nft) L_nf z_nft, z circular complex standard normal.

The pattern follows the reference's exact sampler ``synth.sample_from_model``
(``pkg/src/fastsep/synth.py:42-67``). Init: Q_f = I; g = 1e-2 with
g[m % N, :, m] = 1 (``spatial.py:118-120``); W, H ~ U(0,1) from
``default_rng(seed)``.

``make_mixture`` (numpy, float64) is the parity-grade generator; the torch
variant draws the same distributions on the GPU for the configs too large to
sample on the host in seconds (bench only; the oracle never sees those).
"""

import numpy as np

CONFIGS = {
    # name: (F, T, M, N, K, precision, iterations)
    "c0": dict(F=257, T=128, M=4, N=2, K=8, precision="complex128", iterations=50, batch=1),
    "c1": dict(F=513, T=1024, M=8, N=4, K=16, precision="complex64", iterations=100, batch=1),
    "c2": dict(F=513, T=512, M=4, N=3, K=8, precision="complex64", iterations=100, batch=256),
    "c3": dict(F=1025, T=8192, M=16, N=6, K=32, precision="complex64", iterations=100, batch=1),
    # FastMNMF-DP: speech (deep prior, D=16 -> 128 -> 128 -> F) + NMF noise K=32
    "c4": dict(F=513, T=512, M=8, N=2, K=32, precision="complex64", iterations=100, batch=1),
}


def make_mixture(F, T, M, N, K, seed=0):
    """Config-0 generator in float64 numpy; returns X (F,T,M) complex128."""
    rng = np.random.default_rng(seed)
    W = rng.gamma(1.0, 1.0, (N, F, K))
    H = rng.gamma(1.0, 1.0, (N, K, T))
    lam = W @ H  # (N,F,T)
    A = (rng.standard_normal((N, F, M, M)) + 1j * rng.standard_normal((N, F, M, M))) / np.sqrt(2.0)
    R = A @ np.conj(A.swapaxes(-1, -2)) + 1e-3 * np.eye(M)
    L = np.linalg.cholesky(R)
    X = np.zeros((F, T, M), dtype=np.complex128)
    for n in range(N):  # one source at a time keeps the peak memory at one image
        z = (rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))) / np.sqrt(2.0)
        X += np.sqrt(lam[n])[..., None] * np.einsum("fij,ftj->fti", L[n], z)
    return X


def make_mixture_fast(F, T, M, N, K, seed=0, dtype=np.complex64):
    """The config-0 generator with the same draws as ``make_mixture`` (same
    seed, same order) but the per-bin mixing as a batched matmul, and the
    result cast to ``dtype`` source by source. Used for the full-shape configs
    2-4 (config 3's einsum takes minutes on the host); equal to
    ``make_mixture`` up to float64 rounding."""
    rng = np.random.default_rng(seed)
    W = rng.gamma(1.0, 1.0, (N, F, K))
    H = rng.gamma(1.0, 1.0, (N, K, T))
    A = (rng.standard_normal((N, F, M, M)) + 1j * rng.standard_normal((N, F, M, M))) / np.sqrt(2.0)
    R = A @ np.conj(A.swapaxes(-1, -2)) + 1e-3 * np.eye(M)
    L = np.linalg.cholesky(R)
    X = np.zeros((F, T, M), dtype=np.complex128)
    for n in range(N):
        z = (rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))) / np.sqrt(2.0)
        z = np.matmul(z, L[n].swapaxes(-1, -2))
        z *= np.sqrt(W[n] @ H[n])[..., None]
        X += z
        del z
    return X.astype(dtype, copy=False)


def make_mixture_torch(F, T, M, N, K, seed=0, device="cuda", dtype=None):
    """Same distributions drawn on the device (bench-scale configs)."""
    import torch

    cdt = dtype or torch.complex64
    rdt = torch.float32 if cdt == torch.complex64 else torch.float64
    gen = torch.Generator(device=device)
    gen.manual_seed(int(seed))
    W = torch.empty((N, F, K), device=device, dtype=rdt).exponential_(1.0, generator=gen)
    H = torch.empty((N, K, T), device=device, dtype=rdt).exponential_(1.0, generator=gen)
    lam = torch.bmm(W, H)
    A = torch.complex(torch.randn((N, F, M, M), device=device, dtype=rdt, generator=gen),
                      torch.randn((N, F, M, M), device=device, dtype=rdt, generator=gen)) / np.sqrt(2.0)
    R = A @ A.conj().transpose(-1, -2) + 1e-3 * torch.eye(M, device=device, dtype=cdt)
    L = torch.linalg.cholesky(R)
    X = torch.zeros((F, T, M), device=device, dtype=cdt)
    for n in range(N):
        z = torch.complex(torch.randn((F, T, M), device=device, dtype=rdt, generator=gen),
                          torch.randn((F, T, M), device=device, dtype=rdt, generator=gen)) / np.sqrt(2.0)
        X += lam[n].sqrt().unsqueeze(-1).to(cdt) * torch.einsum("fij,ftj->fti", L[n], z)
    return X


def baseline_init(F, T, M, N, K, seed=0):
    """(Q0, g0, W0, H0) of BASELINE.json config 0 (float64/complex128)."""
    rng = np.random.default_rng(seed)
    Q = np.tile(np.eye(M, dtype=np.complex128), (F, 1, 1))
    g = np.full((N, F, M), 1e-2)
    for m in range(M):
        g[m % N, :, m] = 1.0
    W = rng.uniform(0.0, 1.0, (N, F, K))
    H = rng.uniform(0.0, 1.0, (N, K, T))
    return Q, g, W, H


def make_dp_mixture(F, T, M, K, decoder, seed=0):
    """BASELINE config 4: speech PSD u v exp(dec(z)) at z ~ N(0, I) with
    u = v = 1, noise NMF K (Gamma(1,1)), otherwise the config-0 generator."""
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((T, decoder.latent_dim))
    lam0 = decoder(z).T
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
    """(Q, g, u, v, z, W, H) for config 4: Q = I, one-hot g (N = 2) with the
    1e-2 floor, u = v = 1, z = 0, noise W, H ~ U(0,1) from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    Q = np.tile(np.eye(M, dtype=np.complex128), (F, 1, 1))
    g = np.full((2, F, M), 1e-2)
    for m in range(M):
        g[m % 2, :, m] = 1.0
    W = rng.uniform(0.0, 1.0, (1, F, K))
    H = rng.uniform(0.0, 1.0, (1, K, T))
    return Q, g, np.ones(F), np.ones(T), np.zeros((T, latent_dim)), W, H
