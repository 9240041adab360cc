"""FastMNMF-DP on B200 (BASELINE config 4).

Source 0 is the deep prior lambda_0[f,t] = u_f v_t exp(dec(z_t))_f
(``DeepPriorFactors``, ``sources.py:207-220``, with the config-4 decoder
D -> 128 tanh -> 128 tanh -> F linear); sources 1.. are NMF noise
(``DeepPriorPlusNmfSource``, ``sources.py:223-271``). At the reference's
latent hook (``separate.py:205-213``) the latents take ``adam_steps`` Adam
steps on the FastMNMF negative log-likelihood against the frozen
rest-of-model power (config 4 replaces the Metropolis chain,
``sources.py:292-339``). Everything runs in libfastmnmf.so
(``fm_prologue_dp`` / ``fm_iterate_dp`` / ``fm_run_dp``).
"""

import ctypes

import numpy as np

from . import _lib


class ExpMLPDecoder:
    """The config-4 decoder: z (T, D) -> exp(W3 tanh(W2 tanh(W1 z + b1) + b2) + b3).

    Xavier-normal weights drawn from ``default_rng(seed)`` in the order W1, W2,
    W3 (std sqrt(2 / (fan_in + fan_out))), zero biases. It satisfies the
    reference's decoder interface (a callable with ``latent_dim`` and
    ``n_freq``, ``separate.py:265-273``). ``__call__`` evaluates on the host
    for data synthesis only; the separator evaluates it on the device.
    """

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
    def hidden(self):
        return self.W1.shape[0]

    @property
    def n_freq(self):
        return self.W3.shape[0]

    def __call__(self, z):
        z = np.asarray(z, dtype=np.float64)
        h = np.tanh(np.tanh(z @ self.W1.T + self.b1) @ self.W2.T + self.b2)
        return np.exp(h @ self.W3.T + self.b3)


class DeviceDP:
    """Device tensors of the deep-prior source for a batch of B mixtures."""

    def __init__(self, decoder, u, v, z, dims, real, device, adam_steps=10, lr=1e-2,
                 beta1=0.9, beta2=0.999, eps=1e-8):
        import torch

        def dev(a):
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a))
            return t.to(device, real).contiguous()

        self.decoder = decoder
        self.W1, self.b1 = dev(decoder.W1), dev(decoder.b1)
        self.W2, self.b2 = dev(decoder.W2), dev(decoder.b2)
        self.W3, self.b3 = dev(decoder.W3), dev(decoder.b3)
        B, F, T = dims.B, dims.F, dims.T
        self.u = dev(u).reshape(B, F).contiguous()
        self.v = dev(v).reshape(B, T).contiguous()
        D = decoder.latent_dim
        self.z = dev(z).reshape(B, T, D).contiguous()
        self.r = torch.empty((B, T, F), device=device, dtype=real)
        self.m = torch.zeros((B, T, D), device=device, dtype=real)
        self.v2 = torch.zeros((B, T, D), device=device, dtype=real)
        self.step = torch.zeros((1,), device=device, dtype=torch.int32)
        self.struct = _lib.FmDp(D, decoder.hidden, *[_lib.ptr(t).value for t in (
            self.W1, self.b1, self.W2, self.b2, self.W3, self.b3, self.u, self.v, self.z, self.r,
            self.m, self.v2, self.step)], None, int(adam_steps), float(lr), float(beta1),
            float(beta2), float(eps))
        nbytes = _lib.load().fm_dp_workspace_bytes(ctypes.byref(dims), ctypes.byref(self.struct))
        self.work = torch.empty((max(nbytes, 1),), dtype=torch.uint8, device=device)
        self.struct.work = _lib.ptr(self.work).value

    def lam0(self):
        """lambda_0 (B, F, T) of the current state (sources.py:219-220)."""
        return self.u[:, :, None] * (self.v[:, :, None] * self.r).transpose(1, 2)
