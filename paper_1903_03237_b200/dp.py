"""FastMNMF-DP on B200 (BASELINE config 4).

Source 0 is the deep prior lambda_0[f,t] = u_f v_t exp(dec(z_t))_f
(``DeepPriorFactors``, ``sources.py:207-220``, with the config-4 decoder
D -> 128 tanh -> 128 tanh -> F linear); sources 1.. are NMF noise
(``DeepPriorPlusNmfSource``, ``sources.py:223-271``). At the reference's
latent hook (``separate.py:205-213``) the latents take ``adam_steps`` Adam
steps on the FastMNMF negative log-likelihood against the frozen
rest-of-model power (config 4 replaces the Metropolis chain,
``sources.py:292-339``). The reference's own default -- ``ToyDecoder``
(``sources.py:52-80``) with the Metropolis random walk
(``update_latents_fast``, ``sources.py:307-339``) -- runs too, on the device
(``k_dp_mh``), with the proposal draws taken from the reference's numpy
stream (bit-for-bit the reference's chain) or from a device Philox stream.
Everything runs in libfastmnmf.so (``fm_prologue_dp`` / ``fm_iterate_dp`` /
``fm_run_dp``).
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


class ToyDecoder:
    """The reference's default decoder (``sources.py:52-80``): z (..., D) ->
    max(softplus(tanh(z w1^T + b1) w2^T + b2), 1e-8). Same constructor, seeded
    draws and attribute names, so the weights equal the reference's for the
    same (n_freq, latent_dim, hidden, seed); any object with ``w1, b1, w2,
    b2`` (the reference's own ToyDecoder included) is accepted by ``run``."""

    OUTPUT_FLOOR = 1e-8

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
    def hidden(self):
        return self.w1.shape[0]

    @property
    def n_freq(self):
        return self.w2.shape[0]

    def __call__(self, z):
        z = np.asarray(z, dtype=np.float64)
        h = np.tanh(z @ self.w1.T + self.b1)
        o = h @ self.w2.T + self.b2
        sp = np.log1p(np.exp(-np.abs(o))) + np.maximum(o, 0.0)
        return np.maximum(sp, self.OUTPUT_FLOOR)


def decoder_kind(decoder):
    """0: exp-MLP (W1..W3, b1..b3), 1: reference ToyDecoder (w1, b1, w2, b2)."""
    if all(hasattr(decoder, a) for a in ("W1", "W2", "W3", "b1", "b2", "b3")):
        return 0
    if all(hasattr(decoder, a) for a in ("w1", "b1", "w2", "b2")):
        return 1
    return None


class DeviceDP:
    """Device tensors of the deep-prior source for a batch of B mixtures."""

    def __init__(self, decoder, u, v, z, dims, real, device, adam_steps=10, lr=1e-2,
                 beta1=0.9, beta2=0.999, eps=1e-8, mh_steps=0, mh_var=1e-4, mh_rng=None,
                 mh_seed=0):
        import torch

        def dev(a):
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a))
            return t.to(device, real).contiguous()

        self.decoder = decoder
        self.kind = decoder_kind(decoder)
        if self.kind == 0:
            self.W1, self.b1 = dev(decoder.W1), dev(decoder.b1)
            self.W2, self.b2 = dev(decoder.W2), dev(decoder.b2)
            self.W3, self.b3 = dev(decoder.W3), dev(decoder.b3)
            hidden = decoder.W1.shape[0]
        else:  # ToyDecoder: one hidden layer, output layer in the W3/b3 slots
            self.W1, self.b1 = dev(decoder.w1), dev(decoder.b1)
            self.W2 = self.b2 = None
            self.W3, self.b3 = dev(decoder.w2), dev(decoder.b2)
            hidden = np.asarray(decoder.w1).shape[0]
        B, F, T = dims.B, dims.F, dims.T
        self.u = dev(u).reshape(B, F).contiguous()
        self.v = dev(v).reshape(B, T).contiguous()
        D = decoder.latent_dim
        self.z = dev(z).reshape(B, T, D).contiguous()
        self.r = torch.empty((B, T, F), device=device, dtype=real)
        self.m = torch.zeros((B, T, D), device=device, dtype=real)
        self.v2 = torch.zeros((B, T, D), device=device, dtype=real)
        self.step = torch.zeros((1,), device=device, dtype=torch.int32)
        # Metropolis (sources.py:307-339): mh_rng = the run's numpy Generator ->
        # per-iteration draws in the reference's order (fill_draws), else Philox
        self.mh_steps, self.mh_rng = int(mh_steps), mh_rng
        self.noise = self.unif = None
        if self.mh_steps > 0 and mh_rng is not None:
            self.noise = torch.empty((self.mh_steps, B, T, D), device=device, dtype=real)
            self.unif = torch.empty((self.mh_steps, B, T), device=device, dtype=real)
            # two pinned staging buffers, each guarded by the event of the copy
            # that last read it (fill_draws must not overwrite a buffer whose
            # host->device copy is still queued behind the GPU)
            self._stage = [torch.empty((self.mh_steps * B * T * (D + 1),), dtype=real,
                                       pin_memory=True) for _ in range(2)]
            self._stage_ev = [None, None]
            self._stage_i = 0

        def p(t):
            return None if t is None else _lib.ptr(t).value

        self.struct = _lib.FmDp(D, hidden, *[p(t) for t in (
            self.W1, self.b1, self.W2, self.b2, self.W3, self.b3, self.u, self.v, self.z, self.r,
            self.m, self.v2, self.step)], None, int(adam_steps), float(lr), float(beta1),
            float(beta2), float(eps), int(self.kind), self.mh_steps, float(np.sqrt(mh_var)),
            p(self.noise), p(self.unif), int(mh_seed) & ((1 << 64) - 1))
        nbytes = _lib.load().fm_dp_workspace_bytes(ctypes.byref(dims), ctypes.byref(self.struct))
        self.work = torch.empty((max(nbytes, 1),), dtype=torch.uint8, device=device)
        self.struct.work = _lib.ptr(self.work).value

    def lam0(self):
        """lambda_0 (B, F, T) of the current state (sources.py:219-220)."""
        return self.u[:, :, None] * (self.v[:, :, None] * self.r).transpose(1, 2)

    def fill_draws(self):
        """Draw one iteration's proposals from the run's numpy Generator in the
        reference's order -- per inner step standard_normal((T, D)) then
        uniform(size=T) (sources.py:314-318) -- and upload them (stream-ordered
        before the next iteration). B = 1 (run() is one mixture)."""
        if self.noise is None:
            return
        import torch

        S, B, T, D = self.noise.shape
        n = np.empty((S, T, D))
        u = np.empty((S, T))
        for s in range(S):
            n[s] = self.mh_rng.standard_normal((T, D))
            u[s] = self.mh_rng.uniform(size=T)
        i = self._stage_i
        self._stage_i ^= 1
        if self._stage_ev[i] is not None:
            self._stage_ev[i].synchronize()  # the copy that last read this buffer is done
        st = self._stage[i]
        st[: S * T * D].copy_(torch.from_numpy(n.reshape(-1)))
        st[S * T * D:].copy_(torch.from_numpy(u.reshape(-1)))
        self.noise.view(-1).copy_(st[: S * T * D], non_blocking=True)
        self.unif.view(-1).copy_(st[S * T * D:], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._stage_ev[i] = ev
