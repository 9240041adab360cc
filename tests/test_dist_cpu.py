"""Multi-process host logic of the frequency-sharded run on CPU.

Two gloo ranks run ``paper_1903_03237_b200.dist.FrequencyShardedRun`` -- the
production orchestration: global scale/floor reductions, the per-iteration
all-reduce of the packed H statistics between the two phases, the trace
reduction and the first-error selection -- with a CPU stand-in backend whose
per-shard phases are written with the oracle's numpy kernels (test
infrastructure only). The sharded result must equal the unsharded oracle run.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fastmnmf_oracle as O
from paper_1903_03237_b200.dist import FrequencyShardedRun, shard_batch, shard_range
from paper_1903_03237_b200.synth import baseline_init, make_mixture

TINY = O.TINY


def test_shard_range_partitions():
    for F in (1, 7, 513, 1025):
        for world in (1, 2, 3, 8):
            blocks = [shard_range(F, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == F
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    assert shard_range(1025, 0, 8) == (0, 129)
    assert shard_batch(256, 3, 8) == (96, 128)


class _CpuShardLoop:
    """One frequency shard of the FastMNMF pass in numpy (oracle formulas),
    split at the H-statistic exchange exactly like fm_iterate_phase."""

    def __init__(self, X, Q, g, W, H, floor, normalize, ip_sweeps, n_trace, f_offset, allreduce):
        self.X = X[0].numpy().astype(np.complex128)  # (F_loc, T, M), already scaled
        self.Q = np.array(Q[0], dtype=np.complex128)
        self.g = np.array(g[0], dtype=np.float64)
        self.W = np.array(W[0], dtype=np.float64)
        self.H = np.array(H[0], dtype=np.float64)
        self.floor = float(floor[0])
        self.normalize, self.ip_sweeps = normalize, ip_sweeps
        self.allreduce = allreduce
        self.trace = torch.zeros((n_trace, 1), dtype=torch.float64)
        self.status = torch.full((1,), -1, dtype=torch.int64)
        self.it = 0

    def prologue(self):
        self.xt = O.project_power(self.Q, self.X)
        self.phi1, self.phi2, _, _, _ = O.fast_stats(self.xt, self.g, self.W @ self.H, self.floor)

    def run(self, n):
        for _ in range(n):
            self._iterate()

    def _iterate(self):
        T = self.X.shape[1]
        # phase 0: W MU from the previous pass, refresh, local H statistics
        num = np.matmul(self.phi1, self.H.transpose(0, 2, 1))
        den = np.matmul(self.phi2, self.H.transpose(0, 2, 1))
        self.W = self.W * np.sqrt(num / np.maximum(den, TINY))
        p1, p2, _, _, _ = O.fast_stats(self.xt, self.g, self.W @ self.H, self.floor)
        hstat = torch.from_numpy(np.stack([np.matmul(self.W.transpose(0, 2, 1), p1),
                                           np.matmul(self.W.transpose(0, 2, 1), p2)])[None])
        self.allreduce(hstat)  # <- the one exchange per iteration
        numH, denH = hstat[0, 0].numpy(), hstat[0, 1].numpy()
        self.H = self.H * np.sqrt(numH / np.maximum(denH, TINY))
        # phase 1: per-frequency rest of the pass
        lam = self.W @ self.H
        _, _, gn, gd, _ = O.fast_stats(self.xt, self.g, lam, self.floor, want_gain=True,
                                       want_phi=False)
        self.g = self.g * np.sqrt(gn / np.maximum(gd, TINY))
        y = O.mix_power(lam, self.g, self.floor)
        self.Q = O.update_diagonalizer(self.Q, self.X, y, self.ip_sweeps)
        if self.normalize:
            row = np.sqrt(np.einsum("fmj,fmj->fm", self.Q, self.Q.conj()).real)
            self.Q = self.Q / row[:, :, None]
            self.g = self.g / np.square(row)[None]
        self.xt = O.project_power(self.Q, self.X)
        if self.normalize:
            self.g, c = O.normalize_gains(self.g)
            self.W = self.W * c[:, :, None]
        self.phi1, self.phi2, _, _, ll = O.fast_stats(self.xt, self.g, self.W @ self.H, self.floor)
        self.trace[self.it, 0] = ll + 2.0 * T * float(np.linalg.slogdet(self.Q)[1].sum())
        self.it += 1


class _CpuBackend:
    def observation_stats(self, X):
        a = np.abs(X.numpy()) ** 2
        return a.reshape(a.shape[0], -1).sum(1), a.reshape(a.shape[0], -1).max(1)

    def scale(self, X, scale):
        X /= torch.as_tensor(scale, dtype=torch.float64)[:, None, None, None]

    def make_loop(self, X, Q, g, W, H, floor, normalize, ip_sweeps, n_trace, f_offset, allreduce):
        return _CpuShardLoop(X, Q, g, W, H, floor, normalize, ip_sweeps, n_trace, f_offset,
                             allreduce)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        F, T, M, N, K, it = 10, 40, 3, 2, 4, 4
        X = make_mixture(F, T, M, N, K, seed=11)
        Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, 11)
        f0, f1 = shard_range(F, rank, world)
        Xl = torch.from_numpy(X[f0:f1].copy())[None]
        init = (Q0[None, f0:f1], g0[None, :, f0:f1], W0[None, :, f0:f1], H0[None])
        run = FrequencyShardedRun(Xl, init, F, rank, world, backend=_CpuBackend(),
                                  n_iterations=it)
        run.run()
        trace = run.trace()[0]
        lp = run.loop
        q.put((rank, f0, f1, trace, lp.Q, lp.g, lp.W, lp.H, run.first_error()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_frequency_sharded_equals_unsharded_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda o: o[0])
    F, T, M, N, K, it = 10, 40, 3, 2, 4, 4
    X = make_mixture(F, T, M, N, K, seed=11)
    ref = O.run_fastmnmf(X, *baseline_init(F, T, M, N, K, 11), n_iterations=it, want_images=False)
    for o in outs:  # every rank sees the same global trace and the same H
        np.testing.assert_allclose(o[3], ref["likelihood_trace"], rtol=1e-10)
        np.testing.assert_allclose(o[7], ref["H"], rtol=1e-10)
        assert o[8] is None
    Q = np.concatenate([o[4] for o in outs], axis=0)
    g = np.concatenate([o[5] for o in outs], axis=1)
    W = np.concatenate([o[6] for o in outs], axis=1)
    np.testing.assert_allclose(Q, ref["Q"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(g, ref["g"], rtol=1e-9)
    np.testing.assert_allclose(W, ref["W"], rtol=1e-9)
