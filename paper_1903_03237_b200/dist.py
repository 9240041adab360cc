"""Multi-GPU FastMNMF over torch.distributed (one process per GPU, NCCL).

Two sharding modes:

* **mixture batch** (BASELINE config 2): independent mixtures are split into
  contiguous blocks per rank; no data-path collective at all.
* **frequency** (config 3): rank r owns a contiguous block of bins
  [f0, f1). Q, g, W, X and x~ are per-frequency and stay local; H is
  replicated. The one exchange per iteration is the sum over F of the H
  statistics (sources.py:196-197): the packed [num_H | den_H] (B,2,N,K,T)
  buffer is all-reduced between the two phases of ``fm_iterate_phase``.
  One-time collectives: sum|X|^2 (separate.py:289) and max|Xs|^2
  (spatial.py:64-66); at the end the likelihood-trace partials are summed
  and the first failure (minimum status key) is taken across ranks.

The orchestration is written against a small ``ShardBackend`` protocol so
the host logic can be exercised on CPU with gloo (tests/test_dist_cpu.py);
``DeviceShardBackend`` is the production backend on libfastmnmf.so.
"""

import ctypes

import numpy as np

from . import _lib


def shard_range(F, rank, world):
    """Contiguous block of bins of ``rank``: sizes differ by at most one
    (F=1025 over 8 ranks -> 129,128,...; SURVEY §8(e) load balance)."""
    base, extra = divmod(int(F), int(world))
    f0 = rank * base + min(rank, extra)
    return f0, f0 + base + (1 if rank < extra else 0)


def shard_batch(B, rank, world):
    """Contiguous block of mixtures of ``rank``."""
    return shard_range(B, rank, world)


class DeviceShardBackend:
    """libfastmnmf.so operations for one frequency shard."""

    def __init__(self, torch):
        self.torch = torch

    def observation_stats(self, X):
        B, F, T, M = X.shape
        dims = _lib.FmDims(B, F, T, M, 1, 1, 0,
                           _lib.FM_F32 if X.dtype == self.torch.complex64 else _lib.FM_F64,
                           1, 1, 0)
        s = (ctypes.c_double * B)()
        m = (ctypes.c_double * B)()
        _lib.check(_lib.load().fm_observation_stats(ctypes.byref(dims), _lib.ptr(X), s, m,
                                                    _lib.stream_ptr()), "fm_observation_stats")
        return np.array(s[:]), np.array(m[:])

    def scale(self, X, scale):
        B, F, T, M = X.shape
        dims = _lib.FmDims(B, F, T, M, 1, 1, 0,
                           _lib.FM_F32 if X.dtype == self.torch.complex64 else _lib.FM_F64,
                           1, 1, 0)
        sc = (ctypes.c_double * B)(*[float(v) for v in scale])
        _lib.check(_lib.load().fm_scale_observation(ctypes.byref(dims), _lib.ptr(X), sc,
                                                    _lib.stream_ptr()), "fm_scale_observation")

    def make_loop(self, X, Q, g, W, H, floor, normalize, ip_sweeps, n_trace, f_offset, allreduce):
        from .separate import DeviceLoop

        t = self.torch
        return DeviceLoop(X, Q, g, W, H, t.as_tensor(floor, dtype=t.float64), normalize,
                          ip_sweeps, n_trace=n_trace, f_offset=f_offset, hstat_allreduce=allreduce)


class _Reducer:
    """The H-statistic all-reduce callable, tagged with whether it may be
    captured into a CUDA graph."""

    def __init__(self, fn, capturable):
        self.fn, self.capturable = fn, capturable

    def __call__(self, buf):
        self.fn(buf)


class FrequencyShardedRun:
    """Frequency-sharded fast-mnmf over ``world`` ranks (config 3).

    ``X_local`` (B, F_local, T, M) holds this rank's bins; ``F_global`` the
    total. The init slices must come from one global seeded init so that the
    sharded run equals the unsharded one up to summation order.
    """

    def __init__(self, X_local, init_local, F_global, rank, world, group=None, backend=None,
                 normalize=True, ip_sweeps=1, n_iterations=100):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.rank, self.world = rank, world
        self.backend = backend or DeviceShardBackend(torch)
        B, F_loc, T, M = X_local.shape
        self.f0, self.f1 = shard_range(F_global, rank, world)
        assert self.f1 - self.f0 == F_loc, "X_local does not match this rank's bin block"
        # run() prologue with global reductions (separate.py:289-293, spatial.py:64-66)
        sumsq, _ = self.backend.observation_stats(X_local)
        tot = torch.tensor(sumsq, dtype=torch.float64, device=self._dev(X_local))
        dist.all_reduce(tot, group=group)
        power = tot.cpu().numpy() / float(F_global * T * M)
        self.scale = np.sqrt(power)
        self.backend.scale(X_local, self.scale)
        _, maxsq = self.backend.observation_stats(X_local)
        mx = torch.tensor(maxsq, dtype=torch.float64, device=self._dev(X_local))
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        self.floor = 1e-12 * mx.cpu().numpy()
        Q, g, W, H = init_local
        self.loop = self.backend.make_loop(X_local, Q, g, W, H, self.floor, normalize, ip_sweeps,
                                           n_iterations, self.f0,
                                           _Reducer(self._allreduce, self.capturable))
        self.n_iterations = n_iterations

    @staticmethod
    def _dev(t):
        return t.device if hasattr(t, "device") else "cpu"

    def _allreduce(self, buf):
        self.dist.all_reduce(buf, group=self.group)

    @property
    def capturable(self):
        """NCCL collectives can be captured into a CUDA graph with the
        kernels around them; gloo's cannot."""
        try:
            return self.dist.get_backend(self.group) == "nccl"
        except Exception:
            return False

    def run(self, n=None, use_graph=True):
        """prologue + n iterations; with NCCL the per-iteration phase 0 ->
        all-reduce -> phase 1 is one captured CUDA graph replayed n times."""
        n = self.n_iterations if n is None else n
        self.loop.prologue()
        if hasattr(self.loop, "hstat"):  # DeviceLoop
            self.loop.run(n, use_graph=use_graph)
        else:
            self.loop.run(n)

    def trace(self):
        """Global likelihood trace (B, iterations): sum of the shard partials."""
        t = self.loop.trace.clone()
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy().T

    def first_error(self):
        """The first failure over all ranks (minimum unsigned status key)."""
        torch = self.torch
        st = self.loop.status.clone()
        allv = [torch.zeros_like(st) for _ in range(self.world)]
        self.dist.all_gather(allv, st, group=self.group)
        keys = [int(v.item()) & 0xFFFFFFFFFFFFFFFF for v in allv]
        k = min(keys)
        if k == _lib.FM_STATUS_CLEAR:
            return None
        from . import kernels as K
        from .errors import SingularMatrixError

        code, it, m, f = K.decode_status(k)
        return SingularMatrixError(f"iteration {it}: {K.status_message(code, m, f)}")
