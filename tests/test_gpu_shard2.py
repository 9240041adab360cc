"""Two frequency shards of one mixture on the device (config 3's sharding,
SURVEY §8(e)), driven in one process: each shard is a DeviceLoop over its bin
block (f_offset != 0 for the second), the per-iteration exchange is the sum of
the two shards' packed H statistics between fm_iterate_phase(0) and (1) --
what dist.FrequencyShardedRun's NCCL all-reduce computes across processes.
The sharded run must reproduce the unsharded one (sources.py:195-198 is the
only cross-bin step); both schedules, both precisions."""

import ctypes

import numpy as np
import pytest

from conftest import rel
from paper_1903_03237_b200.synth import baseline_init, make_mixture

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("schedule", ["split", "fused", "bin"])
@pytest.mark.parametrize("precision,tol", [("complex64", 1e-5), ("complex128", 1e-11)])
def test_two_shards_equal_unsharded(precision, tol, schedule, monkeypatch):
    import torch

    from paper_1903_03237_b200 import SeparatorConfig, _lib, run
    from paper_1903_03237_b200.dist import DeviceShardBackend, shard_range
    from paper_1903_03237_b200.separate import DeviceLoop

    monkeypatch.setenv("FM_SCHEDULE", schedule)
    F, T, M, N, K, seed, it = 37, 96, 4, 3, 5, 8, 5
    X = make_mixture(F, T, M, N, K, seed)
    cdt = torch.complex64 if precision == "complex64" else torch.complex128
    if precision == "complex64":
        X = X.astype(np.complex64)
    Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, seed)
    st = {}

    def snap(i, loop):
        st.update(W=loop.source.W_NFK, H=loop.source.H_NKT, g=loop.spatial.g_NFM,
                  Q=loop.spatial.Q_FMM)

    ref = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=it, precision=precision), X,
              init=(Q0, g0, W0, H0), on_iteration=snap)

    dev = torch.device("cuda", 0)
    be = DeviceShardBackend(torch)
    blocks = [shard_range(F, r, 2) for r in range(2)]
    Xl = [torch.from_numpy(np.ascontiguousarray(X[f0:f1])).to(dev, cdt)[None].contiguous()
          for f0, f1 in blocks]
    # run()'s prologue with the global reductions (separate.py:289-293)
    sumsq = sum(be.observation_stats(x)[0] for x in Xl)
    scale = np.sqrt(sumsq / float(F * T * M))
    for x in Xl:
        be.scale(x, scale)
    floor = 1e-12 * max(be.observation_stats(x)[1] for x in Xl)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))[None]
    loops = [DeviceLoop(Xl[r], t(Q0[f0:f1]), t(g0[:, f0:f1]), t(W0[:, f0:f1]), t(H0),
                        torch.as_tensor(floor, dtype=torch.float64), True, 1, n_trace=it,
                        f_offset=f0, hstat_allreduce=lambda buf: None)
             for r, (f0, f1) in enumerate(blocks)]
    assert loops[1].dims.f_offset == blocks[1][0] > 0
    lib = _lib.load()
    for lp in loops:
        lp.prologue()
    for _ in range(it):
        for lp in loops:
            _lib.check(lib.fm_iterate_phase(ctypes.byref(lp.dims), ctypes.byref(lp.state), 0,
                                            _lib.ptr(lp.hstat), _lib.stream_ptr()), "phase 0")
        total = loops[0].hstat + loops[1].hstat  # the all-reduce (sum)
        for lp in loops:
            lp.hstat.copy_(total)
            _lib.check(lib.fm_iterate_phase(ctypes.byref(lp.dims), ctypes.byref(lp.state), 1,
                                            _lib.ptr(lp.hstat), _lib.stream_ptr()), "phase 1")
    torch.cuda.synchronize()
    for lp in loops:
        assert lp.status_error() is None
    trace = (loops[0].trace + loops[1].trace)[:, 0].cpu().numpy()
    np.testing.assert_allclose(trace, ref.likelihood_trace, rtol=tol)
    cat = lambda name, ax: np.concatenate([getattr(lp, name)[0].cpu().numpy() for lp in loops], axis=ax)
    assert rel(cat("W", 1), st["W"]) <= tol
    assert rel(cat("g", 1), st["g"]) <= tol
    assert rel(cat("Q", 0), st["Q"]) <= tol
    for lp in loops:  # H is replicated and identical on both shards
        assert rel(lp.H[0].cpu().numpy(), st["H"]) <= tol
    np.testing.assert_array_equal(loops[0].H.cpu().numpy(), loops[1].H.cpu().numpy())
