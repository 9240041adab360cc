"""The frequency-sharded run (dist.FrequencyShardedRun: fm_iterate_phase(0),
an NCCL all-reduce of the packed H statistics, fm_iterate_phase(1), global
prologue reductions) on a real GPU with an NCCL process group. Only one GPU
is available to the tests, so the group has world_size 1: the NCCL calls and
the split-phase kernels run for real and must reproduce the unsharded fused
iteration. Multi-rank sharding logic is covered by test_dist_cpu.py (gloo)."""

import socket

import numpy as np
import pytest

from conftest import rel
from paper_1903_03237_b200.synth import baseline_init, make_mixture

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("precision", ["complex64", "complex128"])
def test_frequency_sharded_nccl_matches_fused(precision):
    import torch
    import torch.distributed as dist

    from paper_1903_03237_b200 import SeparatorConfig, run
    from paper_1903_03237_b200.dist import FrequencyShardedRun

    F, T, M, N, K, seed, it = 33, 96, 4, 3, 4, 5, 6
    X = make_mixture(F, T, M, N, K, seed)
    cdt = torch.complex64 if precision == "complex64" else torch.complex128
    Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, seed)
    cfg = SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K, n_iterations=it,
                          precision=precision)
    st = {}

    def snap(i, loop):
        st.update(W=loop.source.W_NFK, H=loop.source.H_NKT, g=loop.spatial.g_NFM,
                  Q=loop.spatial.Q_FMM)

    ref = run(cfg, X.astype(np.complex64 if precision == "complex64" else np.complex128),
              init=(Q0, g0, W0, H0), on_iteration=snap)

    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                            world_size=1)
    try:
        dev = torch.device("cuda", 0)
        Xd = torch.from_numpy(X).to(dev, cdt)[None].contiguous()
        init = tuple(torch.from_numpy(np.asarray(a))[None] for a in (Q0, g0, W0, H0))
        runner = FrequencyShardedRun(Xd, init, F, 0, 1, n_iterations=it)
        runner.run()
        torch.cuda.synchronize()
        assert runner.first_error() is None
        tr = runner.trace()[0]
        lp = runner.loop
        got = dict(W=lp.W[0].cpu().numpy(), H=lp.H[0].cpu().numpy(), g=lp.g[0].cpu().numpy(),
                   Q=lp.Q[0].cpu().numpy())
    finally:
        dist.destroy_process_group()
    tol = 1e-5 if precision == "complex64" else 1e-12
    assert np.max(np.abs(tr - ref.likelihood_trace) / np.abs(ref.likelihood_trace)) <= tol
    for k in ("W", "H", "g", "Q"):
        assert rel(got[k], st[k]) <= tol, (k, rel(got[k], st[k]))
