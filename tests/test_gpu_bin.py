"""The per-bin schedule (FM_SCHEDULE=bin: k_hstats, k_binw, k_trace;
fm_bin.cuh) against the same reference goldens and oracle runs as the split
schedule: BASELINE config 0 in complex64 (N = 2, K = 8), the full config-2
shape (N = 3, K = 8, a batch of mixtures), every channel count M = 1..4 with
N = 2..4, ragged T and K < 8 (zero-padded basis rows), normalize=False,
ip_sweeps=2, a mid-run state assignment (fm_refresh) and the schedule
selection itself. Tolerance 1e-3 (BASELINE north_star, complex64)."""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import fastmnmf_oracle as O
from paper_1903_03237_b200.synth import baseline_init, make_mixture

import test_gpu_run as R

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def binsched(monkeypatch):
    monkeypatch.setenv("FM_SCHEDULE", "bin")


def _schedule(F, T, M, N, K, prec="complex64", B=1):
    import ctypes

    from paper_1903_03237_b200 import _lib
    d = _lib.FmDims()
    d.dtype = 0 if prec == "complex64" else 1
    d.B, d.F, d.T, d.M, d.N, d.K = B, F, T, M, N, K
    d.normalize, d.ip_sweeps = 1, 1
    return _lib.SCHEDULES[_lib.load().fm_schedule(ctypes.byref(d))]


def test_schedule_selection():
    assert _schedule(257, 128, 4, 2, 8) == "bin"
    assert _schedule(513, 512, 4, 3, 8) == "bin"
    assert _schedule(257, 128, 4, 2, 8, "complex128") == "split"  # complex64 only
    assert _schedule(513, 1024, 8, 4, 16) == "split"              # M > 4
    assert _schedule(64, 64, 4, 2, 12) == "split"                 # K > 8
    assert _schedule(64, 64, 4, 1, 4) == "split"                  # N < 2


def test_default_schedule(monkeypatch):
    """Without FM_SCHEDULE: per-bin once the batch holds >= 4096 (bin,
    mixture) pairs (config 2), split below and wherever bin is ineligible."""
    monkeypatch.delenv("FM_SCHEDULE")
    assert _schedule(513, 512, 4, 3, 8, B=256) == "bin"
    assert _schedule(513, 512, 4, 3, 8, B=8) == "bin"
    assert _schedule(513, 512, 4, 3, 8, B=4) == "split"
    assert _schedule(513, 512, 4, 3, 8) == "split"
    assert _schedule(513, 1024, 8, 4, 16, B=64) == "split"


def test_bin_config0_c64():
    G = golden("run_c0_c64.npz")
    res, state, _ = R._run(G, "complex64")
    assert res.loop.schedule == "bin"
    R._compare(G, res, state, 1e-3)


@pytest.mark.parametrize("F,T,M,N,K", [
    (9, 77, 1, 2, 5),    # ragged T, M = 1
    (13, 100, 2, 3, 6),
    (11, 64, 3, 4, 8),   # odd M, N = 4
    (17, 96, 4, 3, 3),   # K < 4
    (40, 33, 4, 2, 8),   # T < 32 + 1: lanes without a second frame
    (70, 50, 4, 4, 7),   # bins beyond one CTA's 8 warps
])
def test_bin_shapes_vs_oracle(F, T, M, N, K):
    from paper_1903_03237_b200 import SeparatorConfig, run
    it, seed = 6, 5
    X = make_mixture(F, T, M, N, K, seed).astype(np.complex64)
    init = baseline_init(F, T, M, N, K, seed)
    ref = O.run_fastmnmf(X.astype(np.complex128), *init, n_iterations=it)
    res = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=it, precision="complex64"), X,
              init=init)
    assert res.loop.schedule == "bin"
    tr = ref["likelihood_trace"]
    assert np.max(np.abs(res.likelihood_trace - tr) / np.abs(tr)) <= 1e-3
    assert rel(res.images_NFTM, ref["images"]) <= 1e-3
    for k, t in (("W", res.loop.W), ("H", res.loop.H), ("g", res.loop.g), ("Q", res.loop.Q)):
        assert rel(t[0].cpu().numpy(), ref[k]) <= 1e-3, k


@pytest.mark.parametrize("kw", [{"normalize": False}, {"ip_sweeps": 2}])
def test_bin_options_vs_oracle(kw):
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, T, M, N, K, it, seed = 21, 80, 4, 3, 6, 5, 9
    X = make_mixture(F, T, M, N, K, seed).astype(np.complex64)
    init = baseline_init(F, T, M, N, K, seed)
    ref = O.run_fastmnmf(X.astype(np.complex128), *init, n_iterations=it, **kw)
    res = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=it, precision="complex64", **kw),
              X, init=init)
    assert res.loop.schedule == "bin"
    tr = ref["likelihood_trace"]
    assert np.max(np.abs(res.likelihood_trace - tr) / np.abs(tr)) <= 1e-3
    assert rel(res.images_NFTM, ref["images"]) <= 1e-3


def test_bin_config2_batch_full_shape():
    import test_gpu_fullshape as FS
    FS.test_config2_batch_full_shape()


def test_bin_state_assignment_refreshes():
    """Assigning W between iterations re-derives the per-bin schedule's W step
    (Wn, phi): the continued run equals a fresh run from the assigned state."""
    import torch

    from paper_1903_03237_b200.separate import DeviceLoop
    F, T, M, N, K, seed = 17, 64, 4, 2, 4, 3
    X = make_mixture(F, T, M, N, K, seed).astype(np.complex64)
    Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, seed)
    dev = torch.device("cuda", 0)
    Xd = torch.from_numpy(X).to(dev)[None].contiguous()
    fl = torch.tensor([1e-12 * float((np.abs(X) ** 2).max())], dtype=torch.float64)
    t = lambda a: torch.from_numpy(np.asarray(a))[None]
    a = DeviceLoop(Xd, t(Q0), t(g0), t(W0), t(H0), fl, True, 1, n_trace=8)
    assert a.schedule == "bin"
    a.iterate()
    a.iterate()
    a.source.W_NFK = a.source.W_NFK * 1.5
    st = (a.spatial.Q_FMM, a.spatial.g_NFM, a.source.W_NFK, a.source.H_NKT)
    ll_a = a.iterate()
    b = DeviceLoop(Xd, *(t(v) for v in st), fl, True, 1, n_trace=8)
    ll_b = b.iterate()
    assert abs(ll_a - ll_b) <= 1e-6 * abs(ll_b)
    np.testing.assert_allclose(a.source.W_NFK, b.source.W_NFK, rtol=1e-6)


def test_bin_matches_split_schedule(monkeypatch):
    """The per-bin and the split schedule give the same run up to fp32
    summation order."""
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, T, M, N, K, it, seed = 64, 256, 4, 3, 8, 20, 2
    X = make_mixture(F, T, M, N, K, seed).astype(np.complex64)
    init = baseline_init(F, T, M, N, K, seed)
    cfg = SeparatorConfig(n_sources=N, n_basis=K, n_iterations=it, precision="complex64")
    rb = run(cfg, X, init=init)
    assert rb.loop.schedule == "bin"
    monkeypatch.setenv("FM_SCHEDULE", "split")
    rs = run(cfg, X, init=init)
    assert rs.loop.schedule == "split"
    assert np.max(np.abs(rb.likelihood_trace - rs.likelihood_trace) / np.abs(rs.likelihood_trace)) <= 1e-4
    assert rel(rb.images_NFTM, rs.images_NFTM) <= 1e-4
