"""The fused five-pass schedule (FM_SCHEDULE=fused: k_hpass, k_gpass, k_vacc,
k_ip, k_bpass; fm_fused.cuh) against the same reference goldens as the
default split schedule: the compile-time shape builds (c0 c128, c1 c64), the
generic build (ragged T, odd M, K not a multiple of 4, N = 8 / K = 64 source
groups), the split-phase sharded path and a mid-run state assignment
(fm_refresh). Tolerances as tests/test_gpu_run.py."""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import fastmnmf_oracle as O
from paper_1903_03237_b200.synth import baseline_init, make_mixture

import test_gpu_run as R

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def fused(monkeypatch):
    monkeypatch.setenv("FM_SCHEDULE", "fused")


@pytest.mark.parametrize("name,kw", [
    ("run_small_a.npz", {}), ("run_small_b.npz", {"normalize": False}),
    ("run_small_c.npz", {"ip_sweeps": 2}), ("run_small_d.npz", {}),
])
def test_fused_small_runs_c128(name, kw):
    G = golden(name)
    res, state, _ = R._run(G, "complex128", **kw)
    R._compare(G, res, state, 1e-8)


def test_fused_config0_c128():
    G = golden("run_c0.npz")
    res, state, X = R._run(G, "complex128")
    R._compare(G, res, state, 1e-6)
    assert np.abs(res.images_NFTM.sum(axis=0) - X).max() < 1e-9


def test_fused_config1_c64():
    G = golden("run_c1_c64.npz")
    res, state, _ = R._run(G, "complex64")
    R._compare(G, res, state, 1e-3)


@pytest.mark.parametrize("F,T,M,N,K,prec", [
    (9, 77, 3, 2, 5, "complex128"),     # ragged T, odd M, K % 4 != 0
    (13, 100, 5, 3, 6, "complex64"),
    (7, 64, 16, 8, 64, "complex64"),    # N = 8, K = 64: k_hpass source groups
    (11, 40, 12, 7, 9, "complex128"),
])
def test_fused_generic_shapes_vs_oracle(F, T, M, N, K, prec):
    from paper_1903_03237_b200 import SeparatorConfig, run
    it, seed = 4, 21
    X = make_mixture(F, T, M, N, K, seed)
    if prec == "complex64":
        X = X.astype(np.complex64)
    init = baseline_init(F, T, M, N, K, seed)
    ref = O.run_fastmnmf(X.astype(np.complex128), *init, n_iterations=it)
    res = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=it, precision=prec), X, init=init)
    tol = 1e-9 if prec == "complex128" else 1e-3
    tr = ref["likelihood_trace"]
    assert np.max(np.abs(res.likelihood_trace - tr) / np.abs(tr)) <= tol
    assert rel(res.images_NFTM, ref["images"]) <= tol
    assert rel(res.loop.W[0].cpu().numpy(), ref["W"]) <= tol
    assert rel(res.loop.H[0].cpu().numpy(), ref["H"]) <= tol


def test_fused_state_assignment_refreshes():
    """Assigning W between iterations (the reference loop's attributes are
    plain arrays) re-derives the fused path's W step: the continued run equals
    a fresh run from the assigned state."""
    from paper_1903_03237_b200.separate import DeviceLoop
    import torch
    F, T, M, N, K, seed = 17, 64, 4, 2, 4, 3
    X = make_mixture(F, T, M, N, K, seed)
    Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, seed)
    dev = torch.device("cuda", 0)
    Xd = torch.from_numpy(X).to(dev)[None].contiguous()
    fl = torch.tensor([1e-12 * float((np.abs(X) ** 2).max())], dtype=torch.float64)
    t = lambda a: torch.from_numpy(np.asarray(a))[None]
    a = DeviceLoop(Xd, t(Q0), t(g0), t(W0), t(H0), fl, True, 1, n_trace=8)
    a.iterate()
    a.iterate()
    a.source.W_NFK = a.source.W_NFK * 1.5
    st = (a.spatial.Q_FMM, a.spatial.g_NFM, a.source.W_NFK, a.source.H_NKT)
    ll_a = a.iterate()
    b = DeviceLoop(Xd, *(t(v) for v in st), fl, True, 1, n_trace=8)
    ll_b = b.iterate()
    assert abs(ll_a - ll_b) <= 1e-12 * abs(ll_b)
    np.testing.assert_allclose(a.source.W_NFK, b.source.W_NFK, rtol=1e-12)


@pytest.mark.parametrize("unroll", ["4", "16"])
def test_unrolled_graph_matches_single(unroll, monkeypatch):
    """FM_UNROLL: several iterations captured per CUDA graph (plus single-
    iteration graphs for the remainder) give bit-identical state and trace to
    one graph per iteration."""
    from paper_1903_03237_b200.separate import DeviceLoop
    import torch
    F, T, M, N, K, seed, it = 19, 96, 4, 2, 4, 5, 10
    X = make_mixture(F, T, M, N, K, seed)
    Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, seed)
    dev = torch.device("cuda", 0)
    Xd = torch.from_numpy(X).to(dev)[None].contiguous()
    fl = torch.tensor([1e-12 * float((np.abs(X) ** 2).max())], dtype=torch.float64)
    t = lambda a: torch.from_numpy(np.asarray(a))[None]
    out = []
    for u in ("1", unroll):
        monkeypatch.setenv("FM_UNROLL", u)
        lp = DeviceLoop(Xd, t(Q0), t(g0), t(W0), t(H0), fl, True, 1, n_trace=it)
        lp.prologue()
        lp.run(it, use_graph=True)
        torch.cuda.synchronize()
        assert lp.status_error() is None
        out.append((lp.trace[:, 0].cpu().numpy().copy(), lp.source.W_NFK.copy(), lp.spatial.Q_FMM.copy()))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])
    np.testing.assert_array_equal(out[0][2], out[1][2])
