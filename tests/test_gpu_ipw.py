"""k_ip_w (fm_ipw.cuh: one warp per bin, batched HPD Gauss-Jordan) -- the IP
kernel of large batches (config 2) -- forced on small problems with FM_IP=w
(and the opt-in register-accumulating M <= 4 gain / V kernels, FM_SMALL=1):
every channel count M = 1..8 in both precisions against the oracle, the
rank-deficient T < M error with the reference's message and row, and an
ill-conditioned V_fm whose fp32 pivots fail and are retried in fp64."""

import numpy as np
import pytest

from conftest import rel
from oracle import fastmnmf_oracle as O
from paper_1903_03237_b200.synth import baseline_init, make_mixture

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def warp_ip(monkeypatch):
    monkeypatch.setenv("FM_IP", "w")


@pytest.mark.parametrize("prec,tol", [("complex128", 1e-9), ("complex64", 1e-3)])
@pytest.mark.parametrize("M", list(range(1, 9)))
def test_ipw_every_m_vs_oracle(M, prec, tol):
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, T, N, K, it, seed = 9, 70, 2, 3, 3, 40 + M
    X = make_mixture(F, T, M, N, K, seed)
    if prec == "complex64":
        X = X.astype(np.complex64)
    init = baseline_init(F, T, M, N, K, seed)
    ref = O.run_fastmnmf(X.astype(np.complex128), *init, n_iterations=it)
    res = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=it, precision=prec), X, init=init)
    tr = ref["likelihood_trace"]
    assert np.max(np.abs(res.likelihood_trace - tr) / np.abs(tr)) <= tol
    assert rel(res.loop.Q[0].cpu().numpy(), ref["Q"]) <= tol
    assert rel(res.images_NFTM, ref["images"]) <= tol


def test_ipw_singular_prefix():
    from paper_1903_03237_b200 import SeparatorConfig, SingularMatrixError, run
    F, T, M, N, K = 3, 3, 5, 2, 2
    X = make_mixture(F, T, M, N, K, seed=5)
    init = baseline_init(F, T, M, N, K, 5)
    with pytest.raises(SingularMatrixError) as got:
        run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=2), X, init=init)
    assert str(got.value).startswith("iteration 0: non-positive normalization")
    assert "m=0)" in str(got.value)


@pytest.mark.parametrize("ip", ["w", "cta"])
def test_ipw_ill_conditioned_v_complex64(ip, monkeypatch):
    """Two nearly collinear channels make V_fm ill-conditioned (condition
    number ~1e5, still representable in the fp32-accumulated V): the fp32
    Gauss-Jordan loses most digits of a pivot; the kernel must fall back to
    fp64 and finish like the oracle instead of raising. (Collinearity beyond
    fp32 resolution makes the complex64 V itself indefinite -- a limit of the
    precision mode, not of the solver.) Both IP kernels (k_ip_w, k_ip)."""
    monkeypatch.setenv("FM_IP", ip)
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, T, M, N, K, it = 6, 200, 4, 2, 3, 2
    rng = np.random.default_rng(7)
    X = make_mixture(F, T, M, N, K, 7)
    X[:, :, 1] = X[:, :, 0] + 3e-3 * np.abs(X[:, :, 0]).mean() * (
        rng.standard_normal((F, T)) + 1j * rng.standard_normal((F, T)))
    X = X.astype(np.complex64)
    init = baseline_init(F, T, M, N, K, 7)
    ref = O.run_fastmnmf(X.astype(np.complex128), *init, n_iterations=it)
    res = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=it, precision="complex64"), X,
              init=init)
    tr = ref["likelihood_trace"]
    assert np.all(np.isfinite(res.likelihood_trace))
    assert np.max(np.abs(res.likelihood_trace - tr) / np.abs(tr)) <= 1e-2


@pytest.mark.parametrize("prec,tol", [("complex128", 1e-9), ("complex64", 1e-3)])
@pytest.mark.parametrize("M", [1, 3, 4])
def test_small_m_register_kernels_vs_oracle(M, prec, tol, monkeypatch):
    """k_gain_r / k_vacc_r (fm_small.cuh, FM_SMALL=1): ragged bin count (not a
    multiple of the 4 bins per CTA) and frames (not a multiple of 64)."""
    monkeypatch.setenv("FM_SMALL", "1")
    monkeypatch.setenv("FM_IP", "cta")
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, T, N, K, it, seed = 10, 150, 3, 4, 3, 60 + M
    X = make_mixture(F, T, M, N, K, seed)
    if prec == "complex64":
        X = X.astype(np.complex64)
    init = baseline_init(F, T, M, N, K, seed)
    ref = O.run_fastmnmf(X.astype(np.complex128), *init, n_iterations=it)
    res = run(SeparatorConfig(n_sources=N, n_basis=K, n_iterations=it, precision=prec), X, init=init)
    tr = ref["likelihood_trace"]
    assert np.max(np.abs(res.likelihood_trace - tr) / np.abs(tr)) <= tol
    assert rel(res.loop.g[0].cpu().numpy(), ref["g"]) <= tol
    assert rel(res.images_NFTM, ref["images"]) <= tol
