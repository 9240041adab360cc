"""Pin the CPU oracle (oracle/fastmnmf_oracle.py) to the reference's own outputs.

tests/golden/*.npz were produced by oracle/make_golden.py running the
unmodified reference fastsep (kernels and run() with the SURVEY §8(c) init
injection). CPU only; no GPU.
"""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import fastmnmf_oracle as O
from paper_1903_03237_b200.synth import baseline_init, make_mixture

KG = golden("kernels.npz")


@pytest.mark.parametrize("tag", ["a", "b", "c"])
@pytest.mark.parametrize("floor", [0.0, 0.5])
@pytest.mark.parametrize("wg", [0, 1])
@pytest.mark.parametrize("wp", [0, 1])
def test_fast_stats(tag, floor, wg, wp):
    xt, g, lam = KG[f"fs_{tag}_xt"], KG[f"fs_{tag}_g"], KG[f"fs_{tag}_lam"]
    got = O.fast_stats(xt, g, lam, floor, bool(wg), bool(wp))
    key = f"fs_{tag}_{floor}_{wg}{wp}"
    for i, nm in enumerate(("phi1", "phi2", "gnum", "gden")):
        np.testing.assert_allclose(got[i], KG[f"{key}_{nm}"], rtol=1e-10, atol=1e-14)
    assert abs(got[4] - KG[f"{key}_ll"]) <= 1e-10 * abs(KG[f"{key}_ll"])


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_mix_power(tag):
    got = O.mix_power(KG[f"fs_{tag}_lam"], KG[f"fs_{tag}_g"], 0.5)
    np.testing.assert_allclose(got, KG[f"fs_{tag}_mix"], rtol=1e-13)


@pytest.mark.parametrize("tag", ["a", "b", "c", "d"])
def test_ip_weights_project_diagonalizer(tag):
    X, y, Q = KG[f"ip_{tag}_X"], KG[f"ip_{tag}_y"], KG[f"ip_{tag}_Q"]
    np.testing.assert_allclose(O.ip_weights(X, y), KG[f"ip_{tag}_V"], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(O.project_power(Q, X), KG[f"ip_{tag}_xt"], rtol=1e-10, atol=1e-13)
    for sweeps in (1, 3):
        got = O.update_diagonalizer(KG[f"ip_{tag}_Q0"], X, y, sweeps)
        assert rel(got, KG[f"ip_{tag}_Qnew{sweeps}"]) < 1e-10
    np.testing.assert_allclose(np.linalg.slogdet(Q)[1], KG[f"ip_{tag}_logdet"], rtol=1e-12)


def test_wiener_normalize_loglik():
    X, Q, g, lam = KG["wf_X"], KG["wf_Q"], KG["wf_g"], KG["wf_lam"]
    assert rel(O.wiener_fast(lam, Q, g, X), KG["wf_images"]) < 1e-12
    gn, c = O.normalize_gains(g)
    np.testing.assert_allclose(gn, KG["ng_g"], rtol=1e-14)
    np.testing.assert_allclose(c, KG["ng_c"], rtol=1e-14)
    assert abs(O.loglik_fast(X, Q, g, lam, 1e-3) - KG["ll_fast"]) <= 1e-11 * abs(KG["ll_fast"])


def _check_run(name, tol, round64=False, **kw):
    G = golden(name)
    F, T, M, N, K, seed, it = (int(v) for v in G["shape"])
    X = make_mixture(F, T, M, N, K, seed)
    if round64:
        X = X.astype(np.complex64).astype(np.complex128)
    assert abs(np.abs(X).sum() - G["X_abs_sum"]) <= 1e-10 * G["X_abs_sum"]
    np.testing.assert_allclose(X[::13, ::11, :], G["X_sample"], rtol=1e-12)
    out = O.run_fastmnmf(X, *baseline_init(F, T, M, N, K, seed), n_iterations=it, **kw)
    np.testing.assert_allclose(out["likelihood_trace"], G["trace"], rtol=tol)
    for k in ("W", "H", "g", "Q"):
        assert rel(out[k], G[k]) < max(tol, 1e-6 if round64 else tol), k
    if "images" in G:
        assert rel(out["images"], G["images"]) < tol
    else:
        assert rel(out["images"][:, ::17, ::19, :], G["img_sample"]) < max(tol, 1e-6 if round64 else tol)
    np.testing.assert_allclose(np.linalg.norm(out["images"].reshape(N, -1), axis=1), G["img_norm"],
                               rtol=max(tol, 1e-9))


@pytest.mark.parametrize("name,kw", [
    ("run_small_a.npz", {}), ("run_small_b.npz", {"normalize": False}),
    ("run_small_c.npz", {"ip_sweeps": 2}), ("run_small_d.npz", {}),
])
def test_run_small(name, kw):
    _check_run(name, 1e-9, **kw)


def test_run_config0():
    _check_run("run_c0.npz", 1e-9)


def test_run_config0_c64_input():
    _check_run("run_c0_c64.npz", 1e-9, round64=True)


def test_singular_error_t_less_than_m():
    # T < M makes V rank deficient -> SingularMatrixError
    F, T, M, N, K = 3, 3, 5, 2, 2
    X = make_mixture(F, T, M, N, K, seed=5)
    with pytest.raises(O.OracleError) as ei:
        O.run_fastmnmf(X, *baseline_init(F, T, M, N, K, 5), n_iterations=2)
    assert str(ei.value).startswith("iteration 0: ")
