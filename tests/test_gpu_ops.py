"""Per-op parity of the sm_100a kernels with the reference's kernel outputs
(tests/golden/kernels.npz, produced by the unmodified reference) and with
the CPU oracle. complex128: rtol 1e-10-ish; complex64: norm-wise 1e-5."""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import fastmnmf_oracle as O

pytestmark = pytest.mark.gpu
KG = golden("kernels.npz")


def _t(a, dtype):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


@pytest.mark.parametrize("tag", ["a", "b", "c"])
@pytest.mark.parametrize("floor", [0.0, 0.5])
@pytest.mark.parametrize("wg", [0, 1])
@pytest.mark.parametrize("wp", [0, 1])
def test_fast_stats_c128(tag, floor, wg, wp):
    from paper_1903_03237_b200 import kernels as K
    xt, g, lam = KG[f"fs_{tag}_xt"], KG[f"fs_{tag}_g"], KG[f"fs_{tag}_lam"]
    got = K.fast_stats(xt, g, lam, floor, bool(wg), bool(wp))
    key = f"fs_{tag}_{floor}_{wg}{wp}"
    for i, nm in enumerate(("phi1", "phi2", "gnum", "gden")):
        np.testing.assert_allclose(got[i], KG[f"{key}_{nm}"], rtol=1e-10, atol=1e-14)
    assert abs(got[4] - KG[f"{key}_ll"]) <= 1e-10 * abs(KG[f"{key}_ll"])


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_fast_stats_c64(tag):
    import torch
    from paper_1903_03237_b200 import kernels as K
    xt, g, lam = KG[f"fs_{tag}_xt"], KG[f"fs_{tag}_g"], KG[f"fs_{tag}_lam"]
    got = K.fast_stats(_t(xt, torch.float32), _t(g, torch.float32), _t(lam, torch.float32),
                       0.5, True, True)
    key = f"fs_{tag}_0.5_11"
    for i, nm in enumerate(("phi1", "phi2", "gnum", "gden")):
        assert rel(got[i].cpu().numpy(), KG[f"{key}_{nm}"]) < 1e-5, nm
    assert abs(got[4] - KG[f"{key}_ll"]) <= 1e-5 * abs(KG[f"{key}_ll"])


@pytest.mark.parametrize("tag", ["a", "b", "c"])
def test_mix_power(tag):
    from paper_1903_03237_b200 import kernels as K
    np.testing.assert_allclose(K.mix_power(KG[f"fs_{tag}_lam"], KG[f"fs_{tag}_g"], 0.5),
                               KG[f"fs_{tag}_mix"], rtol=1e-13)


@pytest.mark.parametrize("tag", ["a", "b", "c", "d"])
def test_ip_weights_project(tag):
    from paper_1903_03237_b200 import kernels as K
    X, y, Q = KG[f"ip_{tag}_X"], KG[f"ip_{tag}_y"], KG[f"ip_{tag}_Q"]
    np.testing.assert_allclose(K.ip_weights(X, y), KG[f"ip_{tag}_V"], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(K.project_power(Q, X), KG[f"ip_{tag}_xt"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(K.logdet(Q), KG[f"ip_{tag}_logdet"], rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("tag", ["a", "b", "c", "d"])
@pytest.mark.parametrize("sweeps", [1, 3])
def test_update_diagonalizer(tag, sweeps):
    from paper_1903_03237_b200 import kernels as K
    X, y = KG[f"ip_{tag}_X"], KG[f"ip_{tag}_y"]
    got = K.update_diagonalizer(KG[f"ip_{tag}_Q0"], X, y, sweeps)
    assert rel(got, KG[f"ip_{tag}_Qnew{sweeps}"]) < 1e-10
    # IP invariant q^H V q = 1 (reference test_spatial.py:207-217)
    V = O.ip_weights(X, y)
    for m in range(X.shape[-1]):
        q = np.conj(got[:, m, :])
        r = np.einsum("fi,fij,fj->f", q.conj(), V[:, m], q).real
        assert np.abs(r - 1.0).max() < 1e-10


def test_update_diagonalizer_scalar_oracle(rng):
    # reference test_spatial.py:219-230 (M = 1 closed form)
    from paper_1903_03237_b200 import kernels as K
    F, T = 3, 50
    X = rng.standard_normal((F, T, 1)) + 1j * rng.standard_normal((F, T, 1))
    y = rng.uniform(0.5, 2.0, (F, T, 1))
    q_old = rng.standard_normal(F) + 1j * rng.standard_normal(F)
    V = ((np.abs(X[..., 0]) ** 2) / y[..., 0]).mean(axis=1)
    q_unnorm = 1.0 / (q_old * V)
    oracle = np.conj(q_unnorm / np.sqrt(np.abs(q_unnorm) ** 2 * V))
    got = K.update_diagonalizer(q_old[:, None, None], X, y)
    np.testing.assert_allclose(got[:, 0, 0], oracle, rtol=1e-12)


def test_update_diagonalizer_singular():
    from paper_1903_03237_b200 import SingularMatrixError
    from paper_1903_03237_b200 import kernels as K
    F, T, M = 2, 2, 4  # T < M -> rank-deficient V
    rng = np.random.default_rng(3)
    X = rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))
    y = np.ones((F, T, M))
    Q = np.tile(np.eye(M, dtype=complex), (F, 1, 1))
    with pytest.raises(SingularMatrixError):
        K.update_diagonalizer(Q, X, y)
    with pytest.raises(O.OracleError):
        O.update_diagonalizer(Q, X, y)


def test_wiener_fast():
    from paper_1903_03237_b200 import kernels as K
    X, Q, g, lam = KG["wf_X"], KG["wf_Q"], KG["wf_g"], KG["wf_lam"]
    got = K.wiener_fast(lam, Q, g, X)
    assert rel(got, KG["wf_images"]) < 1e-12
    assert np.abs(got.sum(axis=0) - X).max() < 1e-9  # partition (test_separate.py:93-98)


def test_wiener_fast_scalar_channel(rng):
    # reference test_separate.py:71-80
    from paper_1903_03237_b200 import kernels as K
    F, T = 3, 6
    X = rng.standard_normal((F, T, 1)) + 1j * rng.standard_normal((F, T, 1))
    Q = np.ones((F, 1, 1), dtype=complex)
    g = rng.uniform(0.5, 2.0, (2, F, 1))
    lam = rng.uniform(0.5, 2.0, (2, F, T))
    images = K.wiener_fast(lam, Q, g, X)
    y = np.einsum("nft,nfm->ftm", lam, g)
    np.testing.assert_allclose(images[0], (lam[0, :, :, None] * g[0, :, None, :] / y) * X,
                               rtol=1e-10)


def test_wiener_singular_q():
    from paper_1903_03237_b200 import SingularMatrixError
    from paper_1903_03237_b200 import kernels as K
    Q = np.zeros((2, 3, 3), dtype=complex)
    Q[0] = np.eye(3)
    with pytest.raises(SingularMatrixError, match="singular diagonalizer"):
        K.wiener_fast(np.ones((2, 2, 4)), Q, np.ones((2, 2, 3)), np.ones((2, 4, 3), complex))


@pytest.mark.parametrize("M", list(range(1, 17)))
def test_all_channel_counts_c64(M):
    """Every compiled M (1..16) in complex64 against the oracle."""
    import torch
    from paper_1903_03237_b200 import kernels as K
    rng = np.random.default_rng(M)
    F, T, N = 3, 48, 3
    X = (rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))).astype(np.complex64)
    y = rng.uniform(0.3, 2.0, (F, T, M))
    Q = np.tile(np.eye(M, dtype=complex), (F, 1, 1)) + 0.1 * (
        rng.standard_normal((F, M, M)) + 1j * rng.standard_normal((F, M, M)))
    Xt = _t(X, torch.complex64)
    Vg = K.ip_weights(Xt, _t(y, torch.float32)).cpu().numpy()
    assert rel(Vg, O.ip_weights(X, y)) < 1e-5
    xg = K.project_power(_t(Q, torch.complex64), Xt).cpu().numpy()
    assert rel(xg, O.project_power(Q.astype(np.complex64), X)) < 1e-5
    if T >= M:
        Qn = K.update_diagonalizer(_t(Q, torch.complex64), Xt, _t(y, torch.float32)).cpu().numpy()
        assert rel(Qn, O.update_diagonalizer(Q.astype(np.complex64), X, y.astype(np.float32))) < 1e-4


@pytest.mark.parametrize("M,T", [(1, 20), (3, 40), (8, 64), (16, 200), (6, 4)])
@pytest.mark.parametrize("precision", ["complex128", "complex64"])
def test_spatial_init_vs_numpy(M, T, precision):
    """fm_spatial_init (SCM + Jacobi, descending, clamp_psd) against numpy's
    eigh: eigenvalues, |Q| (eigenvector phases are arbitrary), unitarity and
    Q G1 Q^H diagonal. T < M gives a rank-deficient SCM (clamped eigenvalues)."""
    import ctypes

    import torch

    from paper_1903_03237_b200 import _lib
    F = 5
    rng = np.random.default_rng(M * 100 + T)
    X = (rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))) / np.sqrt(2)
    X *= rng.uniform(0.5, 2.0, (1, 1, M))
    cdt = torch.complex64 if precision == "complex64" else torch.complex128
    Xd = torch.from_numpy(X).to("cuda", cdt).contiguous()
    Xh = Xd.cpu().numpy().astype(np.complex128)
    Q = torch.empty((F, M, M), device="cuda", dtype=cdt)
    w = torch.empty((F, M), device="cuda", dtype=torch.float64)
    dims = _lib.FmDims(1, F, T, M, 1, 1, 0, _lib.FM_F32 if precision == "complex64" else _lib.FM_F64,
                       1, 1, 0)
    _lib.check(_lib.load().fm_spatial_init(ctypes.byref(dims), _lib.ptr(Xd), _lib.ptr(Q), _lib.ptr(w),
                                           _lib.stream_ptr()), "fm_spatial_init")
    torch.cuda.synchronize()
    Qg, wg = Q.cpu().numpy().astype(np.complex128), w.cpu().numpy()
    G1 = np.einsum("fti,ftj->fij", Xh, Xh.conj()) / T
    ww, U = np.linalg.eigh(G1)
    ww = np.maximum(ww, 1e-12 * np.maximum(ww.max(axis=-1, keepdims=True), 0.0))[..., ::-1]
    U = U[..., ::-1]
    scale = np.abs(ww).max()
    assert np.abs(wg - ww).max() <= 1e-12 * scale
    tol = 1e-10 if precision == "complex128" else 1e-5
    eye = np.eye(M)
    assert np.abs(Qg @ np.conj(Qg.swapaxes(-1, -2)) - eye).max() <= tol
    D = Qg @ G1 @ np.conj(Qg.swapaxes(-1, -2))
    off = D - np.einsum("fii->fi", D)[..., None] * eye
    assert np.abs(off).max() <= tol * 10 * scale
    if T >= M:  # distinct eigenvalues: eigenvectors unique up to phase
        assert np.abs(np.abs(Qg) - np.abs(np.conj(U.swapaxes(-1, -2)))).max() <= tol * 100
