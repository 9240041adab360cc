"""Full-rank MNMF comparator on the device against the
reference's outputs (tests/golden/fullrank.npz): the kernels at 1e-10
(complex128) and a run(method="mnmf") at the north_star tolerances
(complex128 <= 1e-6, complex64 <= 1e-3)."""

import numpy as np
import pytest

from conftest import golden, rel
from oracle import fullrank_oracle as FO

pytestmark = pytest.mark.gpu
G = golden("fullrank.npz")


def test_fullrank_kernels_vs_reference():
    from paper_1903_03237_b200 import fullrank as FR
    X, Gm, lam = G["k_X"], G["k_G"], G["k_lam"]
    p1, p2, _, _, ll = FR.fullrank_stats(X, Gm, lam, 1e-3)
    _, _, A, B, _ = FR.fullrank_stats(X, Gm, lam, 1e-3, want_ab=True, want_phi=False)
    assert rel(p1, G["k_phi1"]) < 1e-10 and rel(p2, G["k_phi2"]) < 1e-10
    assert abs(ll - float(G["k_ll"])) < 1e-10 * abs(float(G["k_ll"]))
    assert rel(A, G["k_A"]) < 1e-10 and rel(B, G["k_B"]) < 1e-10
    assert rel(FR.update_scm(Gm, G["k_A"], G["k_B"]), G["k_Gnew"]) < 1e-10
    assert rel(FR.wiener_fullrank(lam, Gm, X, 1e-3), G["k_wiener"]) < 1e-10
    assert rel(FR.reconstruct_scm(G["k_Q"], G["k_g"]), G["k_recon"]) < 1e-12


@pytest.mark.parametrize("precision,tol", [("complex128", 1e-6), ("complex64", 1e-3)])
def test_run_mnmf_vs_reference(precision, tol):
    from paper_1903_03237_b200 import SeparatorConfig, run
    F, T, M, N, K, it = (int(v) for v in G["r_shape"])
    X = G["r_X"]
    if precision == "complex64":
        X = X.astype(np.complex64)
        ref = FO.run_mnmf(X.astype(np.complex128), G["r_G0"], G["r_W0"], G["r_H0"], it)
        ref = dict(trace=ref["likelihood_trace"], images=ref["images"], G=ref["G"], W=ref["W"],
                   H=ref["H"])
    else:
        ref = dict(trace=G["r_trace"], images=G["r_images"], G=G["r_G"], W=G["r_W"], H=G["r_H"])
    cfg = SeparatorConfig(method="mnmf", n_sources=N, n_basis=K, n_iterations=it, seed=8,
                          precision=precision)
    st = {}

    def snap(i, loop):
        st.update(G=loop.spatial.G_NFMM, W=loop.source.W_NFK, H=loop.source.H_NKT)

    res = run(cfg, X, init=(G["r_G0"], G["r_W0"], G["r_H0"]), on_iteration=snap)
    assert np.max(np.abs(res.likelihood_trace - ref["trace"]) / np.abs(ref["trace"])) <= tol
    for k in ("G", "W", "H"):
        assert rel(st[k], ref[k]) <= tol, (k, rel(st[k], ref[k]))
    assert rel(res.images_NFTM, ref["images"]) <= tol
    # partition: the images sum to the observation (separate.py:93-95)
    assert rel(res.images_NFTM.sum(axis=0), X) < (1e-12 if precision == "complex128" else 1e-5)


def test_run_mnmf_default_init():
    """The reference's own init (circular_init -> reconstruct_scm, NmfSource.random)."""
    from paper_1903_03237_b200 import SeparatorConfig, run
    from paper_1903_03237_b200.synth import make_mixture
    X = make_mixture(10, 40, 4, 2, 3, seed=2)
    res = run(SeparatorConfig(method="mnmf", n_sources=2, n_basis=3, n_iterations=5,
                              precision="complex128"), X)
    tr = res.likelihood_trace
    assert np.all(np.isfinite(tr)) and np.all(np.diff(tr) > -1e-6 * np.abs(tr[1:]))
    assert rel(res.images_NFTM.sum(axis=0), X) < 1e-12
