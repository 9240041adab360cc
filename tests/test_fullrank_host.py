"""Full-rank MNMF comparator, CPU part: the oracle
restatement (oracle/fullrank_oracle.py) pinned to the reference's own
outputs (tests/golden/fullrank.npz): fullrank_stats, update_scm,
normalize_trace, reconstruct_scm, wiener_fullrank and a run(method="mnmf")."""

import numpy as np

from conftest import golden, rel
from oracle import fullrank_oracle as FO

G = golden("fullrank.npz")


def test_kernels_pinned_to_reference():
    X, Gm, lam = G["k_X"], G["k_G"], G["k_lam"]
    p1, p2, _, _, ll = FO.fullrank_stats(X, Gm, lam, 1e-3)
    _, _, A, B, _ = FO.fullrank_stats(X, Gm, lam, 1e-3, want_ab=True, want_phi=False)
    assert rel(p1, G["k_phi1"]) < 1e-10 and rel(p2, G["k_phi2"]) < 1e-10
    assert abs(ll - float(G["k_ll"])) < 1e-10 * abs(float(G["k_ll"]))
    assert rel(A, G["k_A"]) < 1e-10 and rel(B, G["k_B"]) < 1e-10
    Gn = FO.update_scm(Gm, G["k_A"], G["k_B"])
    assert rel(Gn, G["k_Gnew"]) < 1e-10
    Gt, c = FO.normalize_trace(Gn)
    assert rel(Gt, G["k_Gnorm"]) < 1e-10 and rel(c, G["k_c"]) < 1e-10
    assert rel(FO.wiener_fullrank(lam, Gm, X, 1e-3), G["k_wiener"]) < 1e-10
    assert rel(FO.reconstruct_scm(G["k_Q"], G["k_g"]), G["k_recon"]) < 1e-12


def test_run_mnmf_pinned_to_reference():
    it = int(G["r_shape"][5])
    out = FO.run_mnmf(G["r_X"], G["r_G0"], G["r_W0"], G["r_H0"], it)
    np.testing.assert_allclose(out["likelihood_trace"], G["r_trace"], rtol=1e-10)
    for k in ("G", "W", "H"):
        assert rel(out[k], G[f"r_{k}"]) < 1e-9, k
    assert rel(out["images"], G["r_images"]) < 1e-9
