"""Generate tests/golden/*.npz by running the UNMODIFIED reference ``fastsep``.

Run in the build container only (``/root/reference`` does not exist on the GPU
box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python oracle/make_golden.py

It imports ``fastsep`` from ``/root/reference/pkg/src`` and drives it through
its own public/kernel API:

* ``kernels.npz``  -- seeded small inputs and the outputs of the reference
  kernels ``_kernels.fast_stats`` / ``ip_weights`` / ``mix_power`` /
  ``project_power``, ``spatial.update_diagonalizer``, ``normalize_gains``,
  ``loglik_fast`` and ``separate.wiener_fast``;
* ``run_*.npz``    -- ``fastsep.run(SeparatorConfig(method="fast-mnmf"), X)``
  with the BASELINE init injected by the SURVEY §8(c) recipe (monkeypatched
  ``_build_spatial`` / ``_build_source``), recording the likelihood trace,
  final W/H/g/Q and the separated images (in full for small shapes, as a
  strided sample plus norms for the larger ones).
"""

import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import fastsep  # noqa: E402  (the reference)
from fastsep import _kernels as K  # noqa: E402
from fastsep import separate as S  # noqa: E402
from fastsep import spatial as SP  # noqa: E402
from fastsep import sources as SRC  # noqa: E402

from paper_1903_03237_b200.synth import baseline_init, make_mixture  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


def kernel_cases():
    out = {}
    rng = np.random.default_rng(20240811)  # reference conftest.py:53-55 seed
    # fast_stats cases: test_kernels.py:28-34 shape and two extra shapes
    for tag, (F, T, M, N) in {"a": (7, 30, 5, 2), "b": (4, 33, 8, 4), "c": (3, 40, 1, 3)}.items():
        xt = rng.uniform(0.0, 3.0, (F, T, M))
        g = rng.uniform(0.1, 2.0, (N, F, M))
        lam = rng.uniform(0.1, 2.0, (N, F, T))
        out[f"fs_{tag}_xt"], out[f"fs_{tag}_g"], out[f"fs_{tag}_lam"] = xt, g, lam
        for floor in (0.0, 0.5):
            for wg in (False, True):
                for wp in (False, True):
                    p1, p2, gn, gd, ll = K.fast_stats(xt, g, lam, floor, wg, wp)
                    key = f"fs_{tag}_{floor}_{int(wg)}{int(wp)}"
                    out[key + "_phi1"], out[key + "_phi2"] = p1, p2
                    out[key + "_gnum"], out[key + "_gden"] = gn, gd
                    out[key + "_ll"] = np.float64(ll)
        out[f"fs_{tag}_mix"] = K.mix_power(lam, g, 0.5)
    # ip_weights / project_power: test_kernels.py:52-67 shapes + M=16
    for tag, (F, T, M) in {"a": (5, 40, 4), "b": (3, 17, 3), "c": (2, 64, 16), "d": (3, 20, 1)}.items():
        X = rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))
        y = rng.uniform(0.2, 2.0, (F, T, M))
        Q = rng.standard_normal((F, M, M)) + 1j * rng.standard_normal((F, M, M))
        out[f"ip_{tag}_X"], out[f"ip_{tag}_y"], out[f"ip_{tag}_Q"] = X, y, Q
        out[f"ip_{tag}_V"] = K.ip_weights(X, y)
        out[f"ip_{tag}_xt"] = K.project_power(Q, X)
        for sweeps in (1, 3):
            Q0 = np.tile(np.eye(M, dtype=complex), (F, 1, 1)) + 0.1 * Q
            out[f"ip_{tag}_Q0"] = Q0
            out[f"ip_{tag}_Qnew{sweeps}"] = SP.update_diagonalizer(Q0, X, y, sweeps)
        out[f"ip_{tag}_logdet"] = np.linalg.slogdet(Q)[1]
    # normalize_gains / wiener_fast / loglik_fast
    F, T, M, N = 6, 25, 4, 3
    X = rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))
    Q = rng.standard_normal((F, M, M)) + 1j * rng.standard_normal((F, M, M)) + 2 * np.eye(M)
    g = rng.uniform(0.1, 2.0, (N, F, M))
    lam = rng.uniform(0.1, 2.0, (N, F, T))
    lam[1, 2, 3:7] = 0.0
    lam[:, 4, 10] = 0.0  # every source zero at one bin -> uniform 1/N gains
    out.update(wf_X=X, wf_Q=Q, wf_g=g, wf_lam=lam)
    out["wf_images"] = S.wiener_fast(lam, Q, g, X)
    gn, c = SP.normalize_gains(g)
    out["ng_g"], out["ng_c"] = gn, c
    out["ll_fast"] = np.float64(SP.loglik_fast(X, Q, g, lam, 1e-3))
    return out


def run_injected(X, Q0, g0, W0, H0, n_iter, normalize=True, ip_sweeps=1, snap_every=0):
    """fastsep.run with the BASELINE init injected."""
    orig_sp, orig_src = S._build_spatial, S._build_source
    S._build_spatial = lambda cfg, Xs: SP.DiagSpatial(Q0.copy(), g0.copy())
    S._build_source = lambda cfg, Xs, rng: SRC.NmfSource(W0.copy(), H0.copy())
    state = {}

    def snap(it, loop):
        state.update(W=loop.source.W_NFK.copy(), H=loop.source.H_NKT.copy(),
                     g=loop.spatial.g_NFM.copy(), Q=loop.spatial.Q_FMM.copy(),
                     floor=loop.floor)

    try:
        N, _, K_ = W0.shape
        cfg = fastsep.SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K_,
                                      n_iterations=n_iter, seed=0, normalize=normalize,
                                      ip_sweeps=ip_sweeps)
        t0 = time.perf_counter()
        res = fastsep.run(cfg, X, on_iteration=snap)
        dt = time.perf_counter() - t0
    finally:
        S._build_spatial, S._build_source = orig_sp, orig_src
    return res, state, dt


def save_run(name, X, F, T, M, N, K_, seed, n_iter, full_images, round64=False, **kw):
    Q0, g0, W0, H0 = baseline_init(F, T, M, N, K_, seed)
    if round64:
        X = X.astype(np.complex64).astype(np.complex128)
    res, st, dt = run_injected(X, Q0, g0, W0, H0, n_iter, **kw)
    d = dict(
        shape=np.array([F, T, M, N, K_, seed, n_iter]),
        X_abs_sum=np.float64(np.abs(X).sum()), X_sample=X[::13, ::11, :],
        trace=res.likelihood_trace, W=st["W"], H=st["H"], g=st["g"], Q=st["Q"],
        floor=np.float64(st["floor"]),
        img_norm=np.linalg.norm(res.images_NFTM.reshape(N, -1), axis=1),
    )
    if full_images:
        d["images"] = res.images_NFTM
    else:
        d["img_sample"] = res.images_NFTM[:, ::17, ::19, :]
    if round64:
        for k in ("W", "H", "g"):
            d[k] = d[k].astype(np.float32)
        d["Q"] = d["Q"].astype(np.complex64)
        if "img_sample" in d:
            d["img_sample"] = d["img_sample"].astype(np.complex64)
    np.savez_compressed(os.path.join(OUT, name), **d)
    print(f"{name}: {n_iter} it in {dt:.1f}s, LL {res.likelihood_trace[0]:.6f} -> "
          f"{res.likelihood_trace[-1]:.6f}", flush=True)


def save_dp(name, F, T, M, K, n_iter, adam_steps, seed=5):
    """fastsep.run(method="fast-mnmf-dp") with the config-4 exp-MLP decoder and
    the Adam latent hook in place of the Metropolis chain (separate.py:205-213
    calls sources.update_latents_fast, monkeypatched here)."""
    from oracle.fastmnmf_dp_oracle import AdamLatents, ExpMLPDecoder, dp_init, make_dp_mixture

    dec = ExpMLPDecoder(F, seed=seed)
    X = make_dp_mixture(F, T, M, K, dec, seed=seed).astype(np.complex64).astype(np.complex128)
    Q0, g0, u0, v0, z0, W0, H0 = dp_init(F, T, M, K, dec.latent_dim, seed)
    hook = AdamLatents(adam_steps)
    orig = (S._build_spatial, S._build_source, SRC.update_latents_fast)
    S._build_spatial = lambda cfg, Xs: SP.DiagSpatial(Q0.copy(), g0.copy())
    S._build_source = lambda cfg, Xs, rng: SRC.DeepPriorPlusNmfSource(
        SRC.DeepPriorFactors(u0.copy(), v0.copy(), z0.copy()), SRC.NmfSource(W0.copy(), H0.copy()),
        dec)
    SRC.update_latents_fast = hook
    st = {}

    def snap(it, loop):
        src = loop.source
        st.update(u=src.dp.u_F.copy(), v=src.dp.v_T.copy(), z=src.dp.z_TD.copy(),
                  W=src.noise.W_NFK.copy(), H=src.noise.H_NKT.copy(),
                  g=loop.spatial.g_NFM.copy(), Q=loop.spatial.Q_FMM.copy())

    try:
        cfg = fastsep.SeparatorConfig(method="fast-mnmf-dp", n_sources=2, n_basis=K,
                                      n_iterations=n_iter, seed=0, decoder=dec,
                                      metropolis_enabled=adam_steps > 0)
        res = fastsep.run(cfg, X, on_iteration=snap)
    finally:
        S._build_spatial, S._build_source, SRC.update_latents_fast = orig
    np.savez_compressed(os.path.join(OUT, name), shape=np.array([F, T, M, K, seed, n_iter, adam_steps]),
                        trace=res.likelihood_trace, images=res.images_NFTM, **st)
    print(f"{name}: LL {res.likelihood_trace[0]:.6f} -> {res.likelihood_trace[-1]:.6f}", flush=True)


def save_dp_mh(name, F, T, M, K, n_iter, seed=5):
    """fastsep.run(method="fast-mnmf-dp") on the reference's own default
    latent path: its ToyDecoder(F) and its Metropolis chain
    (update_latents_fast, sources.py:307-339, NOT patched), with the init
    injected by the SURVEY §8(c) recipe (so the chain's draws come from a
    fresh default_rng(cfg.seed))."""
    from oracle.fastmnmf_dp_oracle import dp_init, make_dp_mixture

    dec = SRC.ToyDecoder(F)
    X = make_dp_mixture(F, T, M, K, dec, seed=seed).astype(np.complex64).astype(np.complex128)
    Q0, g0, u0, v0, z0, W0, H0 = dp_init(F, T, M, K, dec.latent_dim, seed)
    orig = (S._build_spatial, S._build_source)
    S._build_spatial = lambda cfg, Xs: SP.DiagSpatial(Q0.copy(), g0.copy())
    S._build_source = lambda cfg, Xs, rng: SRC.DeepPriorPlusNmfSource(
        SRC.DeepPriorFactors(u0.copy(), v0.copy(), z0.copy()), SRC.NmfSource(W0.copy(), H0.copy()),
        dec)
    st = {}

    def snap(it, loop):
        src = loop.source
        st.update(u=src.dp.u_F.copy(), v=src.dp.v_T.copy(), z=src.dp.z_TD.copy(),
                  W=src.noise.W_NFK.copy(), H=src.noise.H_NKT.copy(),
                  g=loop.spatial.g_NFM.copy(), Q=loop.spatial.Q_FMM.copy())

    try:
        cfg = fastsep.SeparatorConfig(method="fast-mnmf-dp", n_sources=2, n_basis=K,
                                      n_iterations=n_iter, seed=seed)
        res = fastsep.run(cfg, X, on_iteration=snap)
    finally:
        S._build_spatial, S._build_source = orig
    np.savez_compressed(os.path.join(OUT, name), shape=np.array([F, T, M, K, seed, n_iter]),
                        X=X.astype(np.complex64), trace=res.likelihood_trace,
                        images=res.images_NFTM, **st)
    print(f"{name}: LL {res.likelihood_trace[0]:.6f} -> {res.likelihood_trace[-1]:.6f}", flush=True)


def save_stft(name="stft.npz"):
    """The reference's stft / istft (stft.py:27-91) on seeded multichannel
    signals: several window / hop / channel / length combinations, a 1-D
    input, and the round trip with and without ``length``."""
    import importlib

    ST = importlib.import_module("fastsep.stft")

    rng = np.random.default_rng(77)
    out = {}
    cases = {"a": (4096, 2, 1024, 256), "b": (3001, 3, 512, 128), "c": (2048, 1, 256, 256),
             "d": (1500, 4, 64, 48), "e": (1024, 2, 1024, 512)}
    for tag, (n, M, L, hop) in cases.items():
        x = rng.standard_normal((n, M))
        spec = ST.stft(x, L, hop)
        out[f"{tag}_x"], out[f"{tag}_spec"] = x, spec
        out[f"{tag}_y"] = ST.istft(spec, L, hop, length=n)
        out[f"{tag}_yfull"] = ST.istft(spec, L, hop)
        noisy = spec + 0.1 * (rng.standard_normal(spec.shape) + 1j * rng.standard_normal(spec.shape))
        out[f"{tag}_noisy"], out[f"{tag}_ynoisy"] = noisy, ST.istft(noisy, L, hop)
        out[f"{tag}_shape"] = np.array([n, M, L, hop])
    x1 = rng.standard_normal(2000)
    out["mono_x"], out["mono_spec"] = x1, ST.stft(x1, 512, 128)
    np.savez_compressed(os.path.join(OUT, name), **out)
    print(f"{name} written", flush=True)


def save_fullrank(name="fullrank.npz"):
    """The reference's full-rank kernels and a run(method="mnmf") with the
    init injected (monkeypatched _build_spatial / _build_source)."""
    rng = np.random.default_rng(31)
    out = {}
    F, T, M, N = 5, 24, 3, 2
    X = rng.standard_normal((F, T, M)) + 1j * rng.standard_normal((F, T, M))
    Aq = rng.standard_normal((N, F, M, M)) + 1j * rng.standard_normal((N, F, M, M))
    G = Aq @ np.conj(Aq.swapaxes(-1, -2)) + 0.1 * np.eye(M)
    lam = rng.uniform(0.2, 2.0, (N, F, T))
    out.update(k_X=X, k_G=G, k_lam=lam)
    p1, p2, _, _, ll = K.fullrank_stats(X, G, lam, 1e-3, want_ab=False, want_phi=True)
    _, _, A, B, _ = K.fullrank_stats(X, G, lam, 1e-3, want_ab=True, want_phi=False)
    out.update(k_phi1=p1, k_phi2=p2, k_ll=np.array(ll), k_A=A, k_B=B)
    out["k_Gnew"] = SP.update_scm(G, A, B)
    out["k_Gnorm"], out["k_c"] = SP.normalize_trace(out["k_Gnew"])
    out["k_wiener"] = S.wiener_fullrank(lam, G, X, 1e-3)
    Q = np.eye(M) + 0.2 * (rng.standard_normal((F, M, M)) + 1j * rng.standard_normal((F, M, M)))
    g = rng.uniform(0.1, 1.0, (N, F, M))
    out.update(k_Q=Q, k_g=g, k_recon=SP.reconstruct_scm(Q, g))
    # run(method="mnmf") with an injected init (config-0 style mixture)
    Fr, Tr, Mr, Nr, Kr, it = 12, 48, 3, 2, 4, 6
    Xr = make_mixture(Fr, Tr, Mr, Nr, Kr, seed=8)
    Q0, g0, W0, H0 = baseline_init(Fr, Tr, Mr, Nr, Kr, 8)
    G0 = SP.reconstruct_scm(Q0, g0)
    orig = (S._build_spatial, S._build_source)
    S._build_spatial = lambda cfg, Xs: SP.FullRankSpatial(G0.copy())
    S._build_source = lambda cfg, Xs, rng: SRC.NmfSource(W0.copy(), H0.copy())
    st = {}

    def snap(i, loop):
        st.update(G=loop.spatial.G_NFMM.copy(), W=loop.source.W_NFK.copy(),
                  H=loop.source.H_NKT.copy())

    try:
        cfg = fastsep.SeparatorConfig(method="mnmf", n_sources=Nr, n_basis=Kr, n_iterations=it,
                                      seed=8)
        res = fastsep.run(cfg, Xr, on_iteration=snap)
    finally:
        S._build_spatial, S._build_source = orig
    out.update(r_X=Xr, r_G0=G0, r_W0=W0, r_H0=H0, r_trace=res.likelihood_trace,
               r_images=res.images_NFTM, r_G=st["G"], r_W=st["W"], r_H=st["H"],
               r_shape=np.array([Fr, Tr, Mr, Nr, Kr, it]))
    np.savez_compressed(os.path.join(OUT, name), **out)
    print(f"{name} written: LL {res.likelihood_trace[0]:.6f} -> {res.likelihood_trace[-1]:.6f}",
          flush=True)


def _compact(res, st, N, step_f, step_t):
    """Golden record of a full-shape run: state, trace, a strided image
    sample, per-source image norms and per-(n, m) image energies."""
    img = res.images_NFTM
    return dict(
        trace=res.likelihood_trace, W=st["W"].astype(np.float32), H=st["H"].astype(np.float32),
        g=st["g"].astype(np.float32), Q=st["Q"].astype(np.complex64),
        floor=np.float64(st["floor"]),
        img_norm=np.linalg.norm(img.reshape(N, -1), axis=1),
        img_energy=np.einsum("nftm,nftm->nm", img, np.conj(img)).real,
        img_sample=img[:, ::step_f, ::step_t, :].astype(np.complex64))


def save_full_c2(n_mix=8):
    """BASELINE config 2 at full shape: mixtures b = 0..n_mix-1 of the batch,
    each (513, 512, 4, 3, 8) with seed base + b (base 0), complex64-rounded,
    100 iterations, each through an unmodified reference run()."""
    from paper_1903_03237_b200.synth import make_mixture_fast
    F, T, M, N, K_, it = 513, 512, 4, 3, 8, 100
    out = dict(shape=np.array([F, T, M, N, K_, 0, it, n_mix]))
    for b in range(n_mix):
        X = make_mixture_fast(F, T, M, N, K_, seed=b).astype(np.complex128)
        res, st, dt = run_injected(X, *baseline_init(F, T, M, N, K_, b), it)
        for k, v in _compact(res, st, N, 17, 19).items():
            out[f"b{b}_{k}"] = v
        out[f"b{b}_X_abs_sum"] = np.float64(np.abs(X).sum())
        print(f"c2 mixture {b}: {dt:.1f}s LL {res.likelihood_trace[-1]:.6f}", flush=True)
    np.savez_compressed(os.path.join(OUT, "run_c2_full.npz"), **out)


def save_full_c3(n_iter=4):
    """BASELINE config 3 at full shape (F=1025, T=8192, M=16, N=6, K=32),
    complex64-rounded mixture, seed 0, n_iter iterations of an unmodified
    reference run() (~70 s per iteration on the build host)."""
    from paper_1903_03237_b200.synth import make_mixture_fast
    F, T, M, N, K_ = 1025, 8192, 16, 6, 32
    t0 = time.perf_counter()
    X = make_mixture_fast(F, T, M, N, K_, seed=0).astype(np.complex128)
    print(f"c3 mixture generated in {time.perf_counter() - t0:.1f}s", flush=True)
    res, st, dt = run_injected(X, *baseline_init(F, T, M, N, K_, 0), n_iter)
    d = _compact(res, st, N, 64, 97)
    d.update(shape=np.array([F, T, M, N, K_, 0, n_iter]), X_abs_sum=np.float64(np.abs(X).sum()),
             X_sample=X[::64, ::97, :].astype(np.complex64))
    np.savez_compressed(os.path.join(OUT, "run_c3_full.npz"), **d)
    print(f"c3: {n_iter} it in {dt:.1f}s LL {res.likelihood_trace[0]:.6f} -> "
          f"{res.likelihood_trace[-1]:.6f}", flush=True)


def save_full_c4(n_iter=100, adam_steps=10, seed=0):
    """BASELINE config 4 at full shape (F=513, T=512, M=8, N=2, noise K=32,
    exp-MLP decoder D=16 -> 128 -> 128 -> F, 10 Adam steps per iteration,
    100 iterations): the unmodified reference loop with the Adam hook at
    update_latents_fast (as save_dp), images as a sample plus norms."""
    from oracle.fastmnmf_dp_oracle import AdamLatents, ExpMLPDecoder, dp_init, make_dp_mixture
    F, T, M, K_ = 513, 512, 8, 32
    dec = ExpMLPDecoder(F, seed=seed)
    X = make_dp_mixture(F, T, M, K_, dec, seed=seed).astype(np.complex64).astype(np.complex128)
    Q0, g0, u0, v0, z0, W0, H0 = dp_init(F, T, M, K_, dec.latent_dim, seed)
    hook = AdamLatents(adam_steps)
    orig = (S._build_spatial, S._build_source, SRC.update_latents_fast)
    S._build_spatial = lambda cfg, Xs: SP.DiagSpatial(Q0.copy(), g0.copy())
    S._build_source = lambda cfg, Xs, rng: SRC.DeepPriorPlusNmfSource(
        SRC.DeepPriorFactors(u0.copy(), v0.copy(), z0.copy()), SRC.NmfSource(W0.copy(), H0.copy()),
        dec)
    SRC.update_latents_fast = hook
    st = {}

    def snap(it, loop):
        src = loop.source
        st.update(u=src.dp.u_F.copy(), v=src.dp.v_T.copy(), z=src.dp.z_TD.copy(),
                  W=src.noise.W_NFK.copy(), H=src.noise.H_NKT.copy(),
                  g=loop.spatial.g_NFM.copy(), Q=loop.spatial.Q_FMM.copy())

    t0 = time.perf_counter()
    try:
        cfg = fastsep.SeparatorConfig(method="fast-mnmf-dp", n_sources=2, n_basis=K_,
                                      n_iterations=n_iter, seed=0, decoder=dec,
                                      metropolis_enabled=True)
        res = fastsep.run(cfg, X, on_iteration=snap)
    finally:
        S._build_spatial, S._build_source, SRC.update_latents_fast = orig
    img = res.images_NFTM
    np.savez_compressed(
        os.path.join(OUT, "run_c4_full.npz"), shape=np.array([F, T, M, K_, seed, n_iter, adam_steps]),
        trace=res.likelihood_trace, img_norm=np.linalg.norm(img.reshape(2, -1), axis=1),
        img_sample=img[:, ::17, ::19, :].astype(np.complex64), X_abs_sum=np.float64(np.abs(X).sum()),
        **{k: (v.astype(np.complex64) if np.iscomplexobj(v) else v.astype(np.float32))
           for k, v in st.items()})
    print(f"c4: {n_iter} it in {time.perf_counter() - t0:.1f}s LL {res.likelihood_trace[0]:.6f} -> "
          f"{res.likelihood_trace[-1]:.6f}", flush=True)


def main():
    os.makedirs(OUT, exist_ok=True)
    if "--full-c2" in sys.argv:
        save_full_c2()
        return
    if "--full-c3" in sys.argv:
        save_full_c3()
        return
    if "--full-c4" in sys.argv:
        save_full_c4()
        return
    if "--fullrank-only" in sys.argv:
        save_fullrank()
        return
    if "--stft-only" in sys.argv:
        save_stft()
        return
    if "--dp-mh-only" in sys.argv:
        save_dp_mh("run_dp_mh.npz", 33, 64, 4, 8, 6)
        return
    if "--dp-only" in sys.argv:
        save_dp("run_dp_mu.npz", 33, 64, 4, 8, 8, 0)
        save_dp("run_dp_adam.npz", 33, 64, 4, 8, 8, 10)
        save_dp_mh("run_dp_mh.npz", 33, 64, 4, 8, 6)
        return
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **kernel_cases())
    print("kernels.npz written", flush=True)
    # small end-to-end shapes (full images)
    for name, (F, T, M, N, K_, it, kw) in {
        "run_small_a.npz": (16, 40, 3, 2, 4, 10, {}),
        "run_small_b.npz": (9, 48, 5, 3, 3, 8, {"normalize": False}),
        "run_small_c.npz": (12, 36, 4, 2, 5, 6, {"ip_sweeps": 2}),
        "run_small_d.npz": (5, 64, 8, 4, 6, 5, {}),
    }.items():
        X = make_mixture(F, T, M, N, K_, seed=3)
        save_run(name, X, F, T, M, N, K_, 3, it, True, **kw)
    # config 0: complex128, 50 iterations, seed 0
    X0 = make_mixture(257, 128, 4, 2, 8, seed=0)
    save_run("run_c0.npz", X0, 257, 128, 4, 2, 8, 0, 50, False)
    # config 0 shape in complex64 mode (oracle fed the c64-rounded X)
    save_run("run_c0_c64.npz", X0, 257, 128, 4, 2, 8, 0, 50, False, round64=True)
    # config 1 shape, complex64-rounded X, 100 iterations
    save_dp("run_dp_mu.npz", 33, 64, 4, 8, 8, 0)
    save_dp("run_dp_adam.npz", 33, 64, 4, 8, 8, 10)
    save_dp_mh("run_dp_mh.npz", 33, 64, 4, 8, 6)
    save_stft()
    save_fullrank()
    if "--with-c1" in sys.argv:
        X1 = make_mixture(513, 1024, 8, 4, 16, seed=0)
        save_run("run_c1_c64.npz", X1, 513, 1024, 8, 4, 16, 0, 100, False, round64=True)


if __name__ == "__main__":
    main()
