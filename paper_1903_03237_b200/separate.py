"""FastMNMF separator API on B200 -- drop-in for ``fastsep.separate``
(``pkg/src/fastsep/separate.py``) on its hot path (``method="fast-mnmf"``).

The parameter layout, config fields, result type, trace semantics and error
behaviour follow the reference; the iteration itself runs as five sm_100a
kernel launches per pass over device-resident state (libfastmnmf.so,
``fm_iterate``), optionally replayed from one captured CUDA graph.
"""

import ctypes
import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib
from . import kernels as K
from .errors import InvalidInputError, NumericalBreakdownError, SingularMatrixError

METHODS = ("fca", "mnmf", "mnmf-dp", "fast-fca", "fast-mnmf", "fast-mnmf-dp")  # separate.py:39
FAST_METHODS = ("fast-fca", "fast-mnmf", "fast-mnmf-dp")
DP_METHODS = ("mnmf-dp", "fast-mnmf-dp")
# the hot path this backend provides, plus the full-rank MNMF comparator (§8(f) 4)
SUPPORTED_METHODS = ("fast-mnmf", "fast-mnmf-dp", "mnmf")
PRECISIONS = ("complex128", "complex64")


@dataclass
class MetropolisConfig:
    """Random-walk proposal settings of the latent chain (sources.py:38-49),
    used by fast-mnmf-dp's Metropolis update (k_dp_mh)."""

    proposal_var: float = 1e-4
    inner_steps: int = 30

    def __post_init__(self):
        if self.proposal_var <= 0:
            raise InvalidInputError("proposal_var must be positive")
        if self.inner_steps < 1:
            raise InvalidInputError("inner_steps must be >= 1")


@dataclass
class SeparatorConfig:
    """separate.py:44-71, plus the B200 execution fields ``precision``,
    ``use_graph`` and ``device``."""

    method: str = "fast-mnmf"
    n_sources: int = 2
    n_basis: int = 16
    n_iterations: int = 100
    seed: int = 0
    spatial_init: str = "auto"  # auto | circular | observed
    normalize: bool = True
    ip_sweeps: int = 1
    metropolis: MetropolisConfig = field(default_factory=MetropolisConfig)
    metropolis_enabled: bool = True
    decoder: object = None
    record_likelihood: bool = True
    precision: str = "complex128"
    use_graph: bool = True
    device: str = "cuda"
    # FastMNMF-DP latent update (BASELINE config 4): Adam steps on z per outer
    # iteration in place of the reference's Metropolis chain; disabled, like
    # the chain, by metropolis_enabled=False
    adam_steps: int = 10
    adam_lr: float = 1e-2
    # FastMNMF-DP latent update: "auto" = the reference's Metropolis chain
    # (sources.py:307-339) for its ToyDecoder, Adam for an ExpMLPDecoder
    latent_update: str = "auto"  # auto | metropolis | adam
    # Metropolis draws: "numpy" = the run's Generator in the reference's order
    # (bit-for-bit the reference's chain), "device" = Philox on the GPU
    metropolis_rng: str = "numpy"

    def validate(self):  # separate.py:59-71
        if self.method not in METHODS:
            raise InvalidInputError(f"unknown method {self.method!r}")
        if self.n_sources < 1:
            raise InvalidInputError("n_sources must be >= 1")
        if self.method in DP_METHODS and self.n_sources < 2:
            raise InvalidInputError("deep-prior methods need n_sources >= 2")
        if self.n_iterations < 1:
            raise InvalidInputError("n_iterations must be >= 1")
        if self.n_basis < 1:
            raise InvalidInputError("n_basis must be >= 1")
        if self.spatial_init not in ("auto", "circular", "observed"):
            raise InvalidInputError(f"unknown spatial_init {self.spatial_init!r}")
        if self.precision not in PRECISIONS:
            raise InvalidInputError(f"unknown precision {self.precision!r}")
        if self.ip_sweeps < 1:
            raise InvalidInputError("ip_sweeps must be >= 1")
        if self.latent_update not in ("auto", "metropolis", "adam"):
            raise InvalidInputError(f"unknown latent_update {self.latent_update!r}")
        if self.metropolis_rng not in ("numpy", "device"):
            raise InvalidInputError(f"unknown metropolis_rng {self.metropolis_rng!r}")


@dataclass
class SeparationResult:  # separate.py:74-80
    images_NFTM: np.ndarray
    likelihood_trace: np.ndarray
    time_trace: np.ndarray
    method: str
    config: SeparatorConfig


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1903_03237_b200 needs a CUDA device (no CPU fallback)")
    return torch


def wiener_fast(lam_NFT, Q_FMM, g_NFM, X_FTM):
    """Diagonalized-domain Wiener filter (separate.py:110-125) on the device."""
    return K.wiener_fast(lam_NFT, Q_FMM, g_NFM, X_FTM)


# ---------------------------------------------------------------------------
# device-resident loop state
# ---------------------------------------------------------------------------

class _SpatialView:
    """``loop.spatial`` surface (DiagSpatial, spatial.py:47-56): host copies
    on read; assignment uploads (the reference's iterate assigns them)."""

    def __init__(self, loop, b):
        self._loop, self._b = loop, b

    @property
    def Q_FMM(self):
        return self._loop.Q[self._b].cpu().numpy().astype(np.complex128)

    @Q_FMM.setter
    def Q_FMM(self, v):
        self._loop.Q[self._b].copy_(self._loop._as_dev(v, self._loop.Q.dtype))
        self._loop._prologue_done = False  # x~, Ht and the W step derive from the state

    @property
    def g_NFM(self):
        return self._loop.g[self._b].cpu().numpy().astype(np.float64)

    @g_NFM.setter
    def g_NFM(self, v):
        self._loop.g[self._b].copy_(self._loop._as_dev(v, self._loop.real))
        self._loop._prologue_done = False  # x~, Ht and the W step derive from the state

    @property
    def n_sources(self):
        return self._loop.N


class _SourceView:
    """``loop.source`` surface (NmfSource, sources.py:167-204): host copies
    on read; assignment uploads."""

    mu_steps = ("W", "H")

    def __init__(self, loop, b):
        self._loop, self._b = loop, b

    @property
    def W_NFK(self):
        return self._loop.W[self._b].cpu().numpy().astype(np.float64)

    @W_NFK.setter
    def W_NFK(self, v):
        self._loop.W[self._b].copy_(self._loop._as_dev(v, self._loop.real))
        self._loop._prologue_done = False  # x~, Ht and the W step derive from the state

    @property
    def H_NKT(self):
        return self._loop.H[self._b].cpu().numpy().astype(np.float64)

    @H_NKT.setter
    def H_NKT(self, v):
        self._loop.H[self._b].copy_(self._loop._as_dev(v, self._loop.real))
        self._loop._prologue_done = False  # x~, Ht and the W step derive from the state

    @property
    def n_sources(self):
        return self._loop.N

    @property
    def n_basis(self):
        return self._loop.K

    def lam(self):
        return self._loop.lam_device()[self._b].cpu().numpy().astype(np.float64)


def _on_device(fn):
    """Run a DeviceLoop method with the loop's device current, so the kernels
    launch on that device's current stream (SeparatorConfig.device)."""
    import functools

    @functools.wraps(fn)
    def wrapped(self, *a, **kw):
        with self.torch.cuda.device(self.device):
            return fn(self, *a, **kw)

    return wrapped


class DeviceLoop:
    """The _DiagLoop (separate.py:175-243) over a batch of B mixtures held in
    HBM.

    Device state: ``X_dev`` the SCALED observation (B,F,T,M), ``xt_dev`` the
    projected power, ``Q``, ``g``, ``W``, ``H`` and ``floor_dev`` (B,).

    The reference loop's own surface reads mixture 0 back to the host:
    ``X`` (F,T,M) complex128, ``xt`` (F,T,M), ``floor`` (float),
    ``spatial.Q_FMM/g_NFM``, ``source.W_NFK/H_NKT/lam()``, and
    ``iterate(cfg, rng)``, ``loglik()``, ``logdet_term()``, ``images()``.

    Frequency sharding: ``f_offset`` is the global index of local bin 0 and
    ``hstat_allreduce`` (a callable on the packed (B,2,N,K,T) H statistics)
    is invoked between the two phases of every iteration.
    """

    def __init__(self, X, Q, g, W, H, floor, normalize=True, ip_sweeps=1, n_trace=1,
                 f_offset=0, hstat_allreduce=None, dp=None):
        torch = _torch()
        self.torch = torch
        self.device = X.device
        with torch.cuda.device(self.device):
            self._init(X, Q, g, W, H, floor, normalize, ip_sweeps, n_trace, f_offset,
                       hstat_allreduce, dp)

    def _init(self, X, Q, g, W, H, floor, normalize, ip_sweeps, n_trace, f_offset,
              hstat_allreduce, dp):
        torch = self.torch
        self.X_dev = X
        self.real = torch.float32 if X.dtype == torch.complex64 else torch.float64
        self.B, self.F, self.T, self.M = X.shape
        # FastMNMF-DP: (decoder, u, v, z, adam_steps, lr[, mh_steps, mh_var, mh_rng, mh_seed])
        self.dp_args = dp
        self.N, self.K = W.shape[1] + (1 if dp is not None else 0), W.shape[3]
        dev = X.device
        self.Q = Q.to(dev, X.dtype).resolve_conj().contiguous()
        self.g = g.to(dev, self.real).contiguous()
        self.W = W.to(dev, self.real).contiguous()
        self.H = H.to(dev, self.real).contiguous()
        self.floor_dev = floor.to(dev, self.real).contiguous()
        self.xt_dev = torch.empty((self.B, self.F, self.T, self.M), device=dev, dtype=self.real)
        self.n_trace = max(1, int(n_trace))
        self.trace = torch.zeros((self.n_trace, self.B), device=dev, dtype=torch.float64)
        self.status = torch.full((1,), -1, dtype=torch.int64, device=dev)
        self.dims = _lib.FmDims(self.B, self.F, self.T, self.M, self.N, self.K, int(f_offset),
                                _lib.FM_F32 if self.real == torch.float32 else _lib.FM_F64,
                                int(bool(normalize)), int(ip_sweeps), int(dp is not None))
        lib = _lib.load()
        nbytes = lib.fm_workspace_bytes(ctypes.byref(self.dims))
        if nbytes == 0:
            raise InvalidInputError(f"unsupported problem: {lib.fm_last_error().decode()}")
        self.work = torch.empty((nbytes,), dtype=torch.uint8, device=dev)
        self.state = _lib.FmState(*[_lib.ptr(t).value for t in (
            self.X_dev, self.xt_dev, self.Q, self.g, self.W, self.H, self.floor_dev, self.trace,
            self.status, self.work)])
        self.hstat_allreduce = hstat_allreduce
        self.hstat = (torch.empty((self.B, 2, self.N, self.K, self.T), device=dev, dtype=self.real)
                      if hstat_allreduce is not None else None)
        self.iterations_done = 0
        self._prologue_done = False
        self._shard_graph = None
        self.dp = None
        if dp is not None:
            from .dp import DeviceDP

            decoder, u, v, z, steps, lr, *mh = dp
            mh_steps, mh_var, mh_rng, mh_seed = (list(mh) + [0, 1e-4, None, 0][len(mh):])[:4]
            self.dp = DeviceDP(decoder, u, v, z, self.dims, self.real, dev, adam_steps=steps, lr=lr,
                               mh_steps=mh_steps, mh_var=mh_var, mh_rng=mh_rng, mh_seed=mh_seed)
        self.spatial = _SpatialView(self, 0)
        self.source = _SourceView(self, 0)

    def _as_dev(self, v, dtype):
        t = self.torch
        v = v if isinstance(v, t.Tensor) else t.from_numpy(np.ascontiguousarray(v))
        return v.to(self.device, dtype)

    # ---- the reference _DiagLoop surface (separate.py:175-243), mixture 0 ----
    @property
    def X(self):
        """Scaled observation (F,T,M) complex128 on the host (separate.py:179)."""
        return self.X_dev[0].cpu().numpy().astype(np.complex128)

    @property
    def xt(self):
        """Projected power x~ (F,T,M) on the host (separate.py:183)."""
        return self.xt_dev[0].cpu().numpy().astype(np.float64)

    @property
    def floor(self):
        """Model-power floor (separate.py:182, spatial.py:64-66)."""
        return float(self.floor_dev[0])

    @_on_device
    def data_term(self):
        """sum(-x~/y - log y) of the current state, per mixture (B,): the
        first statistics pass of the next iteration (_kernels.py:233)."""
        out = (ctypes.c_double * self.B)()
        _lib.check(_lib.load().fm_data_term(ctypes.byref(self.dims), ctypes.byref(self.state), out,
                                            _lib.stream_ptr()), "fm_data_term")
        return np.array(out[:])

    @_on_device
    def logdet_terms(self):
        """2T sum_f log|det Q_f| per mixture (B,) (separate.py:236-238)."""
        ld = K.logdet(self.Q.reshape(self.B * self.F, self.M, self.M))
        return 2.0 * self.T * ld.reshape(self.B, self.F).double().sum(dim=1).cpu().numpy()

    def logdet_term(self):
        """separate.py:236-238 (mixture 0)."""
        return float(self.logdet_terms()[0])

    def loglik(self):
        """loglik_fast of the current state (separate.py:195-199, spatial.py:233-241)."""
        return float(self.data_term()[0]) + self.logdet_term()

    def iterate(self, cfg=None, rng=None):
        """One pass (separate.py:201-234): returns the data term of the first
        statistics refresh, i.e. of the state before the pass. Raises the
        reference's SingularMatrixError (without run()'s iteration prefix)."""
        if self.iterations_done >= self.n_trace:
            self._grow_trace(self.iterations_done + 1)
        if not self._prologue_done:
            self.prologue() if self.iterations_done == 0 else self.refresh()
        if rng is not None and self.dp is not None and self.dp.noise is not None:
            self.dp.mh_rng = rng
        ll = float(self.data_term()[0])
        self.run(1, use_graph=bool(getattr(cfg, "use_graph", True)))
        err = self.status_error(prefix=False)
        if err is not None:
            raise err
        return ll

    def _grow_trace(self, n):
        torch = self.torch
        t = torch.zeros((max(n, 2 * self.n_trace), self.B), device=self.device, dtype=torch.float64)
        t[: self.n_trace] = self.trace
        self.trace, self.n_trace = t, t.shape[0]
        self.state.trace = _lib.ptr(self.trace).value

    def images(self):
        """separate.py:240-243: Wiener images (N,F,T,M) of mixture 0 in the
        scaled domain, as numpy (run() multiplies by the scale)."""
        img = self.images_batch([1.0] * self.B)[0]
        return img.cpu().numpy()

    # ---- batched device helpers ----
    @property
    def schedule(self):
        """The iteration schedule the library runs for these dims: "split",
        "fused" or "bin" (fastmnmf.h fm_schedule)."""
        return _lib.SCHEDULES[_lib.load().fm_schedule(ctypes.byref(self.dims))]

    @property
    def xt_FTM(self):
        return self.xt_dev[0]

    @_on_device
    def lam_device(self):
        """lambda = W H of the current state (sources.py:184-187), (B,N,F,T)."""
        torch = self.torch
        lam = torch.empty((self.B, self.N, self.F, self.T), device=self.device, dtype=self.real)
        lib = _lib.load()
        _lib.check(lib.fm_nmf_lambda(ctypes.byref(self.dims), _lib.ptr(self.W), _lib.ptr(self.H),
                                     _lib.ptr(lam), _lib.stream_ptr()), "fm_nmf_lambda")
        if self.dp is not None:  # source 0: u v r (sources.py:248-249)
            lam[:, 0] = self.dp.lam0()
        return lam

    @_on_device
    def prologue(self):
        self._prologue_done = True
        lib = _lib.load()
        if self.dp is not None:
            _lib.check(lib.fm_prologue_dp(ctypes.byref(self.dims), ctypes.byref(self.state),
                                          ctypes.byref(self.dp.struct), _lib.stream_ptr()),
                       "fm_prologue_dp")
            return
        _lib.check(lib.fm_prologue(ctypes.byref(self.dims), ctypes.byref(self.state),
                                   _lib.stream_ptr()), "fm_prologue")

    @_on_device
    def refresh(self):
        """Re-derive x~, the transposed H and the coming W step after the
        state was assigned between iterations (fm_refresh); the trace index
        continues."""
        if self.dp is not None:
            raise InvalidInputError("state assignment between deep-prior iterations is not supported")
        self._prologue_done = True
        _lib.check(_lib.load().fm_refresh(ctypes.byref(self.dims), ctypes.byref(self.state),
                                          _lib.stream_ptr()), "fm_refresh")

    @_on_device
    def run(self, n, use_graph=False):
        lib = _lib.load()
        if not self._prologue_done:
            self.prologue() if self.iterations_done == 0 else self.refresh()
        if self.iterations_done + n > self.n_trace:
            raise InvalidInputError("trace buffer too small for the requested iterations")
        if self.dp is not None and self.dp.noise is not None:
            for _ in range(n):  # the reference's numpy draws, one iteration at a time
                self.dp.fill_draws()
                _lib.check(lib.fm_run_dp(ctypes.byref(self.dims), ctypes.byref(self.state),
                                         ctypes.byref(self.dp.struct), 1, int(bool(use_graph)),
                                         _lib.stream_ptr()), "fm_run_dp")
        elif self.dp is not None:
            _lib.check(lib.fm_run_dp(ctypes.byref(self.dims), ctypes.byref(self.state),
                                     ctypes.byref(self.dp.struct), int(n), int(bool(use_graph)),
                                     _lib.stream_ptr()), "fm_run_dp")
        elif self.hstat_allreduce is None:
            _lib.check(lib.fm_run(ctypes.byref(self.dims), ctypes.byref(self.state), int(n),
                                  int(bool(use_graph)), _lib.stream_ptr()), "fm_run")
        elif use_graph and getattr(self.hstat_allreduce, "capturable", False):
            # frequency shard: phase 0, the all-reduce (NCCL, graph-capturable)
            # and phase 1 captured once into one CUDA graph, replayed per iteration
            if self._shard_graph is None:
                torch = self.torch
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._shard_iteration(lib)
                self._shard_graph = g
            for _ in range(n):
                self._shard_graph.replay()
        else:
            for _ in range(n):
                self._shard_iteration(lib)
        self.iterations_done += n

    def _shard_iteration(self, lib):
        """One frequency-sharded iteration: phase 0 (this shard's H
        statistics), the cross-shard sum, phase 1 (H update + the per-bin rest)."""
        _lib.check(lib.fm_iterate_phase(ctypes.byref(self.dims), ctypes.byref(self.state), 0,
                                        _lib.ptr(self.hstat), _lib.stream_ptr()), "fm_iterate_phase(0)")
        self.hstat_allreduce(self.hstat)
        _lib.check(lib.fm_iterate_phase(ctypes.byref(self.dims), ctypes.byref(self.state), 1,
                                        _lib.ptr(self.hstat), _lib.stream_ptr()), "fm_iterate_phase(1)")

    def status_error(self, prefix=True):
        """The first numerical failure as the reference's exception, or None;
        ``prefix`` adds run()'s "iteration {it}: " (separate.py:310-311)."""
        s = K.decode_status(self.status.item())
        if s is None:
            return None
        code, it, m, f = s
        msg = K.status_message(code, m, f)
        return SingularMatrixError(f"iteration {it}: {msg}" if prefix else msg)

    @_on_device
    def images_batch(self, scale, defer_status=False):
        """separate.py:240-243 + the scale-back of :323, for every mixture:
        one wiener_fast launch per mixture on the stream. With
        ``defer_status`` nothing reads back from the device: returns
        (images, status tensors) and the caller runs
        ``kernels.check_wiener_status`` on each once it has to wait anyway."""
        lam = self.lam_device()
        out, sts = [], []
        for b in range(self.B):
            img = K.wiener_fast(lam[b], self.Q[b], self.g[b], self.X_dev[b], defer_status=defer_status)
            if defer_status:
                img, st = img
                sts.append(st)
            if float(scale[b]) != 1.0:
                img.mul_(float(scale[b]))
            out.append(img)
        return (out, sts) if defer_status else out


# ---------------------------------------------------------------------------
# initialisation (separate.py:246-264)
# ---------------------------------------------------------------------------

def default_init(cfg, Xs, rng, n_nmf=None):
    """Reference default init: circular spatial init (spatial.py:109-121) and
    NmfSource.random (sources.py:177-182) drawn from the run's rng.

    The spatial part -- time-averaged SCM, clamp_psd and the descending
    Hermitian eigendecomposition (spatial.py:93-105, linalg.py:23-33, 85-94)
    -- is one native kernel (fm_spatial_init: fp64 SCM + warp-level cyclic
    complex Jacobi per bin).
    """
    torch = _torch()
    F, T, M = Xs.shape
    N = cfg.n_sources
    init = cfg.spatial_init
    if init == "auto":
        init = "observed" if cfg.method in DP_METHODS else "circular"
    X1 = Xs.contiguous()
    dims = _lib.FmDims(1, F, T, M, 1, 1, 0,
                       _lib.FM_F32 if X1.dtype == torch.complex64 else _lib.FM_F64, 1, 1, 0)
    Q = torch.empty((F, M, M), device=X1.device, dtype=X1.dtype)
    w = torch.empty((F, M), device=X1.device, dtype=torch.float64)
    _lib.check(_lib.load().fm_spatial_init(ctypes.byref(dims), _lib.ptr(X1), _lib.ptr(Q), _lib.ptr(w),
                                           _lib.stream_ptr()), "fm_spatial_init")
    if init == "circular":  # spatial.py:109-121
        g = torch.full((N, F, M), 1e-2, dtype=torch.float64, device=X1.device)
        for m in range(M):
            g[m % N, :, m] = 1.0
    else:  # "observed": init_spatial diagonalizable (spatial.py:100-105)
        g = torch.ones((N, F, M), dtype=torch.float64, device=X1.device)
        g[0] = torch.maximum(w, w.max(dim=-1, keepdim=True).values * 1e-12)
    Nn = N if n_nmf is None else n_nmf  # DP: the noise NMF holds n_sources - 1
    Wn = rng.uniform(0.1, 1.1, (Nn, F, cfg.n_basis))  # sources.py:180-181
    Hn = rng.uniform(0.1, 1.1, (Nn, cfg.n_basis, T))
    return Q, g, torch.from_numpy(Wn), torch.from_numpy(Hn)


# ---------------------------------------------------------------------------
# run
# ---------------------------------------------------------------------------

def _check_method(cfg):
    if cfg.method not in SUPPORTED_METHODS:
        raise InvalidInputError(
            f"method {cfg.method!r} is outside this backend's hot path; "
            f"supported: {SUPPORTED_METHODS}")


def _prepare_observation(X, cfg, torch):
    """separate.py:284-293 + spatial.py:64-66 on the device: returns
    (Xs device (B,F,T,M), scale (B,) np, floor (B,) tensor)."""
    cdt = torch.complex64 if cfg.precision == "complex64" else torch.complex128
    if isinstance(X, torch.Tensor):
        Xd = X.to(device=cfg.device, dtype=cdt).contiguous()
        if Xd.data_ptr() == X.data_ptr():  # never scale the caller's tensor in place
            Xd = Xd.clone()
    else:  # host numpy: copy at its own width, convert on the device (non-finite values
        # surface in the device power statistics below)
        Xn = np.ascontiguousarray(np.asarray(X))
        if not np.iscomplexobj(Xn):
            Xn = Xn.astype(np.complex128)
        Xd = torch.from_numpy(Xn).to(cfg.device).to(cdt).contiguous()
    if Xd.dim() == 3:
        Xd = Xd.unsqueeze(0)
    B, F, T, M = Xd.shape
    dims = _lib.FmDims(B, F, T, M, 1, 1, 0,
                       _lib.FM_F32 if cdt == torch.complex64 else _lib.FM_F64, 1, 1, 0)
    lib = _lib.load()
    sumsq = (ctypes.c_double * B)()
    maxsq = (ctypes.c_double * B)()
    _lib.check(lib.fm_observation_stats(ctypes.byref(dims), _lib.ptr(Xd), sumsq, maxsq,
                                        _lib.stream_ptr()), "fm_observation_stats")
    power = np.array(sumsq[:]) / float(F * T * M)
    if not np.all(np.isfinite(power)):
        raise InvalidInputError("observation contains non-finite values")
    if np.any(power == 0.0):
        raise InvalidInputError("observation is identically zero")
    scale = np.sqrt(power)
    sc = (ctypes.c_double * B)(*scale.tolist())
    _lib.check(lib.fm_scale_observation(ctypes.byref(dims), _lib.ptr(Xd), sc, _lib.stream_ptr()),
               "fm_scale_observation")
    _lib.check(lib.fm_observation_stats(ctypes.byref(dims), _lib.ptr(Xd), sumsq, maxsq,
                                        _lib.stream_ptr()), "fm_observation_stats")
    floor = torch.tensor([1e-12 * v for v in maxsq[:]], dtype=torch.float64)  # spatial.py:64-66
    return Xd, scale, floor.to(cfg.device)


def _to_host(t, wait=True):
    """Device tensor -> host tensor in page-locked memory from torch's caching
    host allocator: one async DMA at full PCIe/C2C speed and no host-side copy
    (a plain .cpu() of a large tensor runs at pageable-DMA speed, and a copy
    into fresh pageable memory pays first-touch page faults). The returned
    tensor (and any numpy view of it) owns the pinned block; when it is freed
    the block goes back to the allocator's cache for the next call."""
    torch = _torch()
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t.contiguous(), non_blocking=True)
    if wait:
        torch.cuda.current_stream().synchronize()
    return out


def _as_batch(a, torch, B):
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a))
    if t.dim() == 3:
        t = t.unsqueeze(0).expand(B, *t.shape)
    return t


def run(cfg: SeparatorConfig, X_FTM, on_iteration=None, init=None) -> SeparationResult:
    """fastsep.run (separate.py:276-330) for method="fast-mnmf".

    ``init`` optionally injects the initial (Q_FMM, g_NFM, W_NFK, H_NKT) in
    the scaled domain -- where the reference's _build_spatial/_build_source
    place theirs; by default the reference's own init is used.
    The input is never modified. Everything runs on ``cfg.device``.
    """
    cfg.validate()
    _check_method(cfg)
    torch = _torch()
    with torch.cuda.device(torch.device(cfg.device)):
        return _run(cfg, X_FTM, on_iteration, init, torch)


def _run(cfg, X_FTM, on_iteration, init, torch):
    if not isinstance(X_FTM, torch.Tensor):
        Xn = np.asarray(X_FTM)
        if Xn.ndim != 3:
            raise InvalidInputError(f"observation must have shape (F, T, M), got {Xn.shape}")
    elif X_FTM.dim() != 3:
        raise InvalidInputError(f"observation must have shape (F, T, M), got {tuple(X_FTM.shape)}")
    Xs, scale, floor = _prepare_observation(X_FTM, cfg, torch)
    rng = np.random.default_rng(cfg.seed)  # separate.py:295
    if cfg.method == "mnmf":
        return _run_mnmf(cfg, Xs, scale, rng, on_iteration, init)
    dp = None
    if cfg.method == "fast-mnmf-dp":
        from .dp import ToyDecoder, decoder_kind

        F, T = Xs.shape[1], Xs.shape[2]
        # the reference's default decoder (separate.py:265)
        decoder = cfg.decoder if cfg.decoder is not None else ToyDecoder(F)
        if getattr(decoder, "n_freq", F) != F:  # separate.py:266-270
            raise InvalidInputError(f"decoder output length {decoder.n_freq} does not match F={F}")
        kind = decoder_kind(decoder)
        if kind is None:
            raise InvalidInputError("the B200 deep prior needs a ToyDecoder (w1, b1, w2, b2) or an "
                                    "ExpMLPDecoder (W1, b1, W2, b2, W3, b3)")
        update = cfg.latent_update
        if update == "auto":  # the reference's chain for its decoder, Adam for config 4's
            update = "metropolis" if kind == 1 else "adam"
        if update == "adam" and kind != 0:
            raise InvalidInputError("latent_update='adam' needs an ExpMLPDecoder")
        if init is None:
            Q0, g0, W0, H0 = default_init(cfg, Xs[0], rng, n_nmf=cfg.n_sources - 1)
            u0, v0 = np.ones(F), np.ones(T)  # DeepPriorPlusNmfSource.init (sources.py:240-244)
            z0 = np.zeros((T, decoder.latent_dim))
        else:
            Q0, g0, u0, v0, z0, W0, H0 = init
        on = cfg.metropolis_enabled  # separate.py:205
        adam = cfg.adam_steps if (on and update == "adam") else 0
        mh = cfg.metropolis.inner_steps if (on and update == "metropolis") else 0
        mh_rng = rng if cfg.metropolis_rng == "numpy" else None
        dp = (decoder, u0, v0, z0, adam, cfg.adam_lr, mh, cfg.metropolis.proposal_var, mh_rng,
              cfg.seed)
    elif init is None:
        Q0, g0, W0, H0 = default_init(cfg, Xs[0], rng)
    else:
        Q0, g0, W0, H0 = init
    loop = DeviceLoop(Xs, _as_batch(Q0, torch, 1), _as_batch(g0, torch, 1),
                      _as_batch(W0, torch, 1), _as_batch(H0, torch, 1), floor,
                      cfg.normalize, cfg.ip_sweeps, n_trace=cfg.n_iterations, dp=dp)
    loop.prologue()
    time_trace = []
    start = torch.cuda.Event(enable_timing=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(cfg.n_iterations)]
    start.record()
    for it in range(cfg.n_iterations):
        loop.run(1, use_graph=cfg.use_graph)
        ev[it].record()
        if on_iteration is not None:
            torch.cuda.synchronize()
            err = loop.status_error()
            if err is not None:
                raise err
            on_iteration(it, loop)
    torch.cuda.synchronize()
    err = loop.status_error()
    if err is not None:
        raise err
    # images at the run's precision (complex64 runs return complex64), in pinned host
    # memory: the Wiener kernels and the DMA are queued first, the host-side trace
    # bookkeeping runs while they do, the one wait comes last
    imgs, sts = loop.images_batch(scale, defer_status=True)
    images_t = _to_host(imgs[0], wait=False)
    prev = start
    for e in ev:  # per-iteration device time (separate.py:307-312 analogue)
        time_trace.append(prev.elapsed_time(e) / 1e3)
        prev = e
    ll = loop.trace[:, 0].cpu().numpy().copy() if cfg.record_likelihood else np.zeros(0)
    torch.cuda.current_stream().synchronize()
    for st in sts:
        K.check_wiener_status(st)
    images = images_t.numpy()
    res = SeparationResult(images_NFTM=images, likelihood_trace=np.asarray(ll),
                           time_trace=np.asarray(time_trace), method=cfg.method,
                           config=replace(cfg))
    res.loop = loop
    return res


def _run_mnmf(cfg, Xs, scale, rng, on_iteration, init):
    """run() (separate.py:276-330) for method="mnmf": the _FullRankLoop
    (separate.py:128-172) on the device (fullrank.FullRankDeviceLoop).
    ``init`` optionally injects (G_NFMM, W_NFK, H_NKT) in the scaled domain;
    by default the reference's init: circular_init -> reconstruct_scm
    (separate.py:246-256) and NmfSource.random from the run's rng."""
    from . import fullrank as FR

    torch = _torch()
    X1 = Xs[0]
    F, T, M = X1.shape
    if M > 8:
        raise InvalidInputError(f"the full-rank model supports M <= 8, got M={M}")
    if init is None:
        Q0, g0, W0, H0 = default_init(cfg, X1, rng)  # device Q (F,M,M), g (N,F,M)
        G0 = FR.reconstruct_scm(Q0.to("cuda", X1.dtype),
                                torch.as_tensor(g0).to("cuda", torch.float64 if X1.dtype ==
                                                       torch.complex128 else torch.float32))
    else:
        G0, W0, H0 = init
    G0 = G0 if isinstance(G0, torch.Tensor) else torch.from_numpy(np.asarray(G0))
    W0 = W0 if isinstance(W0, torch.Tensor) else torch.from_numpy(np.asarray(W0))
    H0 = H0 if isinstance(H0, torch.Tensor) else torch.from_numpy(np.asarray(H0))
    # mixture_ridge (spatial.py:59-61) of the scaled observation
    dims = _lib.FmDims(1, F, T, M, 1, 1, 0,
                       _lib.FM_F32 if X1.dtype == torch.complex64 else _lib.FM_F64, 1, 1, 0)
    sumsq, maxsq = (ctypes.c_double * 1)(), (ctypes.c_double * 1)()
    _lib.check(_lib.load().fm_observation_stats(ctypes.byref(dims), _lib.ptr(X1), sumsq, maxsq,
                                                _lib.stream_ptr()), "fm_observation_stats")
    ridge = 1e-12 * sumsq[0] / float(F * T * M)
    loop = FR.FullRankDeviceLoop(X1, G0, W0, H0, ridge, cfg.normalize, n_trace=cfg.n_iterations)
    time_trace = []
    for it in range(cfg.n_iterations):
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        loop.iterate()
        end.record()
        err = loop.status_error()  # synchronises
        if err is not None:
            raise type(err)(f"iteration {it}: {err}")
        time_trace.append(start.elapsed_time(end) / 1e3)
        if on_iteration is not None:
            on_iteration(it, loop)
    loop.final_loglik()
    ll = loop.ll[1:cfg.n_iterations + 1].cpu().numpy().copy() if cfg.record_likelihood else np.zeros(0)
    images = _to_host(loop.images(scale[0])).numpy()
    res = SeparationResult(images_NFTM=images, likelihood_trace=np.asarray(ll),
                           time_trace=np.asarray(time_trace), method=cfg.method,
                           config=replace(cfg))
    res.loop = loop
    return res


@dataclass
class BatchSeparationResult:
    """run_batch output: per-mixture results of B independent runs."""

    images_BNFTM: object
    likelihood_trace: np.ndarray  # (B, n_iterations)
    seconds: float
    config: SeparatorConfig
    loop: object = None


def run_batch(cfg: SeparatorConfig, X_BFTM, init, want_images=True) -> BatchSeparationResult:
    """B independent fast-mnmf runs in lock-step on one device (BASELINE
    config 2); equal to B separate ``run`` calls."""
    cfg.validate()
    if cfg.method != "fast-mnmf":
        raise InvalidInputError(f"run_batch runs method='fast-mnmf' only, got {cfg.method!r}")
    torch = _torch()
    with torch.cuda.device(torch.device(cfg.device)):
        return _run_batch(cfg, X_BFTM, init, want_images, torch)


def _run_batch(cfg, X_BFTM, init, want_images, torch):
    Xs, scale, floor = _prepare_observation(X_BFTM, cfg, torch)
    Q0, g0, W0, H0 = init
    B = Xs.shape[0]
    loop = DeviceLoop(Xs, _as_batch(Q0, torch, B), _as_batch(g0, torch, B),
                      _as_batch(W0, torch, B), _as_batch(H0, torch, B), floor,
                      cfg.normalize, cfg.ip_sweeps, n_trace=cfg.n_iterations)
    loop.prologue()
    t0 = time.perf_counter()
    loop.run(cfg.n_iterations, use_graph=cfg.use_graph)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    err = loop.status_error()
    if err is not None:
        raise err
    imgs = torch.stack(loop.images_batch(scale)) if want_images else None
    ll = loop.trace.cpu().numpy().T if cfg.record_likelihood else np.zeros((B, 0))
    return BatchSeparationResult(images_BNFTM=imgs, likelihood_trace=ll,
                                 seconds=dt, config=replace(cfg), loop=loop)
