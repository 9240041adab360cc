#!/usr/bin/env python
"""FastMNMF throughput on B200 (BASELINE.json metric: iterations/s and
TF-bin*channel updates/s; roofline fraction; CPU baseline).

Default workload (N=1): BASELINE config 1 -- one mixture, F=513, T=1024, M=8,
N=4, K=16, complex64, 100 iterations. A *step* is one full fit: prologue +
100 FastMNMF iterations over the device-resident mixture (CUDA-graph replays
of the 6-launch iteration). L2 (126 MB) is flushed between timed steps with a
256 MiB write; each step is bracketed by its own CUDA events.

--gpus N under torchrun: config 1 is a single-mixture problem that does not
shard, so every rank runs an independent replica (weak scaling, "replicas
only"); ``--config c2`` shards the 256-mixture batch across ranks and
``--config c3`` shards the long recording by frequency with one NCCL
all-reduce of the H statistics per iteration.

--impl reference: the unmodified reference package (fastsep, pip-installed
into baseline/_ref) on the host cores, rank 0 only, one iteration per step
(bounded sample), same metric and units; config 4's Adam latent update has
no reference implementation and runs the numpy restatement (oracle/).
"""

import argparse
import contextlib
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CONFIGS = {
    "c1": dict(F=513, T=1024, M=8, N=4, K=16, B=1, iters=100, precision="complex64"),
    "c2": dict(F=513, T=512, M=4, N=3, K=8, B=256, iters=100, precision="complex64"),
    "c3": dict(F=1025, T=8192, M=16, N=6, K=32, B=1, iters=100, precision="complex64"),
    "c0": dict(F=257, T=128, M=4, N=2, K=8, B=1, iters=50, precision="complex128"),
    "c4": dict(F=513, T=512, M=8, N=2, K=32, B=1, iters=100, precision="complex64", dp=True),
    # config-4 shape on the reference's own default latent path: ToyDecoder +
    # Metropolis (30 proposals/iteration, device Philox draws)
    "c4mh": dict(F=513, T=512, M=8, N=2, K=32, B=1, iters=100, precision="complex64", dp=True,
                 mh=True),
}
METRIC = "FastMNMF TF-bin*ch updates/s (F*T*M*mixtures*iterations/s)"
UNIT = "TF-bin*ch/s"


@contextlib.contextmanager
def _stdout_to_stderr():
    """File descriptor 1 -> 2 for the duration: native libraries (NCCL's version
    banner) write to stdout, where the contract wants exactly one JSON line."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        yield
    finally:
        os.dup2(saved, 1)
        os.close(saved)


def _free_port():
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_problem(cfg, seed, torch, dev):
    """Synthetic mixture(s) of the config-0 generator and the BASELINE init."""
    from paper_1903_03237_b200.synth import baseline_init, make_mixture, make_mixture_torch

    F, T, M, N, K, B = cfg["F"], cfg["T"], cfg["M"], cfg["N"], cfg["K"], cfg["B"]
    cdt = torch.complex64 if cfg["precision"] == "complex64" else torch.complex128
    Xs, inits = [], []
    for b in range(B):
        if F * T * M * N <= 20_000_000:
            X = torch.from_numpy(make_mixture(F, T, M, N, K, seed + b)).to(dev, cdt)
        else:
            X = make_mixture_torch(F, T, M, N, K, seed + b, device=dev, dtype=cdt)
        Xs.append(X)
        inits.append(baseline_init(F, T, M, N, K, seed + b))
    X = torch.stack(Xs)
    init = tuple(torch.from_numpy(np.stack([i[k] for i in inits])) for k in range(4))
    return X, init


REF_DIR = os.path.join(REPO, "baseline", "_ref")


def _import_reference():
    """The UNMODIFIED reference package (pip-installed into baseline/_ref; see
    DESIGN.md "Reference arm"), its numba kernels cached outside the tree."""
    if not os.path.isdir(os.path.join(REF_DIR, "fastsep")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/fastsep_numba_cache")
    sys.path.insert(0, REF_DIR)
    import fastsep  # noqa: E402
    from fastsep import separate as S, sources as SRC, spatial as SP  # noqa: E402

    return fastsep, S, SRC, SP


def run_reference(args, cfg, world, rank):
    """--impl reference: the reference's own CPU implementation on the host
    cores (rank 0 only). fastsep.run() from baseline/_ref with the BASELINE
    init injected by the SURVEY §8(c) recipe (monkeypatched _build_spatial /
    _build_source -- the iteration itself is the stock code path: numba
    kernels, numpy/OpenBLAS on every host core). One step = one iteration
    (the reference's own per-iteration time_trace); --warmup iterations
    (numba JIT included) are discarded. Config 4 (Adam + exp-MLP decoder) has
    no reference implementation: that arm runs the numpy restatement."""
    if rank != 0:
        return
    from paper_1903_03237_b200.synth import baseline_init, make_mixture

    F, T, M, N, K = cfg["F"], cfg["T"], cfg["M"], cfg["N"], cfg["K"]
    ref = _import_reference()
    n_it = args.warmup + args.steps
    kind, dts = "reference", None
    if cfg.get("dp") and not cfg.get("mh") or ref is None:
        kind = "port"
    if kind == "reference":
        fastsep, S, SRC, SP = ref
        orig = (S._build_spatial, S._build_source)
        if cfg.get("dp"):  # c4mh: the reference's own ToyDecoder + Metropolis chain
            from oracle.fastmnmf_dp_oracle import dp_init, make_dp_mixture

            dec = SRC.ToyDecoder(F)
            X = make_dp_mixture(F, T, M, K, dec, 0).astype(np.complex64).astype(np.complex128)
            Q0, g0, u0, v0, z0, W0, H0 = dp_init(F, T, M, K, dec.latent_dim, 0)
            S._build_spatial = lambda c, Xs: SP.DiagSpatial(Q0.copy(), g0.copy())
            S._build_source = lambda c, Xs, rng: SRC.DeepPriorPlusNmfSource(
                SRC.DeepPriorFactors(u0.copy(), v0.copy(), z0.copy()),
                SRC.NmfSource(W0.copy(), H0.copy()), dec)
            rcfg = fastsep.SeparatorConfig(method="fast-mnmf-dp", n_sources=2, n_basis=K,
                                           n_iterations=n_it, seed=0)
        else:
            X = make_mixture(F, T, M, N, K, 0)
            if cfg["precision"] == "complex64":
                X = X.astype(np.complex64).astype(np.complex128)
            Q0, g0, W0, H0 = baseline_init(F, T, M, N, K, 0)
            S._build_spatial = lambda c, Xs: SP.DiagSpatial(Q0.copy(), g0.copy())
            S._build_source = lambda c, Xs, rng: SRC.NmfSource(W0.copy(), H0.copy())
            rcfg = fastsep.SeparatorConfig(method="fast-mnmf", n_sources=N, n_basis=K,
                                           n_iterations=n_it, seed=0)
        try:
            res = fastsep.run(rcfg, X)
        finally:
            S._build_spatial, S._build_source = orig
        dts = np.asarray(res.time_trace, dtype=np.float64)[args.warmup:]
        sample = (f"{args.steps} iterations of {args.config} after {args.warmup} warm-up (numba "
                  "JIT included there), unmodified fastsep.run from baseline/_ref (numba kernels "
                  "single-threaded, numpy/OpenBLAS on all host cores)")
    else:
        from oracle.fastmnmf_oracle import run_fastmnmf

        if cfg.get("dp"):
            from oracle import fastmnmf_dp_oracle as DO

            dec = DO.ExpMLPDecoder(F, seed=0)
            X = DO.make_dp_mixture(F, T, M, K, dec, 0).astype(np.complex64).astype(np.complex128)
            init = DO.dp_init(F, T, M, K, dec.latent_dim, 0)

            def one():
                DO.run_fastmnmf_dp(X, *init, dec, 1, adam_steps=10, hook=None, want_images=False)
        else:
            X = make_mixture(F, T, M, N, K, 0)
            if cfg["precision"] == "complex64":
                X = X.astype(np.complex64).astype(np.complex128)
            init = baseline_init(F, T, M, N, K, 0)

            def one():
                run_fastmnmf(X, *init, n_iterations=1, want_images=False)
        for _ in range(args.warmup):
            one()
        dl = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            one()
            dl.append(time.perf_counter() - t0)
        dts = np.asarray(dl)
        sample = (f"{args.steps} single iterations of {args.config} after {args.warmup} warm-up, "
                  "numpy restatement of the reference path (oracle/, fp64)"
                  + ("; config 4's Adam/exp-MLP latent update has no reference implementation"
                     if cfg.get("dp") else "; baseline/_ref missing"))
    dt = float(np.mean(dts))
    value = F * T * M / dt
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config-0 generator, seed 0)",
        "config": {"workload": f"{args.config}: F={F} T={T} M={M} N={N} K={K}, "
                               "one FastMNMF iteration per step (bounded CPU sample)"},
        "iters_per_s": 1.0 / dt,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(cfg, n_iter=2):
    from oracle.fastmnmf_oracle import run_fastmnmf
    from paper_1903_03237_b200.synth import baseline_init, make_mixture

    F, T, M, N, K = cfg["F"], cfg["T"], cfg["M"], cfg["N"], cfg["K"]
    X = make_mixture(F, T, M, N, K, 0)
    init = baseline_init(F, T, M, N, K, 0)
    run_fastmnmf(X[:, :64], init[0], init[1], init[2], init[3][:, :, :64], 1, want_images=False)
    t0 = time.perf_counter()
    run_fastmnmf(X, *init, n_iterations=n_iter, want_images=False)
    dt = (time.perf_counter() - t0) / n_iter
    return {"value": F * T * M / dt, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"{n_iter} FastMNMF iterations of the full config ({F}x{T}x{M}) with the "
                      "numpy oracle (fp64; einsum single-threaded, BLAS on all cores)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS))
    ap.add_argument("--shard", action="store_true",
                    help="c3: frequency-sharded path even at one rank (NCCL group of 1)")
    ap.add_argument("--iters", type=int, default=None, help="override iterations per step")
    ap.add_argument("--mixtures", type=int, default=None, help="c2: override the batch size (A/B runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.config_given = args.config is not None
    args.config = args.config or "c1"
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.iters:
        cfg["iters"] = args.iters
    if args.mixtures and args.config == "c2":
        cfg["B"] = args.mixtures
    world, rank, local = dist_env()
    if world > 1 and not args.config_given:
        # N > 1 measures the config that shards with an exchange: the long
        # recording (config 3) split by frequency (strong scaling)
        args.config = "c3"
        cfg = dict(CONFIGS["c3"])
        if args.iters:
            cfg["iters"] = args.iters

    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return

    import ctypes


    import torch
    import torch.distributed as dist

    from paper_1903_03237_b200 import _lib
    from paper_1903_03237_b200.dist import shard_batch, shard_range
    from paper_1903_03237_b200.separate import DeviceLoop, SeparatorConfig, _prepare_observation, run

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        with _stdout_to_stderr():  # NCCL's version banner goes to stdout at communicator init
            dist.init_process_group("nccl", device_id=dev)
            dist.all_reduce(torch.zeros(1, device=dev))
            torch.cuda.synchronize()
    lib = _lib.load()

    F, T, M, N, K, iters = cfg["F"], cfg["T"], cfg["M"], cfg["N"], cfg["K"], cfg["iters"]
    B_total = cfg["B"]
    sharded_f = args.config == "c3" and (world > 1 or args.shard)
    if sharded_f and world == 1:
        with _stdout_to_stderr():
            dist.init_process_group("nccl", device_id=dev, rank=0, world_size=1,
                                    init_method=f"tcp://127.0.0.1:{_free_port()}")
            dist.all_reduce(torch.zeros(1, device=dev))
            torch.cuda.synchronize()
    if args.config == "c2":
        b0, b1 = shard_batch(B_total, rank, world)
        cfg["B"] = b1 - b0
        seed0 = b0
    else:
        seed0 = 0 if args.config == "c3" else rank
    X, init = make_problem(cfg, seed0, torch, dev)
    scfg = SeparatorConfig(n_sources=N, n_basis=K, n_iterations=iters,
                           precision=cfg["precision"])
    allreduce = None
    f_off = 0
    if sharded_f:
        from paper_1903_03237_b200.dist import FrequencyShardedRun

        f0, f1 = shard_range(F, rank, world)
        Xl = X[:, f0:f1].contiguous()
        initl = (init[0][:, f0:f1], init[1][:, :, f0:f1], init[2][:, :, f0:f1], init[3])
        runner = FrequencyShardedRun(Xl, initl, F, rank, world, n_iterations=iters)
        loop = runner.loop
        Xs = Xl
        f_off = f0
    elif cfg.get("dp"):
        from paper_1903_03237_b200.dp import ExpMLPDecoder
        from paper_1903_03237_b200.synth import dp_init, make_dp_mixture

        from paper_1903_03237_b200.dp import ToyDecoder

        dec = ToyDecoder(F) if cfg.get("mh") else ExpMLPDecoder(F, seed=0)
        X = torch.from_numpy(make_dp_mixture(F, T, M, K, dec, 0)).to(dev, torch.complex64)[None]
        Q0, g0, u0, v0, z0, W0, H0 = dp_init(F, T, M, K, dec.latent_dim, 0)
        init = tuple(torch.from_numpy(a)[None] for a in (Q0, g0, W0, H0))
        Xs, scale, floor = _prepare_observation(X, scfg, torch)
        latent = (0, 1e-2, 30, 1e-4, None, 0) if cfg.get("mh") else (10, 1e-2)
        loop = DeviceLoop(Xs, init[0], init[1], init[2], init[3], floor, True, 1, n_trace=iters,
                          dp=(dec, u0, v0, z0) + latent)
        dp_init_dev = [t.clone() for t in (loop.dp.u, loop.dp.v, loop.dp.z)]
    else:
        Xs, scale, floor = _prepare_observation(X, scfg, torch)
        loop = DeviceLoop(Xs, init[0], init[1], init[2], init[3], floor, True, 1, n_trace=iters)
    init_dev = [t.to(dev, d.dtype) for t, d in zip(init if not sharded_f else initl,
                                                   (loop.Q, loop.g, loop.W, loop.H))]
    def reset():
        loop.Q.copy_(init_dev[0].reshape(loop.Q.shape))
        loop.g.copy_(init_dev[1].reshape(loop.g.shape))
        loop.W.copy_(init_dev[2].reshape(loop.W.shape))
        loop.H.copy_(init_dev[3].reshape(loop.H.shape))
        loop.status.fill_(-1)
        loop.iterations_done = 0
        if loop.dp is not None:
            for dst, src in zip((loop.dp.u, loop.dp.v, loop.dp.z), dp_init_dev):
                dst.copy_(src)
            loop.dp.m.zero_()
            loop.dp.v2.zero_()
            loop.dp.step.zero_()

    use_graph = True  # sharded: phase 0 + NCCL all-reduce + phase 1 in one graph
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step():
        loop.prologue()
        loop.run(iters, use_graph=use_graph)

    for _ in range(args.warmup):
        reset()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for i in range(args.steps):
        reset()
        flush.fill_(i & 0xFF)  # write 256 MiB > L2 between timed steps
        ev[i][0].record()
        step()
        ev[i][1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    err = loop.status_error()
    if err is not None:
        raise err
    # whole-job units: every rank's mixtures (c1 replicas, c2 batch shards) or the
    # one sharded recording (c3) -- F*T*M*B*iterations per step
    if args.config == "c2":
        units = F * T * M * B_total * iters
    elif sharded_f:
        units = F * T * M * iters
    else:
        units = F * T * M * cfg["B"] * iters * world
    value = units / (ms_per_step / 1e3)
    iters_per_s = iters / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel: per-kernel device times from CUDA
    # event-record nodes between the launches of one graph-replayed iteration
    # (the production path), median of nprof replays
    rs = 4 if cfg["precision"] == "complex64" else 8
    Bl = cfg["B"]
    ftm = F * T * M * Bl if not sharded_f else (loop.F * T * M)
    nprof = 10
    if loop.dp is None:
        sched = int(lib.fm_schedule(ctypes.byref(loop.dims)))  # 0 split, 1 fused, 2 per-bin
        names = (["k_hpass", "k_gpass", "k_vacc", "k_ip", "k_bpass", "k_trace"] if sched == 1 else
                 ["k_hstats", "k_binw", "k_trace"] if sched == 2 else
                 ["k_wstats", "k_lambda", "k_phi", "k_hstats", "k_lambda", "k_gain", "k_vacc",
                  "k_ip", "k_back", "k_trace"])
        samples = []
        if not sharded_f:
            ms = (ctypes.c_float * 16)()
            nint = ctypes.c_int(0)
            for _ in range(nprof):
                reset()
                loop.prologue()
                _lib.check(lib.fm_iterate_profiled(ctypes.byref(loop.dims), ctypes.byref(loop.state),
                                                   ms, ctypes.byref(nint), _lib.stream_ptr()),
                           "fm_iterate_profiled")
                samples.append(list(ms[:nint.value]))
    else:
        lat = "k_dp_mh" if cfg.get("mh") else "k_dp_latent"
        names = ["k_lambda", "k_dp_lambda", lat, "k_dp_lambda", "k_phi", "k_dp_umu", "k_dp_lambda",
                 "k_phi", "k_dp_vmu", "k_dp_lambda", "k_phi", "k_wstats", "k_lambda", "k_phi",
                 "k_hstats", "k_lambda", "k_gain", "k_vacc", "k_ip", "k_back", "k_trace"]
        samples = []
        ms = (ctypes.c_float * 24)()
        nint = ctypes.c_int(0)
        for _ in range(nprof):
            reset()
            loop.prologue()
            _lib.check(lib.fm_iterate_dp_profiled(ctypes.byref(loop.dims), ctypes.byref(loop.state),
                                                  ctypes.byref(loop.dp.struct), ms, ctypes.byref(nint),
                                                  _lib.stream_ptr()), "fm_iterate_dp_profiled")
            samples.append(list(ms[:nint.value]))
    kernel_ms = {}
    if samples:
        med = np.median(np.array(samples), axis=0)
        for n_, v in zip(names, med):  # launches of the same kernel summed per iteration
            kernel_ms[n_] = kernel_ms.get(n_, 0.0) + float(v)
    dom = max(kernel_ms, key=kernel_ms.get) if kernel_ms else None
    launches_of = {n_: names.count(n_) for n_ in kernel_ms}
    # algorithmic bytes per launch: x~ reads (P1-P3), X reads
    # (P4, P5) and the x~ write (P5); lambda / phi / y are on-chip by definition
    FT = ftm // M
    alg_tab = {
        "k_wstats": 0, "k_hstats": 0, "k_lambda": 0,  # phi / lambda traffic: not algorithmic
        "k_hpass": ftm * rs,                  # read x~ (H step)
        "k_gpass": ftm * rs,                  # read x~ (gain step)
        "k_vacc": ftm * 2 * rs,               # read X (V accumulation)
        "k_bpass": ftm * 3 * rs,              # read X, write x~ (projection + next W step)
        "k_back": ftm * 3 * rs,               # deep prior: read X, write x~
        "k_binw": ftm * 7 * rs,               # read x~ (gains), X twice (V, projection), write x~
        "k_phi": ftm * rs, "k_gain": ftm * rs,
        "k_dp_latent": ftm * rs + FT * rs,    # x~ and y_rest (F,T) per Adam step
        "k_dp_mh": ftm * rs + FT * rs,
    }
    hbm, peak_kind = peaks()
    roofline = {"bound": "hbm", "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None,
                "traffic": None, "kernel": dom, "peak_kind": peak_kind,
                "kernel_ms": kernel_ms, "kernel_ms_source": "graph replay, event nodes, median of "
                f"{nprof}" if kernel_ms else None}
    if dom is not None:
        per_launch_ms = kernel_ms[dom] / launches_of[dom]
        alg = alg_tab.get(dom, 0)
        achieved = alg / (per_launch_ms / 1e3) / 1e9 if alg and per_launch_ms > 0 else None
        traffic = None
        tpath = os.path.join(REPO, "profiles", "traffic.json")
        if os.path.exists(tpath):
            traffic = json.load(open(tpath)).get(f"{args.config}:{dom}")
        roofline.update(achieved=achieved, frac=(achieved / hbm) if achieved else None,
                        traffic=traffic, alg_bytes_per_launch=alg,
                        step_share=float(kernel_ms[dom] * iters / ms_per_step))
        if dom == "k_vacc":
            # the V accumulation is FP32-pipe bound at M >= 8: its
            # compute roofline beside the contract's HBM one. Algorithmic flops
            # per (f, t): M weights x P = M(M+1)/2 Hermitian pairs x 2 FMA (real
            # weight x complex product) + 3 FMA per pair product + the model
            # power (N M FMA), all x 2 flop/FMA
            P = M * (M + 1) // 2
            flops = 2 * (2 * P * M + 3 * P + N * M) * FT
            peak_sm = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["sm_max_mhz"]) \
                if os.path.exists(os.path.join(REPO, "MEASURED_PEAKS.json")) else 1965.0
            fp32_peak = 148 * 128 * 2 * peak_sm * 1e6 / 1e12  # TFLOP/s (FFMA, all SMs, max clock)
            ach = flops / (per_launch_ms / 1e3) / 1e12
            roofline["compute"] = {"bound": "fp32-fma", "achieved": ach, "peak": fp32_peak,
                                   "unit": "TFLOP/s", "frac": ach / fp32_peak,
                                   "alg_flops_per_launch": flops,
                                   "peak_kind": "nominal 148 SM x 128 FP32 lanes x 2 x max SM clock"}
            tc_v = (cfg["precision"] == "complex64" and M >= 10 and M % 2 == 0
                    and os.environ.get("FM_VACC") in (None, "tc"))
            if tc_v:
                # k_vacc_tc: the contraction D[j][m] = sum_t A[j][t] w[m][t] (M*M real rows,
                # M weights) runs as 3xTF32 tcgen05 MMAs; the SIMT work left is the
                # operand build. Against the TF32 tensor peak (half the measured bf16
                # figure), counting the three TF32 products each fp32-class product costs.
                pk = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))) \
                    if os.path.exists(os.path.join(REPO, "MEASURED_PEAKS.json")) else {}
                tf32_peak = float(pk.get("bf16_tflops", 1675.0)) / 2
                gemm = 2 * M * M * M * FT
                roofline["compute"] = {
                    "bound": "tensor", "kind": "tf32 (3xTF32 split)",
                    "achieved": 3 * gemm / (per_launch_ms / 1e3) / 1e12, "peak": tf32_peak,
                    "unit": "TFLOP/s", "frac": 3 * gemm / (per_launch_ms / 1e3) / 1e12 / tf32_peak,
                    "alg_flops_per_launch": gemm, "issued_flops_per_launch": 3 * gemm,
                    "peak_kind": "measured bf16 cuBLAS peak / 2",
                    "note": "shape-limited: N = M = 16 weight columns per MMA (M=128 x N=32|16 x K=8)"}
    # whole iteration against B_it = (4 b_r + 2 b_c) F T M per mixture
    b_it = 8 * rs * (F * T * M * (B_total if args.config == "c2" else Bl))
    it_s = ms_per_step / 1e3 / iters
    roofline["iteration"] = {"B_it": b_it, "ms": it_s * 1e3, "achieved": b_it / it_s / 1e9,
                             "frac": b_it / it_s / 1e9 / hbm,
                             "kernel_ms_sum": float(sum(kernel_ms.values())) if kernel_ms else None}

    # ---- e2e: the public API call with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e and not sharded_f and args.config in ("c1", "c0"):
        Xh = X[0].cpu().pin_memory()
        # warm: two results alive at once, as in the timed loop below (the pinned
        # image blocks come from torch's caching host allocator)
        w1 = run(scfg, Xh, init=tuple(a[0].numpy() for a in init))
        w2 = run(scfg, Xh, init=tuple(a[0].numpy() for a in init))
        del w1
        w1 = run(scfg, Xh, init=tuple(a[0].numpy() for a in init))
        del w1, w2
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()  # every replica's e2e calls run concurrently
        reps = 9
        prof = None
        if os.environ.get("BENCH_E2E_PROFILE"):
            import cProfile

            prof = cProfile.Profile()
            prof.enable()
        calls = []
        for _ in range(reps):  # per-call wall times; the median is reported (robust to a
            t0 = time.perf_counter()  # stray host hiccup), every call is listed
            res = run(scfg, Xh, init=tuple(a[0].numpy() for a in init))
            calls.append(time.perf_counter() - t0)
        dt = float(np.median(calls))
        if world > 1:  # whole-job: the slowest replica's wall time, all replicas' units
            tdt = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(tdt, op=dist.ReduceOp.MAX)
            dt = float(tdt.item())
        if prof is not None:
            import pstats

            prof.disable()
            pstats.Stats(prof, stream=sys.stderr).sort_stats("cumulative").print_stats(20)
        cb = 8 if cfg["precision"] == "complex64" else 16
        # bytes per step of the whole job (every replica copies its own)
        h2d = (F * T * M * cb + F * M * M * 16 + N * F * M * 8 + N * F * K * 8 + N * K * T * 8) * world
        d2h = (N * F * T * M * cb + iters * 8) * world
        e2e = {"value": F * T * M * iters * world / dt, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "seconds_per_step": dt,
               "seconds_per_call": [round(c, 5) for c in calls],
               "api": "paper_1903_03237_b200.run(SeparatorConfig, X_host_pinned, init=...)"}
        del res

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config in ("c1", "c0"):
        cpu = cpu_baseline_sample(cfg)

    # per iteration, split schedule: k_wstats, k_lambda, k_phi, k_hstats, k_lambda,
    # k_gain, k_vacc, k_ip, k_back, k_trace; fused: k_hpass, k_gpass, k_vacc,
    # k_ip, k_bpass, k_trace (+ the counter advance when B > 1); prologue 2
    sched_names = {0: "split", 1: "fused", 2: "bin"}
    sched = 0 if loop.dp is not None else int(lib.fm_schedule(ctypes.byref(loop.dims)))
    per_it = {0: 10, 1: 6, 2: 3}[sched]
    launches = args.steps * (2 + (per_it if cfg['B'] == 1 else per_it + 1) * iters)
    if sharded_f:  # + the H update after the all-reduce
        launches = args.steps * (2 + (per_it + 1) * iters)
    if cfg.get("dp"):  # 21 per iteration (one latent-hook launch: Adam or Metropolis), 5 in the prologue
        launches = args.steps * (5 + 21 * iters)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak" if not sharded_f else "strong", "vs_baseline": None,
            "dtype": "f32" if cfg["precision"] == "complex64" else "f64",
            "data": "synthetic (BASELINE config-0 generator: Gamma NMF PSDs, random full-rank "
                    "SCMs, circular Gaussian excitation; seeded)",
            "config": {"workload": f"{args.config}: F={F} T={T} M={M} N={N} K={K} "
                                   f"mixtures={B_total if args.config == 'c2' else cfg['B']} "
                                   f"{cfg['precision']}, {iters} iterations per step",
                       "parallelism": ("frequency-sharded" if sharded_f else
                                       "batch-sharded" if args.config == "c2" else "replicas")
                                      + f" x{world}",
                       "l2": "flushed between steps (256 MiB write)",
                       "schedule": sched_names[sched]},
            "iters_per_s": iters_per_s, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1 or sharded_f:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
